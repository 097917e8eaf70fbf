// Transports of the partitioned solve: halo exchange, parent broadcast, scalar allreduce.
#pragma once
#include <memory>
#include <vector>

#include "octmg_internal.cuh"
#include "partition.h"

namespace octmg {

// device copy of the halo item lists a part sends / receives, with packing buffers
struct PartLinks {
  // per (level, peer): items this part sends to peer / receives from peer
  std::vector<int2*> send_items, recv_items;  // [level * nranks + peer]
  std::vector<int*> send_offs, recv_offs;     // float offsets of the items (exclusive scan)
  std::vector<int> send_n, recv_n;            // item counts
  std::vector<int> send_floats, recv_floats;  // buffer sizes
  std::vector<float*> send_buf, recv_buf;
  int parent_first[64] = {}, parent_count[64] = {};  // level lg-1 inner tiles each rank writes
  std::vector<void*> allocs;
  ~PartLinks();
};

struct PartPlanHolder {
  PartPlan plan;
  std::vector<std::unique_ptr<PartLinks>> links;  // per part of the group
};

struct Comm {
  virtual ~Comm() {}
  // u of `level` (field selector 0) or the PCG direction (1, leaf tiles of every level)
  virtual octmg_status exchange(Group& g, int level, int field, const std::vector<Fld>& f, cudaStream_t s) = 0;
  virtual octmg_status bcast_parents(Group& g, cudaStream_t s) = 0;
  // sum Scalars fields [first, first + count) (doubles) over all parts, in place
  virtual octmg_status allreduce(Group& g, int first, int count, cudaStream_t s) = 0;
  virtual const char* name() const = 0;
};

Comm* make_loopback_comm();
Comm* make_nccl_comm(void* nccl_comm, int rank, int nranks);
octmg_status build_links(Group& g, const PartPlan& plan, cudaStream_t s);

// NCCL bootstrap (dlopen'ed libnccl.so.2; the single-GPU path never loads it)
octmg_status nccl_unique_id(void* out128);
octmg_status nccl_comm_init(int rank, int nranks, const void* id128, void** comm);
void nccl_comm_destroy(void* comm);

}  // namespace octmg
