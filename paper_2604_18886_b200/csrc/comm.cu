// Transports of the partitioned solve: packed halo exchange of face layers /
// whole tiles, broadcast of the partition parents after the restriction into the
// replicated coarse levels, and the fp64 scalar allreduce of the PCG dots.  Two
// implementations of one interface: NCCL (one process per GPU; grouped ncclSend/ncclRecv,
// ncclBroadcast, ncclAllReduce over NVLink/NVSwitch) and loopback (several parts of a
// partition living in one process on one GPU, for testing the distributed logic).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>

#include "comm.h"

namespace octmg {

namespace {

__device__ __forceinline__ int item_cell(int kind, int c) {
  if (kind == 6) return c;
  const int ax = kind >> 1;
  const int layer = (kind & 1) ? 7 : 0;
  const int o1 = ax == 0 ? 1 : 0, o2 = ax == 2 ? 1 : 2;
  int xyz[3];
  xyz[ax] = layer;
  xyz[o1] = c & 7;
  xyz[o2] = c >> 3;
  return cslot(xyz[0], xyz[1], xyz[2]);
}

__global__ void k_pack(Fld f, int NL, const int2* items, const int* offs, float* buf) {
  const int2 it = items[blockIdx.x];
  if (it.x >= NL && f.inner == nullptr) return;  // leaf-only field
  const float* src = tptr(f, it.x, NL);
  const int n = it.y == 6 ? TB3 : 64;
  float* dst = buf + offs[blockIdx.x];
  for (int c = threadIdx.x; c < n; c += blockDim.x) dst[c] = src[item_cell(it.y, c)];
}

__global__ void k_unpack(Fld f, int NL, const int2* items, const int* offs, const float* buf) {
  const int2 it = items[blockIdx.x];
  if (it.x >= NL && f.inner == nullptr) return;
  float* dst = tptr(f, it.x, NL);
  const int n = it.y == 6 ? TB3 : 64;
  const float* src = buf + offs[blockIdx.x];
  for (int c = threadIdx.x; c < n; c += blockDim.x) dst[item_cell(it.y, c)] = src[c];
}

// sum fields [first, first+count) of every part's Scalars (part order), write back to all
__global__ void k_sum_scalars(Scalars* const* scs, int nparts, int first, int count) {
  const int k = threadIdx.x;
  if (k >= count) return;
  double s = 0.0;
  for (int p = 0; p < nparts; ++p) s += reinterpret_cast<const double*>(scs[p])[first + k];
  for (int p = 0; p < nparts; ++p) reinterpret_cast<double*>(scs[p])[first + k] = s;
}

template <class T>
octmg_status dalloc(std::vector<void*>& list, T** p, size_t count) {
  void* q = dev_malloc(std::max<size_t>(count, 1) * sizeof(T));
  if (!q) {
    set_error("device allocation failed (halo buffers)");
    return OCTMG_E_OOM;
  }
  list.push_back(q);
  *p = (T*)q;
  return OCTMG_OK;
}

octmg_status upload(std::vector<void*>& allocs, const std::vector<HaloItem>& items, int2** d_items, int** d_offs,
                    int* n, int* floats) {
  std::vector<int2> it(items.size());
  std::vector<int> off(items.size());
  int acc = 0;
  for (size_t k = 0; k < items.size(); ++k) {
    it[k] = make_int2(items[k].tile, items[k].kind);
    off[k] = acc;
    acc += items[k].kind == 6 ? TB3 : 64;
  }
  *n = (int)items.size();
  *floats = acc;
  *d_items = nullptr;
  *d_offs = nullptr;
  if (items.empty()) return OCTMG_OK;
  OCTMG_TRY(dalloc(allocs, d_items, it.size()));
  OCTMG_TRY(dalloc(allocs, d_offs, off.size()));
  OCTMG_CUDA(cudaMemcpy(*d_items, it.data(), sizeof(int2) * it.size(), cudaMemcpyHostToDevice));
  OCTMG_CUDA(cudaMemcpy(*d_offs, off.data(), sizeof(int) * off.size(), cudaMemcpyHostToDevice));
  return OCTMG_OK;
}

void pack(Hier& h, PartLinks& L, int idx, const Fld& f, cudaStream_t s) {
  if (L.send_n[idx]) k_pack<<<L.send_n[idx], 128, 0, s>>>(f, h.tree->NL, L.send_items[idx], L.send_offs[idx], L.send_buf[idx]);
}

void unpack(Hier& h, PartLinks& L, int idx, const Fld& f, const float* buf, cudaStream_t s) {
  if (L.recv_n[idx]) k_unpack<<<L.recv_n[idx], 128, 0, s>>>(f, h.tree->NL, L.recv_items[idx], L.recv_offs[idx], buf);
}

// levels an exchange covers: one level of u, or every partitioned level of the direction
void levels_of(const Group& g, int level, int field, int* l0, int* l1) {
  const int lg = g.parts[0]->lg, L = g.parts[0]->tree->L;
  if (field == 0) { *l0 = level; *l1 = level; }
  else { *l0 = lg; *l1 = L; }
}

// ------------------------------------------------------------------------------------
// loopback: all parts in this process, on one device
// ------------------------------------------------------------------------------------
struct LoopbackComm : Comm {
  Scalars** d_scs = nullptr;
  ~LoopbackComm() override {
    if (d_scs) { cudaDeviceSynchronize(); dev_free(d_scs); }
  }
  const char* name() const override { return "loopback"; }
  octmg_status exchange(Group& g, int level, int field, const std::vector<Fld>& f, cudaStream_t s) override {
    const int n = (int)g.parts.size();
    int l0, l1;
    levels_of(g, level, field, &l0, &l1);
    for (int l = l0; l <= l1; ++l) {
      for (int r = 0; r < n; ++r)
        for (int q = 0; q < n; ++q)
          if (q != r) pack(*g.parts[r], *g.plan->links[r], l * n + q, f[r], s);
      for (int q = 0; q < n; ++q)
        for (int r = 0; r < n; ++r)
          if (q != r) unpack(*g.parts[q], *g.plan->links[q], l * n + r, f[q], g.plan->links[r]->send_buf[l * n + q], s);
    }
    return cuda_status_ok();
  }
  octmg_status bcast_parents(Group& g, cudaStream_t s) override {
    const int n = (int)g.parts.size();
    for (int r = 0; r < n; ++r) {
      const PartLinks& L = *g.plan->links[r];
      const int first = L.parent_first[r], cnt = L.parent_count[r];
      if (!cnt) continue;
      Hier& src = *g.parts[r];
      const size_t off = (size_t)(first - src.tree->NL) * TB3, bytes = (size_t)cnt * TB3 * sizeof(float);
      for (int q = 0; q < n; ++q) {
        if (q == r) continue;
        Hier& dst = *g.parts[q];
        OCTMG_CUDA(cudaMemcpyAsync(dst.uinA + off, src.uinA + off, bytes, cudaMemcpyDeviceToDevice, s));
        OCTMG_CUDA(cudaMemcpyAsync(dst.ustar + off, src.ustar + off, bytes, cudaMemcpyDeviceToDevice, s));
        OCTMG_CUDA(cudaMemcpyAsync(dst.binner + off, src.binner + off, bytes, cudaMemcpyDeviceToDevice, s));
      }
    }
    return OCTMG_OK;
  }
  octmg_status allreduce(Group& g, int first, int count, cudaStream_t s) override {
    const int n = (int)g.parts.size();
    if (!d_scs) {
      std::vector<Scalars*> v;
      for (Hier* h : g.parts) v.push_back(h->sc);
      d_scs = (Scalars**)dev_malloc(sizeof(Scalars*) * n);
      if (!d_scs) { set_error("device allocation failed (loopback scalars)"); return OCTMG_E_OOM; }
      OCTMG_CUDA(cudaMemcpy(d_scs, v.data(), sizeof(Scalars*) * n, cudaMemcpyHostToDevice));
    }
    k_sum_scalars<<<1, 32, 0, s>>>(d_scs, n, first, count);
    return cuda_status_ok();
  }
  static octmg_status cuda_status_ok() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? OCTMG_OK : cuda_status(e, "loopback transport");
  }
};

// ------------------------------------------------------------------------------------
// NCCL (dlopen'ed): one part per process
// ------------------------------------------------------------------------------------
struct NcclApi {
  void* lib = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  const char* (*GetErrorString)(ncclResult_t);
};

NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return nullptr;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
    api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    if (api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.AllReduce && api.Broadcast) api.lib = h;
  }
  return api.lib ? &api : nullptr;
}

#define OCTMG_NCCL(call)                                                                 \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess) {                                                             \
      set_error(std::string("NCCL error ") + nccl()->GetErrorString(r_) + " in " #call); \
      return OCTMG_E_NCCL;                                                               \
    }                                                                                    \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm;
  int rank, nranks;
  NcclComm(void* c, int r, int n) : comm((ncclComm_t)c), rank(r), nranks(n) {}
  const char* name() const override { return "nccl"; }
  octmg_status exchange(Group& g, int level, int field, const std::vector<Fld>& f, cudaStream_t s) override {
    Hier& h = *g.parts[0];
    PartLinks& L = *g.plan->links[0];
    int l0, l1;
    levels_of(g, level, field, &l0, &l1);
    for (int l = l0; l <= l1; ++l)
      for (int q = 0; q < nranks; ++q)
        if (q != rank) pack(h, L, l * nranks + q, f[0], s);
    OCTMG_NCCL(nccl()->GroupStart());
    for (int l = l0; l <= l1; ++l)
      for (int q = 0; q < nranks; ++q) {
        if (q == rank) continue;
        const int idx = l * nranks + q;
        if (L.send_floats[idx]) OCTMG_NCCL(nccl()->Send(L.send_buf[idx], L.send_floats[idx], ncclFloat32, q, comm, s));
        if (L.recv_floats[idx]) OCTMG_NCCL(nccl()->Recv(L.recv_buf[idx], L.recv_floats[idx], ncclFloat32, q, comm, s));
      }
    OCTMG_NCCL(nccl()->GroupEnd());
    for (int l = l0; l <= l1; ++l)
      for (int q = 0; q < nranks; ++q)
        if (q != rank) unpack(h, L, l * nranks + q, f[0], L.recv_buf[l * nranks + q], s);
    return OCTMG_OK;
  }
  octmg_status bcast_parents(Group& g, cudaStream_t s) override {
    Hier& h = *g.parts[0];
    PartLinks& L = *g.plan->links[0];
    OCTMG_NCCL(nccl()->GroupStart());
    for (int r = 0; r < nranks; ++r) {
      if (!L.parent_count[r]) continue;
      const size_t off = (size_t)(L.parent_first[r] - h.tree->NL) * TB3, n = (size_t)L.parent_count[r] * TB3;
      OCTMG_NCCL(nccl()->Broadcast(h.uinA + off, h.uinA + off, n, ncclFloat32, r, comm, s));
      OCTMG_NCCL(nccl()->Broadcast(h.ustar + off, h.ustar + off, n, ncclFloat32, r, comm, s));
      OCTMG_NCCL(nccl()->Broadcast(h.binner + off, h.binner + off, n, ncclFloat32, r, comm, s));
    }
    OCTMG_NCCL(nccl()->GroupEnd());
    return OCTMG_OK;
  }
  octmg_status allreduce(Group& g, int first, int count, cudaStream_t s) override {
    double* p = reinterpret_cast<double*>(g.parts[0]->sc) + first;
    OCTMG_NCCL(nccl()->AllReduce(p, p, count, ncclFloat64, ncclSum, comm, s));
    return OCTMG_OK;
  }
};

}  // namespace

PartLinks::~PartLinks() {
  for (void* p : allocs) dev_free(p);
}

Comm* make_loopback_comm() { return new LoopbackComm(); }
Comm* make_nccl_comm(void* c, int rank, int nranks) { return new NcclComm(c, rank, nranks); }

octmg_status build_links(Group& g, const PartPlan& P, cudaStream_t s) {
  (void)s;
  const int n = P.nranks;
  const bool loop = (int)g.parts.size() == n;  // loopback holds every part; NCCL one
  const int L = g.parts[0]->tree->L;
  g.plan->links.clear();
  for (Hier* h : g.parts) {
    auto lk = std::make_unique<PartLinks>();
    const int r = h->rank;
    const size_t m = (size_t)(L + 1) * n;
    lk->send_items.assign(m, nullptr); lk->recv_items.assign(m, nullptr);
    lk->send_offs.assign(m, nullptr); lk->recv_offs.assign(m, nullptr);
    lk->send_n.assign(m, 0); lk->recv_n.assign(m, 0);
    lk->send_floats.assign(m, 0); lk->recv_floats.assign(m, 0);
    lk->send_buf.assign(m, nullptr); lk->recv_buf.assign(m, nullptr);
    for (int l = P.lg; l <= L; ++l)
      for (int q = 0; q < n; ++q) {
        if (q == r) continue;
        const size_t idx = (size_t)l * n + q;
        OCTMG_TRY(upload(lk->allocs, P.list(l, r, q), &lk->send_items[idx], &lk->send_offs[idx], &lk->send_n[idx],
                         &lk->send_floats[idx]));
        OCTMG_TRY(upload(lk->allocs, P.list(l, q, r), &lk->recv_items[idx], &lk->recv_offs[idx], &lk->recv_n[idx],
                         &lk->recv_floats[idx]));
        if (lk->send_floats[idx]) OCTMG_TRY(dalloc(lk->allocs, &lk->send_buf[idx], lk->send_floats[idx]));
        if (!loop && lk->recv_floats[idx]) OCTMG_TRY(dalloc(lk->allocs, &lk->recv_buf[idx], lk->recv_floats[idx]));
      }
    for (int q = 0; q < n && q < 64; ++q) {
      const auto& pt = P.parent_tiles[q];
      lk->parent_first[q] = pt.empty() ? 0 : pt.front();
      lk->parent_count[q] = (int)pt.size();
      for (size_t k = 1; k < pt.size(); ++k)
        if (pt[k] != pt[k - 1] + 1) { set_error("partition parents are not contiguous"); return OCTMG_E_INVALID; }
    }
    g.plan->links.push_back(std::move(lk));
  }
  return OCTMG_OK;
}

octmg_status nccl_unique_id(void* out128) {
  if (!nccl()) { set_error("libnccl.so.2 not loadable"); return OCTMG_E_NCCL; }
  ncclUniqueId id;
  OCTMG_NCCL(nccl()->GetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
  return OCTMG_OK;
}

octmg_status nccl_comm_init(int rank, int nranks, const void* id128, void** comm) {
  if (!nccl()) { set_error("libnccl.so.2 not loadable"); return OCTMG_E_NCCL; }
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  ncclComm_t c;
  OCTMG_NCCL(nccl()->CommInitRank(&c, nranks, id, rank));
  *comm = c;
  return OCTMG_OK;
}

void nccl_comm_destroy(void* comm) {
  if (comm && nccl()) nccl()->CommDestroy((ncclComm_t)comm);
}

}  // namespace octmg
