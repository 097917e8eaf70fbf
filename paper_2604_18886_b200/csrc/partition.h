// Morton-range partition of the octree and halo plans (host; see partition.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace octmg {

struct PartInput {
  int L = 0, NL = 0, NI = 0;
  const int* lb;
  const int* lc;
  const int* ib;
  const int* ic;
  std::vector<int> tiles4;      // (level, i, j, k) per tile
  std::vector<int> nbr;         // 6 per tile
  std::vector<int> parent;      // per tile
  std::vector<int> child;       // 8 per inner tile
  std::vector<uint64_t> morton; // per tile (at its own level)
};

struct HaloItem {
  int tile;
  int kind;  // 0..5: face layer of that face (64 cells), 6: whole tile (512 cells)
};

struct PartPlan {
  int nranks = 1;
  int lg = 0;                                  // partition level
  std::vector<int> owner;                      // per tile: rank, -1 = replicated (level < lg)
  std::vector<std::vector<int>> lg_tiles;      // per rank: its level-lg tiles (Morton order)
  std::vector<std::vector<int>> parent_tiles;  // per rank: level-(lg-1) tiles it restricts into
  // items[(level * nranks + from) * nranks + to]: cells of `from`'s level tiles read by `to`
  std::vector<std::vector<HaloItem>> items;
  const std::vector<HaloItem>& list(int level, int from, int to) const {
    return items[((size_t)level * nranks + from) * nranks + to];
  }
};

// levels with fewer cells are replicated (gathered) rather than partitioned unless the
// caller sets octmg_mg_params.gather_below_cells (2^21 cells: one 128^3 level)
constexpr int64_t DEFAULT_GATHER_BELOW_CELLS = (int64_t)1 << 21;
int choose_partition_level(const PartInput& in, int nranks, int64_t gather_below_cells);
void build_partition(const PartInput& in, int nranks, int lg, PartPlan& P);

}  // namespace octmg
