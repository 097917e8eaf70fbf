// Morton-range partition of the octree and halo plans (host code).
//
// Ownership: the level-lg tiles (lg <= the coarsest leaf level, so every leaf is owned)
// in Morton order are cut into nranks contiguous ranges balanced by the number of
// descendant cells (boundaries aligned to whole level-(lg-1) parents, so a restriction into
// the replicated level lg-1 writes whole parent tiles of one rank).  A tile at level >= lg
// is owned by the owner of its level-lg ancestor; tiles at levels < lg are replicated and
// computed redundantly by every rank.
//
// Halo plan: the cells of rank r's level-l tiles that rank s's kernels read:
//   (a) face layers of same-level face neighbours of s's tiles (stencils),
//   (b) whole coarse-leaf tiles of ghost faces of s's level-(l+1) tiles (Eq. 12 sources),
//   (c) whole child tiles of r's inner tiles that are same-level neighbours of s's leaves
//       (the composite operator's inner-neighbour means).
// Items are listed in a canonical order (tile index, then face), so the receiver unpacks
// with the sender's list; every rank computes every list from the replicated tables.
#include <algorithm>
#include <cstdint>
#include <map>
#include <set>
#include <vector>

#include "partition.h"

namespace octmg {

static int tile_level(const std::vector<int>& tiles4, int t) { return tiles4[4 * (size_t)t]; }

int choose_partition_level(const PartInput& in, int nranks, int64_t gather_below_cells) {
  // coarsest leaf level (every leaf must be owned, so lg <= lmin)
  int lmin = in.L;
  for (int l = 0; l <= in.L; ++l)
    if (in.lc[l] > 0) { lmin = l; break; }
  // the coarsest level <= lmin with at least 8 tiles per rank and at least
  // gather_below_cells cells: the levels below it are small enough that a rank solves them
  // faster redundantly (after gathering the restricted parents) than partitioned with a
  // halo exchange per pass (BASELINE north_star: "coarse levels below a size threshold are
  // gathered")
  const int64_t thr = gather_below_cells > 0 ? gather_below_cells : DEFAULT_GATHER_BELOW_CELLS;
  for (int l = 0; l <= lmin; ++l) {
    const int64_t tiles = (int64_t)in.lc[l] + in.ic[l];
    if (tiles >= 8 * (int64_t)nranks && tiles * 512 >= thr) return l;
  }
  return lmin;
}

void build_partition(const PartInput& in, int nranks, int lg, PartPlan& P) {
  const int T = in.NL + in.NI;
  P.nranks = nranks;
  P.lg = lg;
  P.owner.assign(T, -1);
  // level-lg tiles in Morton order = canonical order within the level: leaves then inners
  // each Morton-sorted; merge them by Morton key
  std::vector<int> lvl;
  for (int t = in.lb[lg]; t < in.lb[lg] + in.lc[lg]; ++t) lvl.push_back(t);
  for (int t = in.ib[lg]; t < in.ib[lg] + in.ic[lg]; ++t) lvl.push_back(t);
  std::sort(lvl.begin(), lvl.end(), [&](int a, int b) { return in.morton[a] < in.morton[b]; });
  // weight of each level-lg tile = descendant tile count (cells / 512)
  std::vector<double> wsub(T, 0.0);
  for (int l = in.L; l >= lg; --l) {
    auto acc = [&](int t) {
      double w = 1.0;
      if (t >= in.NL)
        for (int d = 0; d < 8; ++d) {
          int c = in.child[8 * (size_t)(t - in.NL) + d];
          if (c >= 0) w += wsub[c];
        }
      wsub[t] = w;
    };
    for (int t = in.lb[l]; t < in.lb[l] + in.lc[l]; ++t) acc(t);
    for (int t = in.ib[l]; t < in.ib[l] + in.ic[l]; ++t) acc(t);
  }
  double total = 0.0;
  for (int t : lvl) total += wsub[t];
  // contiguous ranges, cut only between different level-(lg-1) parents
  std::vector<int> cut(nranks + 1, (int)lvl.size());
  cut[0] = 0;
  double acc = 0.0;
  int r = 1;
  for (size_t k = 0; k < lvl.size() && r < nranks; ++k) {
    acc += wsub[lvl[k]];
    bool boundary = k + 1 < lvl.size() && (lg == 0 || in.parent[lvl[k]] != in.parent[lvl[k + 1]]);
    if (boundary && acc >= total * r / nranks) cut[r++] = (int)k + 1;
  }
  for (; r < nranks; ++r) cut[r] = (int)lvl.size();
  P.lg_tiles.assign(nranks, {});
  for (int q = 0; q < nranks; ++q)
    for (int k = cut[q]; k < cut[q + 1]; ++k) {
      P.owner[lvl[k]] = q;
      P.lg_tiles[q].push_back(lvl[k]);
    }
  // descendants inherit the owner
  for (int l = lg; l < in.L; ++l) {
    auto push = [&](int t) {
      if (t < in.NL) return;
      for (int d = 0; d < 8; ++d) {
        int c = in.child[8 * (size_t)(t - in.NL) + d];
        if (c >= 0) P.owner[c] = P.owner[t];
      }
    };
    for (int t = in.ib[l]; t < in.ib[l] + in.ic[l]; ++t) push(t);
  }
  // parents at lg-1 written by each rank (whole tiles by construction)
  P.parent_tiles.assign(nranks, {});
  if (lg >= 1)
    for (int q = 0; q < nranks; ++q) {
      std::set<int> ps;
      for (int t : P.lg_tiles[q]) ps.insert(in.parent[t]);
      P.parent_tiles[q].assign(ps.begin(), ps.end());
    }
  // halo items per (level, sender, receiver): key -> kind (0..5 face, 6 whole)
  P.items.assign((size_t)(in.L + 1) * nranks * nranks, {});
  std::vector<std::map<int, int>> sets((size_t)(in.L + 1) * nranks * nranks);
  auto add = [&](int l, int from, int to, int tile, int kind) {
    if (from == to || from < 0 || to < 0) return;
    auto& m = sets[((size_t)l * nranks + from) * nranks + to];
    auto it = m.find(tile);
    if (it == m.end()) m[tile] = 1 << kind;
    else it->second |= 1 << kind;
  };
  for (int t = 0; t < T; ++t) {
    const int l = tile_level(in.tiles4, t);
    if (l < lg) continue;
    const int s = P.owner[t];
    for (int f = 0; f < 6; ++f) {
      int n = in.nbr[6 * (size_t)t + f];
      if (n >= 0) {
        // (a) t (owned by s) reads the face layer of n facing it: n's face f^1
        add(l, P.owner[n], s, n, f ^ 1);
        // (c) s-owned leaf t next to an inner tile n owned elsewhere: the children of n
        //     on the face toward t
        if (t < in.NL && n >= in.NL) {
          for (int d = 0; d < 8; ++d) {
            int dd[3] = {d & 1, (d >> 1) & 1, d >> 2};
            const int a = f >> 1;
            const int facing = (f & 1) ? 0 : 1;  // n on t's + side -> children with d_a = 0
            if (dd[a] != facing) continue;
            int c = in.child[8 * (size_t)(n - in.NL) + d];
            if (c >= 0) add(l + 1, P.owner[c], s, c, 6);
          }
        }
      } else if (n <= -2) {
        // (b) the coarse leaf of a ghost face: whole tile (level l-1 >= lg only)
        int C = -2 - n;
        if (l - 1 >= lg) add(l - 1, P.owner[C], s, C, 6);
      }
    }
  }
  for (size_t k = 0; k < sets.size(); ++k)
    for (auto& kv : sets[k]) {
      if (kv.second & (1 << 6)) P.items[k].push_back({kv.first, 6});
      else
        for (int f = 0; f < 6; ++f)
          if (kv.second & (1 << f)) P.items[k].push_back({kv.first, f});
    }
}

}  // namespace octmg
