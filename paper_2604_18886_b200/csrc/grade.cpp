// 2:1 face-grading repair of a leaf-tile list (host, "refine
// the coarser side to fixpoint"; grading P:L548-550).  A leaf tile T at level l requires
// every in-domain face-neighbour position Q at level l to be covered by a leaf at level
// l-1 or l, or by finer leaves; a covering leaf at level <= l-2 is replaced by its 8
// children.  Sweeps mark against the current set and refine all marked leaves, until no
// leaf is marked: the least graded refinement, independent of the order of the input.
#include <array>
#include <cstdint>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/octmg.h"

namespace octmg {

void set_error(const std::string& msg);

namespace {

// 19 bits per axis (the tree's own limit, tree.cu: ext << level <= 2^19) and the level
inline uint64_t key(int l, int64_t i, int64_t j, int64_t k) {
  return ((uint64_t)l << 57) | ((uint64_t)i << 38) | ((uint64_t)j << 19) | (uint64_t)k;
}
constexpr int64_t KEY_AXIS = int64_t(1) << 19;
inline bool key_fits(const int32_t* ext, int level) {
  for (int a = 0; a < 3; ++a)
    if (ext[a] < 1 || ((int64_t)ext[a] << level) > KEY_AXIS) return false;
  return true;
}

}  // namespace

octmg_status grade_repair(const octmg_tile* in, int64_t n, const int32_t* ext, std::vector<octmg_tile>& out) {
  std::unordered_set<uint64_t> set;
  std::vector<octmg_tile> cur(in, in + n);
  for (const octmg_tile& t : cur) {
    if (t.level < 0 || t.level >= OCTMG_MAX_LEVELS || t.i < 0 || t.j < 0 || t.k < 0 ||
        ((int64_t)t.i >> t.level) >= ext[0] || ((int64_t)t.j >> t.level) >= ext[1] ||
        ((int64_t)t.k >> t.level) >= ext[2]) {
      set_error("leaf tile out of range");
      return OCTMG_E_INVALID;
    }
    if (!key_fits(ext, t.level)) {
      set_error("domain too fine: ext << level exceeds 2^19 tiles per axis");
      return OCTMG_E_INVALID;
    }
    set.insert(key(t.level, t.i, t.j, t.k));
  }
  while (true) {
    std::unordered_set<uint64_t> marked;
    std::vector<octmg_tile> refine;
    for (const octmg_tile& t : cur) {
      for (int f = 0; f < 6; ++f) {
        int64_t q[3] = {t.i, t.j, t.k};
        q[f >> 1] += (f & 1) ? 1 : -1;
        if (q[f >> 1] < 0 || q[f >> 1] >= ((int64_t)ext[f >> 1] << t.level)) continue;
        // the covering leaf: the first level m <= l holding (q >> (l - m))
        for (int m = t.level; m >= 0; --m) {
          const int sh = t.level - m;
          const uint64_t kq = key(m, q[0] >> sh, q[1] >> sh, q[2] >> sh);
          if (set.count(kq)) {
            if (m <= t.level - 2 && marked.insert(kq).second)
              refine.push_back(octmg_tile{m, (int32_t)(q[0] >> sh), (int32_t)(q[1] >> sh), (int32_t)(q[2] >> sh)});
            break;
          }
        }
      }
    }
    if (refine.empty()) break;
    std::vector<octmg_tile> next;
    next.reserve(cur.size() + 7 * refine.size());
    for (const octmg_tile& t : cur)
      if (!marked.count(key(t.level, t.i, t.j, t.k))) next.push_back(t);
    for (const octmg_tile& t : refine) {
      set.erase(key(t.level, t.i, t.j, t.k));
      if (t.level + 1 >= OCTMG_MAX_LEVELS || !key_fits(ext, t.level + 1)) {
        set_error("grading repair exceeds the maximum level");
        return OCTMG_E_INVALID;
      }
      for (int d = 0; d < 8; ++d) {
        octmg_tile c{t.level + 1, 2 * t.i + (d & 1), 2 * t.j + ((d >> 1) & 1), 2 * t.k + (d >> 2)};
        next.push_back(c);
        set.insert(key(c.level, c.i, c.j, c.k));
      }
    }
    cur.swap(next);
  }
  out.swap(cur);
  return OCTMG_OK;
}

}  // namespace octmg

extern "C" octmg_status octmg_grade_repair_host(const octmg_tile* tiles, int64_t n, const int32_t* ext3,
                                                 octmg_tile* out, int64_t cap, int64_t* n_out) {
  if (!tiles || !ext3 || !n_out || n < 0) {
    octmg::set_error("null argument");
    return OCTMG_E_INVALID;
  }
  std::vector<octmg_tile> res;
  octmg_status st = octmg::grade_repair(tiles, n, ext3, res);
  if (st != OCTMG_OK) return st;
  *n_out = (int64_t)res.size();
  if (!out || cap < (int64_t)res.size()) {
    octmg::set_error("output capacity too small (n_out holds the required count)");
    return OCTMG_E_INVALID;
  }
  for (size_t k = 0; k < res.size(); ++k) out[k] = res[k];
  return OCTMG_OK;
}
