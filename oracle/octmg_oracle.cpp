// octmg oracle — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, double-precision CPU implementation of what arXiv 2604.18886
// ("Matrix-Free Multigrid with Algebraically Consistent Coarsening on Adaptive
// Octrees") defines: the graded tile octree (Sec. 3), the
// compact matrix-free Poisson coefficients (Eq. 3), the T-junction
// stencil (Eqs. 9-12), Galerkin coarsening (Alg. 3), RBGS
// (L407-409), the FAS-style mu-cycle (Alg. 4), the standard mu-cycle
// (Alg. 2, used only as an equivalence check on uniform trees), PCG
// (Alg. 1), multigrid as a standalone solver (L145, L411) and the cut-cell
// geometry of the tank scene (L1605-1616, L1924).  Readings of silent/ambiguous passages follow SURVEY.md
// 8(c) and are listed in DESIGN.md "Readings".
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load this library.  It shares no code, header, table or
// constant generator with the CUDA path (paper_2604_18886_b200/csrc).
//
// Style: cell-centric, global integer coordinates, hash-map tile lookup,
// everything computed in the order the paper states it.  Loops over cells are
// OpenMP-parallel only where each output cell is independent; every reduction is
// a serial sum in cell order, so results do not depend on the thread count.
//
// Parity status: every function below is pinned by tests/test_oracle_*.py
// (see DESIGN.md "Oracle pins"); none is "parity unpinned".
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

namespace {

enum Kind { K_FLUID = 0, K_DIRICHLET = 1, K_NEUMANN = 2 };
enum What { L_WALL = 0, L_CELL = 1, L_GHOST = 2, L_UNCOVERED = 3 };

// status codes (same numeric meaning as the ABI's, but defined independently here)
enum { S_OK = 0, S_INVALID = 1, S_OVERLAP = 2, S_GAP = 3, S_NOT_GRADED = 4, S_BREAKDOWN = 9, S_MAXITER = 10 };

thread_local std::string g_err;

struct Loc {
  int what;   // L_*
  int tile;   // CELL: level-l tile; GHOST: coarse leaf tile at l-1
  int off;    // cell offset within that tile
};

uint64_t pack3(int64_t i, int64_t j, int64_t k) {
  return (uint64_t)i | ((uint64_t)j << 21) | ((uint64_t)k << 42);
}

// Morton interleave, x in the lowest bit of each triple (canonical order, SURVEY c-1).
uint64_t morton(int64_t i, int64_t j, int64_t k) {
  uint64_t m = 0;
  for (int b = 0; b < 21; ++b) {
    m |= (uint64_t)((i >> b) & 1) << (3 * b);
    m |= (uint64_t)((j >> b) & 1) << (3 * b + 1);
    m |= (uint64_t)((k >> b) & 1) << (3 * b + 2);
  }
  return m;
}

struct MG {
  double alpha = 2.0, beta = 2.0;
  int mu = 1, nu_pre = 2, nu_post = 2, nu_coarsest = 10;
  int coarsest = 0;  // 0: nu_b RBGS iterations at level 0; 1: direct solve (Alg. 4 line 4)
};

struct Oracle {
  int B = 8, B3 = 512;
  int ext[3] = {1, 1, 1};
  int wall[6] = {1, 1, 1, 1, 1, 1};  // 1 = Dirichlet wall (p = 0), 0 = Neumann wall
  int L = 0;                         // finest leaf level
  int NL = 0, NI = 0, T = 0;
  std::vector<std::array<int, 4>> tile;  // canonical order: leaves then inners
  std::vector<std::unordered_map<uint64_t, int>> leafmap, innermap;
  std::vector<int> nbr, parent, child;
  std::vector<int> lb, lc, ib, ic;  // per-level leaf/inner segment begin & count

  // inputs and coefficients
  std::vector<uint8_t> kind;         // leaf cells
  std::vector<float> w[6];           // leaf cells (the fp32 inputs, read as exact doubles)
  std::vector<double> c, cm[3];      // all tiles' cells
  std::unordered_map<uint64_t, std::array<double, 3>> gcoef;  // ghost-cell -face coefficients
  double alpha = 2.0;
  bool setup = false;

  // multigrid work arrays (all tiles' cells)
  std::vector<double> u, b, ustar;
  // scratch (all tiles' cells): the pass-start snapshot of an RBGS pass (only the level's
  // cells and the coarse leaves its ghosts read are refreshed) and A^{l-1} u* of the FAS
  // restriction (only level l-1's cells are written and read)
  std::vector<double> snap, Au;
  // Eq. 14 check: after each prolongation, the largest |mean of the active
  // children - coarse value| and the largest |coarse value| seen (off unless enabled)
  bool check_eq14 = false;
  double eq14_dev = 0.0, eq14_scale = 0.0;
  // direct coarsest solve (built on first use after setup): the level-0 cells (all-tile
  // indices, leaf segment then inner segment) and the dense solution operator M0 (row-major)
  std::vector<size_t> c0_cells;
  std::vector<double> M0;
  // GMG comparison mode (setup_gmg): the cycle's records, = c / cm on the leaf cells and the
  // grid-assembled records on the inner cells; the preconditioner swaps them in for its cycle
  bool gmg = false;
  std::vector<double> gmg_c, gmg_cm[3];

  int levels() const { return L + 1; }
  int tlev(int t) const { return tile[t][0]; }
  int64_t dim(int l, int a) const { return (int64_t)ext[a] * B << l; }
  double hcell(int l) const { return std::ldexp(1.0, -l) / B; }

  int find_tile(int l, int64_t ti, int64_t tj, int64_t tk, bool* is_leaf) const {
    if (l < 0 || l > L) return -1;
    uint64_t k = pack3(ti, tj, tk);
    auto it = leafmap[l].find(k);
    if (it != leafmap[l].end()) { *is_leaf = true; return it->second; }
    auto jt = innermap[l].find(k);
    if (jt != innermap[l].end()) { *is_leaf = false; return jt->second; }
    return -1;
  }

  int offset(int64_t X, int64_t Y, int64_t Z) const {
    return (int)((X % B) + B * (Y % B) + B * B * (Z % B));
  }

  // What covers the level-l cell position (X,Y,Z): the domain wall, a cell of C_l,
  // or (ghost) the level-(l-1) leaf cell containing it.
  Loc locate(int l, int64_t X, int64_t Y, int64_t Z) const {
    if (X < 0 || Y < 0 || Z < 0 || X >= dim(l, 0) || Y >= dim(l, 1) || Z >= dim(l, 2))
      return {L_WALL, -1, -1};
    bool lf;
    int t = find_tile(l, X / B, Y / B, Z / B, &lf);
    if (t >= 0) return {L_CELL, t, offset(X, Y, Z)};
    if (l >= 1) {
      int64_t x = X >> 1, y = Y >> 1, z = Z >> 1;
      auto it = leafmap[l - 1].find(pack3(x / B, y / B, z / B));
      if (it != leafmap[l - 1].end()) return {L_GHOST, it->second, offset(x, y, z)};
    }
    return {L_UNCOVERED, -1, -1};
  }

  // locate() with a shortcut for positions inside tile t (same result, no hash lookup)
  Loc near(int l, int t, int64_t X, int64_t Y, int64_t Z) const {
    if (X >= 0 && Y >= 0 && Z >= 0 && X / B == tile[t][1] && Y / B == tile[t][2] && Z / B == tile[t][3])
      return {L_CELL, t, offset(X, Y, Z)};
    return locate(l, X, Y, Z);
  }

  void coords(int t, int off, int64_t* X, int64_t* Y, int64_t* Z) const {
    *X = (int64_t)tile[t][1] * B + off % B;
    *Y = (int64_t)tile[t][2] * B + (off / B) % B;
    *Z = (int64_t)tile[t][3] * B + off / (B * B);
  }

  size_t idx(int t, int off) const { return (size_t)t * B3 + off; }
  bool active(size_t i) const { return c[i] != 0.0; }
  bool loc_active(const Loc& n) const {
    if (n.what == L_CELL || n.what == L_GHOST) return c[idx(n.tile, n.off)] != 0.0;
    return false;
  }
  uint8_t leaf_kind(size_t i) const { return kind[i]; }
  double wf(int f, size_t i) const { return (double)w[f][i]; }
};

// -------------------------------------------------------------------------------------
// Tree
// -------------------------------------------------------------------------------------
int build(Oracle& o, const int32_t* tiles, int64_t n) {
  if (n <= 0) { g_err = "empty leaf list"; return S_INVALID; }
  int L = 0;
  for (int64_t t = 0; t < n; ++t) {
    int l = tiles[4 * t];
    if (l < 0 || l > 20) { g_err = "bad level"; return S_INVALID; }
    L = std::max(L, l);
    for (int a = 0; a < 3; ++a) {
      int64_t v = tiles[4 * t + 1 + a];
      if (v < 0 || v >= ((int64_t)o.ext[a] << l)) { g_err = "tile outside domain"; return S_INVALID; }
    }
  }
  o.L = L;
  for (int a = 0; a < 3; ++a)
    if (((int64_t)o.ext[a] * o.B << L) >= (1 << 20)) { g_err = "domain too fine for the oracle"; return S_INVALID; }
  o.leafmap.assign(L + 1, {});
  o.innermap.assign(L + 1, {});
  // leaves, duplicate check
  for (int64_t t = 0; t < n; ++t) {
    int l = tiles[4 * t];
    uint64_t k = pack3(tiles[4 * t + 1], tiles[4 * t + 2], tiles[4 * t + 3]);
    if (!o.leafmap[l].emplace(k, -1).second) { g_err = "duplicate leaf tile"; return S_OVERLAP; }
  }
  // inner tiles = all strict ancestors of leaves
  for (int64_t t = 0; t < n; ++t) {
    int l = tiles[4 * t];
    int64_t i = tiles[4 * t + 1], j = tiles[4 * t + 2], k = tiles[4 * t + 3];
    for (int m = l - 1; m >= 0; --m) {
      i >>= 1; j >>= 1; k >>= 1;
      o.innermap[m].emplace(pack3(i, j, k), -1);
    }
  }
  // overlap: a leaf that is also an ancestor of another leaf
  for (int l = 0; l <= L; ++l)
    for (auto& kv : o.leafmap[l])
      if (o.innermap[l].count(kv.first)) { g_err = "leaf tile overlaps a finer leaf"; return S_OVERLAP; }
  // gap: total leaf volume equals the domain (exact integer arithmetic)
  unsigned __int128 vol = 0, dom = (unsigned __int128)o.ext[0] * o.ext[1] * o.ext[2];
  for (int l = 0; l <= L; ++l) vol += (unsigned __int128)o.leafmap[l].size() << (3 * (L - l));
  dom <<= 3 * L;
  if (vol != dom) { g_err = "leaf tiles leave a gap"; return S_GAP; }

  // canonical order: leaves (level L..0, Morton ascending), then inners (same)
  struct E { int l; int64_t i, j, k; uint64_t m; };
  auto collect = [&](std::vector<std::unordered_map<uint64_t, int>>& maps) {
    std::vector<E> v;
    for (int l = L; l >= 0; --l) {
      std::vector<E> lv;
      for (auto& kv : maps[l]) {
        int64_t i = kv.first & 0x1FFFFF, j = (kv.first >> 21) & 0x1FFFFF, k = (kv.first >> 42) & 0x1FFFFF;
        lv.push_back({l, i, j, k, morton(i, j, k)});
      }
      std::sort(lv.begin(), lv.end(), [](const E& a, const E& b) { return a.m < b.m; });
      v.insert(v.end(), lv.begin(), lv.end());
    }
    return v;
  };
  std::vector<E> leaves = collect(o.leafmap), inners = collect(o.innermap);
  o.NL = (int)leaves.size();
  o.NI = (int)inners.size();
  o.T = o.NL + o.NI;
  o.tile.resize(o.T);
  o.lb.assign(L + 1, 0); o.lc.assign(L + 1, 0); o.ib.assign(L + 1, 0); o.ic.assign(L + 1, 0);
  for (int t = 0; t < o.T; ++t) {
    const E& e = t < o.NL ? leaves[t] : inners[t - o.NL];
    o.tile[t] = {e.l, (int)e.i, (int)e.j, (int)e.k};
    auto& mp = t < o.NL ? o.leafmap : o.innermap;
    mp[e.l][pack3(e.i, e.j, e.k)] = t;
  }
  for (int l = L; l >= 0; --l) {
    o.lb[l] = -1; o.ib[l] = -1;
  }
  for (int t = 0; t < o.T; ++t) {
    int l = o.tile[t][0];
    if (t < o.NL) { if (o.lb[l] < 0) o.lb[l] = t; o.lc[l]++; }
    else { if (o.ib[l] < 0) o.ib[l] = t; o.ic[l]++; }
  }
  for (int l = 0; l <= L; ++l) { if (o.lb[l] < 0) o.lb[l] = 0; if (o.ib[l] < 0) o.ib[l] = 0; }

  // grading across faces: every face-neighbour position of a leaf at level l
  // is in C_l or inside a leaf at level l-1.
  for (int t = 0; t < o.NL; ++t) {
    int l = o.tile[t][0];
    for (int f = 0; f < 6; ++f) {
      int a = f / 2, s = (f & 1) ? 1 : -1;
      int64_t q[3] = {o.tile[t][1], o.tile[t][2], o.tile[t][3]};
      q[a] += s;
      if (q[a] < 0 || q[a] >= ((int64_t)o.ext[a] << l)) continue;
      bool lf;
      if (o.find_tile(l, q[0], q[1], q[2], &lf) >= 0) continue;
      if (l >= 1 && o.leafmap[l - 1].count(pack3(q[0] >> 1, q[1] >> 1, q[2] >> 1))) continue;
      g_err = "leaf tiles are not 2:1 face graded";
      return S_NOT_GRADED;
    }
  }

  // tables: nbr (>=0 same-level tile, -1 wall, -2-idx ghost with coarse-leaf tile idx),
  // parent, child (octant dx + 2dy + 4dz)
  o.nbr.assign((size_t)o.T * 6, -1);
  o.parent.assign(o.T, -1);
  o.child.assign((size_t)o.NI * 8, -1);
  for (int t = 0; t < o.T; ++t) {
    int l = o.tile[t][0];
    for (int f = 0; f < 6; ++f) {
      int a = f / 2, s = (f & 1) ? 1 : -1;
      int64_t q[3] = {o.tile[t][1], o.tile[t][2], o.tile[t][3]};
      q[a] += s;
      if (q[a] < 0 || q[a] >= ((int64_t)o.ext[a] << l)) { o.nbr[6 * t + f] = -1; continue; }
      bool lf;
      int nt = o.find_tile(l, q[0], q[1], q[2], &lf);
      if (nt >= 0) { o.nbr[6 * t + f] = nt; continue; }
      auto it = l >= 1 ? o.leafmap[l - 1].find(pack3(q[0] >> 1, q[1] >> 1, q[2] >> 1)) : o.leafmap[0].end();
      if (t < o.NL && l >= 1 && it != o.leafmap[l - 1].end()) { o.nbr[6 * t + f] = -2 - it->second; continue; }
      g_err = "inner tile without same-level neighbour (not graded)";
      return S_NOT_GRADED;
    }
    if (l >= 1) {
      auto it = o.innermap[l - 1].find(pack3(o.tile[t][1] >> 1, o.tile[t][2] >> 1, o.tile[t][3] >> 1));
      o.parent[t] = it->second;
    }
    if (t >= o.NL) {
      for (int d = 0; d < 8; ++d) {
        bool lf;
        o.child[8 * (t - o.NL) + d] = o.find_tile(l + 1, 2 * (int64_t)o.tile[t][1] + (d & 1),
                                                  2 * (int64_t)o.tile[t][2] + ((d >> 1) & 1),
                                                  2 * (int64_t)o.tile[t][3] + (d >> 2), &lf);
      }
    }
  }
  return S_OK;
}

// ghost-cell key: level and 20-bit cell coordinates (build() checks the range)
uint64_t gkey(int l, int64_t X, int64_t Y, int64_t Z) {
  return ((uint64_t)l << 60) | ((uint64_t)X << 40) | ((uint64_t)Y << 20) | (uint64_t)Z;
}

// -------------------------------------------------------------------------------------
// Leaf coefficients: Eq. 3, cell kinds, T-junction faces
// (Eqs. 9-10).  kappa = w * h is the face conductance beta*S/h.
// -------------------------------------------------------------------------------------
// Fine sub-cells (level l+1) of the inner cell n (level l) that touch cell i across
// face f of i: the children of n on the side facing i.
void fine_subcells(const Oracle& o, int l, const Loc& n, int f, std::vector<size_t>& out) {
  out.clear();
  int64_t X, Y, Z;
  o.coords(n.tile, n.off, &X, &Y, &Z);
  int a = f / 2;
  int facing = (f & 1) ? 0 : 1;  // neighbour on i's + side -> its children with d_a = 0
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        int d[3] = {dx, dy, dz};
        if (d[a] != facing) continue;
        Loc s = o.locate(l + 1, 2 * X + dx, 2 * Y + dy, 2 * Z + dz);
        // grading guarantees these are leaf cells (inner tile next to a leaf has leaf
        // children on that face)
        if (s.what != L_CELL || s.tile >= o.NL) { out.push_back((size_t)-1); continue; }
        out.push_back(o.idx(s.tile, s.off));
      }
}

int assemble(Oracle& o) {
  const int B3 = o.B3;
  size_t NC = (size_t)o.T * B3;
  o.c.assign(NC, 0.0);
  for (int a = 0; a < 3; ++a) o.cm[a].assign(NC, 0.0);
  o.gcoef.clear();
  int err = S_OK;  // first error seen by any thread (each cell's outputs are independent)
  std::string err_msg;
  auto fail = [&](int st, const char* msg) {
#pragma omp critical(orc_assemble_err)
    if (err == S_OK) { err = st; err_msg = msg; }
  };
  // pass 1: diagonals of leaf cells from geometry
#pragma omp parallel for schedule(dynamic, 64)
  for (int t = 0; t < o.NL; ++t) {
    std::vector<size_t> subs;
    int l = o.tlev(t);
    double h = o.hcell(l);
    for (int off = 0; off < B3; ++off) {
      size_t i = o.idx(t, off);
      if (o.kind[i] != K_FLUID) { o.c[i] = 0.0; continue; }
      int64_t X, Y, Z;
      o.coords(t, off, &X, &Y, &Z);
      double s = 0.0;
      for (int f = 0; f < 6; ++f) {
        int a = f / 2, sg = (f & 1) ? 1 : -1;
        int64_t q[3] = {X, Y, Z};
        q[a] += sg;
        Loc n = o.locate(l, q[0], q[1], q[2]);
        if (n.what == L_WALL) {
          if (o.wall[f] == 1) s += o.wf(f, i) * h;
        } else if (n.what == L_CELL && n.tile < o.NL) {
          size_t j = o.idx(n.tile, n.off);
          if (o.kind[j] != K_NEUMANN) s += (sg < 0 ? o.wf(f, i) : o.wf(f ^ 1, j)) * h;
        } else if (n.what == L_CELL) {
          fine_subcells(o, l, n, f, subs);
          for (size_t sidx : subs) {
            if (sidx == (size_t)-1) { fail(S_NOT_GRADED, "fine sub-cell is not a leaf"); continue; }
            if (o.kind[sidx] != K_NEUMANN) s += 0.5 * o.wf(f ^ 1, sidx) * (0.5 * h);
          }
        } else if (n.what == L_GHOST) {
          if (o.kind[o.idx(n.tile, n.off)] != K_NEUMANN) s += o.wf(f, i) * h;
        } else {
          fail(S_NOT_GRADED, "uncovered neighbour");
        }
      }
      o.c[i] = s;  // a fluid cell with c == 0 is isolated and therefore inactive
    }
  }
  if (err) { g_err = err_msg; return err; }
  // pass 2: -face off-diagonals and ghost-cell coefficients of the + faces (the ghost
  // entries are collected per tile and inserted in tile order afterwards)
  struct GEntry { uint64_t key; int a; double v; };
  std::vector<std::vector<GEntry>> gent(o.NL);
#pragma omp parallel for schedule(dynamic, 64)
  for (int t = 0; t < o.NL; ++t) {
    std::vector<size_t> subs;
    int l = o.tlev(t);
    double h = o.hcell(l);
    for (int off = 0; off < B3; ++off) {
      size_t i = o.idx(t, off);
      if (o.kind[i] == K_NEUMANN) continue;  // all coefficients 0
      int64_t X, Y, Z;
      o.coords(t, off, &X, &Y, &Z);
      for (int a = 0; a < 3; ++a) {
        int64_t q[3] = {X, Y, Z};
        q[a] -= 1;
        int f = 2 * a;
        Loc n = o.locate(l, q[0], q[1], q[2]);
        double v = 0.0;
        if (n.what == L_CELL && n.tile < o.NL) {
          if (o.kind[o.idx(n.tile, n.off)] != K_NEUMANN) v = -o.wf(f, i) * h;
        } else if (n.what == L_CELL) {
          fine_subcells(o, l, n, f, subs);
          double acc = 0.0;
          for (size_t sidx : subs)
            if (o.c[sidx] != 0.0) acc += o.wf(f ^ 1, sidx) * (0.5 * h);
          v = -0.5 * acc;
        } else if (n.what == L_GHOST) {
          if (o.kind[o.idx(n.tile, n.off)] != K_NEUMANN) v = -o.wf(f, i) * h;
        }
        o.cm[a][i] = v;
        // + face toward a ghost: the ghost cell's -face coefficient (c_{6,x-})
        int64_t p[3] = {X, Y, Z};
        p[a] += 1;
        Loc g = o.locate(l, p[0], p[1], p[2]);
        if (g.what == L_GHOST) {
          double gv = o.kind[o.idx(g.tile, g.off)] != K_NEUMANN ? -o.wf(f + 1, i) * h : 0.0;
          gent[t].push_back({gkey(l, p[0], p[1], p[2]), a, gv});
        }
      }
    }
  }
  for (int t = 0; t < o.NL; ++t)
    for (const GEntry& e : gent[t]) o.gcoef[e.key][e.a] = e.v;
  return S_OK;
}

// Alg. 3 with the activity test on the off-diagonal branch (SURVEY c-3 / c-8
// #3): c^{l-1}_I from the 8 children i = 2I + d at level l.  literal = 1: Alg. 3 exactly as
// printed (the non-diagonal branch adds c^l_{i,e-}/alpha
// with no activity test).
void coarsen_level(Oracle& o, int l, bool literal) {
  const double al = o.alpha;
  int lc = l - 1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int t = o.ib[lc]; t < o.ib[lc] + o.ic[lc]; ++t) {
    for (int off = 0; off < o.B3; ++off) {
      int64_t IX, IY, IZ;
      o.coords(t, off, &IX, &IY, &IZ);
      double cI = 0.0, cIm[3] = {0.0, 0.0, 0.0};
      int active_cnt = 0;
      for (int dz = 0; dz < 2; ++dz)
        for (int dy = 0; dy < 2; ++dy)
          for (int dx = 0; dx < 2; ++dx) {
            int d[3] = {dx, dy, dz};
            int64_t ch[3] = {2 * IX + dx, 2 * IY + dy, 2 * IZ + dz};
            Loc ci = o.locate(l, ch[0], ch[1], ch[2]);
            size_t i = o.idx(ci.tile, ci.off);
            bool act = o.c[i] != 0.0;
            if (act) { active_cnt++; cI += o.c[i] / al; }  // diagonal
            for (int a = 0; a < 3; ++a) {
              int64_t q[3] = {ch[0], ch[1], ch[2]};
              q[a] -= 1;
              Loc nb = o.locate(l, q[0], q[1], q[2]);
              bool nact = o.loc_active(nb);
              if (d[a] == 1) {
                if (act && nact) cI += (2.0 / al) * o.cm[a][i];  // 2 cross terms in the diagonal
              } else {
                if (literal || (act && nact)) cIm[a] += o.cm[a][i] / al;  // non-diagonal
              }
            }
          }
      size_t I = o.idx(t, off);
      o.c[I] = active_cnt == 0 ? 0.0 : cI;
      for (int a = 0; a < 3; ++a) o.cm[a][I] = cIm[a];
    }
  }
}

int setup(Oracle& o, const uint8_t* kind, const float* w, double alpha, bool literal) {
  size_t N = (size_t)o.NL * o.B3;
  o.kind.assign(kind, kind + N);
  for (int f = 0; f < 6; ++f) {
    if (w) o.w[f].assign(w + (size_t)f * N, w + (size_t)(f + 1) * N);
    else o.w[f].assign(N, 1.0f);
  }
  for (size_t i = 0; i < N; ++i)
    if (o.kind[i] > 2) { g_err = "bad cell kind"; return S_INVALID; }
  o.alpha = alpha;
  int st = assemble(o);
  if (st) return st;
  for (int l = o.L; l >= 1; --l) coarsen_level(o, l, literal);
  o.setup = true;
  size_t NC = (size_t)o.T * o.B3;
  o.u.assign(NC, 0.0); o.b.assign(NC, 0.0); o.ustar.assign(NC, 0.0);
  o.snap.assign(NC, 0.0); o.Au.assign(NC, 0.0);
  o.M0.clear(); o.c0_cells.clear();
  return S_OK;
}

// -------------------------------------------------------------------------------------
// Operators (SURVEY c-4).  Face order x-, x+, y-, y+, z-, z+.
// -------------------------------------------------------------------------------------
double coef_plus(const Oracle& o, int l, int a, const Loc& n, int64_t X, int64_t Y, int64_t Z) {
  if (n.what == L_CELL) return o.cm[a][o.idx(n.tile, n.off)];
  if (n.what == L_GHOST) {
    auto it = o.gcoef.find(gkey(l, X, Y, Z));
    return it == o.gcoef.end() ? 0.0 : it->second[a];
  }
  return 0.0;
}

// mean over the active children of cell i's parent (the 2x2x2 block holding i), values v
double parent_mean(const Oracle& o, int l, int t, int64_t X, int64_t Y, int64_t Z, const double* v) {
  double s = 0.0;
  int n = 0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        Loc q = o.near(l, t, (X & ~1LL) + dx, (Y & ~1LL) + dy, (Z & ~1LL) + dz);
        size_t j = o.idx(q.tile, q.off);
        if (o.c[j] != 0.0) { s += v[j]; n++; }
      }
  return n ? s / n : 0.0;
}

// mean over the active children (level l+1) of the inner cell n (level l)
double child_mean(const Oracle& o, int l, const Loc& n, const double* v) {
  int64_t X, Y, Z;
  o.coords(n.tile, n.off, &X, &Y, &Z);
  double s = 0.0;
  int k = 0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        Loc q = o.locate(l + 1, 2 * X + dx, 2 * Y + dy, 2 * Z + dz);
        size_t j = o.idx(q.tile, q.off);
        if (o.c[j] != 0.0) { s += v[j]; k++; }
      }
  return k ? s / k : 0.0;
}

// Level operator row (A^l u)_i for a cell i of C_l.  Same-level neighbours use the level
// value; a ghost uses g = u_i + (u^{l-1}_C - m_P)/2 (Eq. 12), m_P from `snap`; inactive
// neighbours and walls contribute 0.  `uval` gives same-level/ghost-source values, `snap`
// the state the ghost reconstruction uses (equal to uval except inside an RBGS pass).
double level_row(const Oracle& o, int l, int t, int off, const double* uval, const double* snap,
                 bool skip_diag) {
  size_t i = o.idx(t, off);
  int64_t X, Y, Z;
  o.coords(t, off, &X, &Y, &Z);
  double s = skip_diag ? 0.0 : o.c[i] * uval[i];
  double mP = 0.0;
  bool have_mP = false;
  for (int f = 0; f < 6; ++f) {
    int a = f / 2, sg = (f & 1) ? 1 : -1;
    int64_t q[3] = {X, Y, Z};
    q[a] += sg;
    Loc n = o.near(l, t, q[0], q[1], q[2]);
    double coef = sg < 0 ? o.cm[a][i] : coef_plus(o, l, a, n, q[0], q[1], q[2]);
    double v = 0.0;
    if (n.what == L_CELL) {
      size_t j = o.idx(n.tile, n.off);
      v = o.c[j] != 0.0 ? uval[j] : 0.0;
    } else if (n.what == L_GHOST) {
      size_t C = o.idx(n.tile, n.off);
      if (o.c[C] != 0.0) {
        if (!have_mP) { mP = parent_mean(o, l, t, X, Y, Z, snap); have_mP = true; }
        v = snap[i] + 0.5 * (snap[C] - mP);
      }
    }
    s += coef * v;
  }
  return s;
}

// Composite operator row for a leaf cell (inner neighbour value = mean of its active
// children; ghost source = the coarse leaf's composite value).
double composite_row(const Oracle& o, int t, int off, const double* x) {
  int l = o.tlev(t);
  size_t i = o.idx(t, off);
  int64_t X, Y, Z;
  o.coords(t, off, &X, &Y, &Z);
  double s = o.c[i] * x[i];
  for (int f = 0; f < 6; ++f) {
    int a = f / 2, sg = (f & 1) ? 1 : -1;
    int64_t q[3] = {X, Y, Z};
    q[a] += sg;
    Loc n = o.near(l, t, q[0], q[1], q[2]);
    double coef = sg < 0 ? o.cm[a][i] : coef_plus(o, l, a, n, q[0], q[1], q[2]);
    double v = 0.0;
    if (n.what == L_CELL && n.tile < o.NL) {
      size_t j = o.idx(n.tile, n.off);
      v = o.c[j] != 0.0 ? x[j] : 0.0;
    } else if (n.what == L_CELL) {
      v = child_mean(o, l, n, x);
    } else if (n.what == L_GHOST) {
      size_t C = o.idx(n.tile, n.off);
      if (o.c[C] != 0.0) v = x[i] + 0.5 * (x[C] - parent_mean(o, l, t, X, Y, Z, x));
    }
    s += coef * v;
  }
  return s;
}

void apply_composite(const Oracle& o, const double* x, double* y) {
  // x, y are leaf vectors (NL*B3); leaf tiles come first in the canonical order, so a
  // leaf slot is also its all-tile index.
#pragma omp parallel for schedule(static) if (o.NL >= 256)
  for (int t = 0; t < o.NL; ++t)
    for (int off = 0; off < o.B3; ++off) {
      size_t i = o.idx(t, off);
      y[i] = o.c[i] != 0.0 ? composite_row(o, t, off, x) : 0.0;
    }
}

template <class F>
void for_level_tiles(const Oracle& o, int l, F fn) {
  std::vector<int> ts;
  for (int t = o.lb[l]; t < o.lb[l] + o.lc[l]; ++t) ts.push_back(t);
  for (int t = o.ib[l]; t < o.ib[l] + o.ic[l]; ++t) ts.push_back(t);
#pragma omp parallel for schedule(static) if (ts.size() >= 256)
  for (size_t k = 0; k < ts.size(); ++k) fn(ts[k]);
}

void apply_level(const Oracle& o, int l, const double* u, double* y) {
  for_level_tiles(o, l, [&](int t) {
    for (int off = 0; off < o.B3; ++off) {
      size_t i = o.idx(t, off);
      y[i] = o.c[i] != 0.0 ? level_row(o, l, t, off, u, u, false) : 0.0;
    }
  });
}

// One red-black Gauss-Seidel colour pass at level l.  Colour = parity of
// the global level-l cell coordinates (0 = red).  Ghost values and m_P come from the
// state at the start of the pass (SURVEY c-5 / c-8 #1).
void rbgs_pass(Oracle& o, int l, int colour, double* u, const double* b) {
  // pass-start snapshot of what the pass reads: level l's cells (leaf and inner segments)
  // and the level-(l-1) leaf cells behind its ghosts (not written by the pass)
  std::vector<double>& snap = o.snap;
  auto keep = [&](int first, int count) {
    std::copy(u + o.idx(first, 0), u + o.idx(first + count, 0), snap.begin() + o.idx(first, 0));
  };
  keep(o.lb[l], o.lc[l]);
  keep(o.ib[l], o.ic[l]);
  if (l >= 1) keep(o.lb[l - 1], o.lc[l - 1]);
  for_level_tiles(o, l, [&](int t) {
    for (int off = 0; off < o.B3; ++off) {
      int64_t X, Y, Z;
      o.coords(t, off, &X, &Y, &Z);
      if (((X + Y + Z) & 1) != colour) continue;
      size_t i = o.idx(t, off);
      if (o.c[i] == 0.0) continue;
      double offd = level_row(o, l, t, off, snap.data(), snap.data(), true);
      u[i] = (b[i] - offd) / o.c[i];
    }
  });
}

void smooth(Oracle& o, int l, int iters, bool red_first) {
  for (int k = 0; k < iters; ++k) {
    rbgs_pass(o, l, red_first ? 0 : 1, o.u.data(), o.b.data());
    rbgs_pass(o, l, red_first ? 1 : 0, o.u.data(), o.b.data());
  }
}

void smooth_coarsest(Oracle& o, const MG& p) {
  // nu_b split into two opposite-order halves
  smooth(o, 0, p.nu_coarsest / 2, true);
  smooth(o, 0, p.nu_coarsest - p.nu_coarsest / 2, false);
}

// Direct solve at the coarsest level (Alg. 4 line 4, "Or direct solve"; DESIGN
// reading 9b).  A0 = the level-0 operator over the cells of C_0, assembled column by column
// with apply_level (a symmetric matrix: level 0 has no ghosts, and a same-level coupling is
// the +side cell's -face entry in both rows).  Over the active cells:
//  * a connected component (coupling graph A0_ij != 0) is FLOATING when every row sum
//    |sum_j A0_ij| <= 1e-5 A0_ii (no Dirichlet coupling: A0 1_C = 0);
//  * M0 = R^{-1} P: R = A0 + sum_{floating C} (s_C / |C|) 1_C 1_C^T (s_C = mean diagonal of
//    C), P removes the mean of b over each floating component — so M0 b is the exact
//    solution on nonsingular components and the minimum-norm (pseudo-inverse) solution on
//    floating ones;
//  * R^{-1} by Gauss-Jordan elimination with partial pivoting (textbook), fp64.
// Inactive cells keep u = 0.
void build_direct_coarsest(Oracle& o) {
  std::vector<size_t>& cells = o.c0_cells;
  cells.clear();
  for (int t = o.lb[0]; t < o.lb[0] + o.lc[0]; ++t)
    for (int off = 0; off < o.B3; ++off) cells.push_back(o.idx(t, off));
  for (int t = o.ib[0]; t < o.ib[0] + o.ic[0]; ++t)
    for (int off = 0; off < o.B3; ++off) cells.push_back(o.idx(t, off));
  const size_t n = cells.size();
  // unit vectors and columns in the level-local scratch arrays (apply_level at level 0 reads
  // and writes only level-0 cells)
  std::vector<double>& e = o.snap;
  std::vector<double>& y = o.Au;
  std::vector<double> A(n * n, 0.0);
  for (size_t j = 0; j < n; ++j) e[cells[j]] = 0.0;
  for (size_t j = 0; j < n; ++j) {
    e[cells[j]] = 1.0;
    apply_level(o, 0, e.data(), y.data());
    for (size_t i = 0; i < n; ++i) A[i * n + j] = y[cells[i]];
    e[cells[j]] = 0.0;
  }
  std::vector<char> act(n);
  for (size_t i = 0; i < n; ++i) act[i] = o.c[cells[i]] != 0.0;
  // connected components of the active cells (breadth-first)
  std::vector<int> comp(n, -1);
  int ncomp = 0;
  for (size_t s0 = 0; s0 < n; ++s0) {
    if (!act[s0] || comp[s0] >= 0) continue;
    std::vector<size_t> q{s0};
    comp[s0] = ncomp;
    for (size_t k = 0; k < q.size(); ++k)
      for (size_t j = 0; j < n; ++j)
        if (act[j] && comp[j] < 0 && (A[q[k] * n + j] != 0.0 || A[j * n + q[k]] != 0.0)) {
          comp[j] = ncomp;
          q.push_back(j);
        }
    ncomp++;
  }
  std::vector<char> floating(ncomp, 1);
  std::vector<double> csum(ncomp, 0.0);
  std::vector<int> csize(ncomp, 0);
  for (size_t i = 0; i < n; ++i) {
    if (!act[i]) continue;
    double rs = 0.0;
    for (size_t j = 0; j < n; ++j) rs += A[i * n + j];
    if (std::fabs(rs) > 1e-5 * A[i * n + i]) floating[comp[i]] = 0;
    csum[comp[i]] += A[i * n + i];
    csize[comp[i]]++;
  }
  // R = A0 on the active block + the floating components' rank-one terms; identity rows
  // and columns for inactive cells
  std::vector<double> R(n * n, 0.0);
  for (size_t i = 0; i < n; ++i)
    for (size_t j = 0; j < n; ++j) {
      if (!act[i] || !act[j]) { R[i * n + j] = i == j ? 1.0 : 0.0; continue; }
      R[i * n + j] = A[i * n + j];
      if (comp[i] == comp[j] && floating[comp[i]]) R[i * n + j] += (csum[comp[i]] / csize[comp[i]]) / csize[comp[i]];
    }
  // Gauss-Jordan with partial pivoting: [R | I] -> [I | R^{-1}]
  std::vector<double> Ri(n * n, 0.0);
  for (size_t i = 0; i < n; ++i) Ri[i * n + i] = 1.0;
  for (size_t k = 0; k < n; ++k) {
    size_t piv = k;
    for (size_t i = k + 1; i < n; ++i)
      if (std::fabs(R[i * n + k]) > std::fabs(R[piv * n + k])) piv = i;
    if (piv != k)
      for (size_t j = 0; j < n; ++j) { std::swap(R[k * n + j], R[piv * n + j]); std::swap(Ri[k * n + j], Ri[piv * n + j]); }
    const double d = R[k * n + k];
    for (size_t j = 0; j < n; ++j) { R[k * n + j] /= d; Ri[k * n + j] /= d; }
    for (size_t i = 0; i < n; ++i) {
      if (i == k) continue;
      const double f = R[i * n + k];
      if (f == 0.0) continue;
      for (size_t j = 0; j < n; ++j) { R[i * n + j] -= f * R[k * n + j]; Ri[i * n + j] -= f * Ri[k * n + j]; }
    }
  }
  // M0 = R^{-1} P (P: mean removal over each floating component), zero for inactive cells
  o.M0.assign(n * n, 0.0);
  std::vector<double> rowmean(ncomp);
  for (size_t i = 0; i < n; ++i) {
    if (!act[i]) continue;
    std::fill(rowmean.begin(), rowmean.end(), 0.0);
    for (size_t j = 0; j < n; ++j)
      if (act[j] && floating[comp[j]]) rowmean[comp[j]] += Ri[i * n + j];
    for (size_t j = 0; j < n; ++j) {
      if (!act[j]) continue;
      double v = Ri[i * n + j];
      if (floating[comp[j]]) v -= rowmean[comp[j]] / csize[comp[j]];
      o.M0[i * n + j] = v;
    }
  }
}

void direct_coarsest(Oracle& o) {
  if (o.M0.empty()) build_direct_coarsest(o);
  const std::vector<size_t>& cells = o.c0_cells;
  const size_t n = cells.size();
  std::vector<double> bb(n), uu(n, 0.0);
  for (size_t j = 0; j < n; ++j) bb[j] = o.b[cells[j]];
  for (size_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (size_t j = 0; j < n; ++j) s += o.M0[i * n + j] * bb[j];
    uu[i] = s;
  }
  for (size_t i = 0; i < n; ++i)
    if (o.c[cells[i]] != 0.0) o.u[cells[i]] = uu[i];
}

void coarsest(Oracle& o, const MG& p) {
  if (p.coarsest == 1) direct_coarsest(o);
  else smooth_coarsest(o, p);
}

void residual(const Oracle& o, int l, std::vector<double>& r) {
  for_level_tiles(o, l, [&](int t) {
    for (int off = 0; off < o.B3; ++off) {
      size_t i = o.idx(t, off);
      r[i] = o.c[i] != 0.0 ? o.b[i] - level_row(o, l, t, off, o.u.data(), o.u.data(), false) : 0.0;
    }
  });
}

// children of inner cell (t, off) at level l-1, as all-tile indices (octant order)
void children_of(const Oracle& o, int lc, int t, int off, size_t out[8]) {
  int64_t X, Y, Z;
  o.coords(t, off, &X, &Y, &Z);
  for (int d = 0; d < 8; ++d) {
    Loc q = o.locate(lc + 1, 2 * X + (d & 1), 2 * Y + ((d >> 1) & 1), 2 * Z + (d >> 2));
    out[d] = o.idx(q.tile, q.off);
  }
}

// Eq. 14 as a check: after the prolongation of the inner cells of level lc,
// the mean of each inner cell's active children equals its coarse value u^{lc}_I.  Records
// the largest deviation and the largest |u^{lc}_I| (serial, inner-cell order).
void eq14_check(Oracle& o, int lc) {
  for (int t = o.ib[lc]; t < o.ib[lc] + o.ic[lc]; ++t)
    for (int off = 0; off < o.B3; ++off) {
      size_t ch[8];
      children_of(o, lc, t, off, ch);
      double s = 0.0;
      int n = 0;
      for (int d = 0; d < 8; ++d)
        if (o.c[ch[d]] != 0.0) { s += o.u[ch[d]]; n++; }
      if (!n) continue;
      size_t I = o.idx(t, off);
      o.eq14_dev = std::max(o.eq14_dev, std::fabs(s / n - o.u[I]));
      o.eq14_scale = std::max(o.eq14_scale, std::fabs(o.u[I]));
    }
}

// Alg. 4, FAS-style mu-cycle, readings SURVEY c-6.
void fas(Oracle& o, int l, const MG& p, std::vector<double>& r) {
  if (l == 0) { coarsest(o, p); return; }
  smooth(o, l, p.nu_pre, true);                  // pre-smoothing (R,B)
  residual(o, l, r);                             // r^l = b^l - A^l u^l
  int lc = l - 1;
  // u*_I = Avg(u^l) over active children; u^{l-1}_I := u*_I  (inner cells of level l-1)
#pragma omp parallel for schedule(dynamic, 16)
  for (int t = o.ib[lc]; t < o.ib[lc] + o.ic[lc]; ++t)
    for (int off = 0; off < o.B3; ++off) {
      size_t ch[8];
      children_of(o, lc, t, off, ch);
      double s = 0.0;
      int n = 0;
      for (int d = 0; d < 8; ++d)
        if (o.c[ch[d]] != 0.0) { s += o.u[ch[d]]; n++; }
      size_t I = o.idx(t, off);
      o.ustar[I] = n ? s / n : 0.0;
      o.u[I] = o.ustar[I];
    }
  // b^{l-1}_I = beta R r^l + (A^{l-1} u^{l-1})_I  on inner rows; leaf(l-1) rows keep b
  std::vector<double>& Au = o.Au;  // only level l-1's entries are written and read
  apply_level(o, lc, o.u.data(), Au.data());
#pragma omp parallel for schedule(dynamic, 16)
  for (int t = o.ib[lc]; t < o.ib[lc] + o.ic[lc]; ++t)
    for (int off = 0; off < o.B3; ++off) {
      size_t ch[8];
      children_of(o, lc, t, off, ch);
      double rs = 0.0;
      for (int d = 0; d < 8; ++d)
        if (o.c[ch[d]] != 0.0) rs += r[ch[d]];
      size_t I = o.idx(t, off);
      o.b[I] = p.beta * (rs / p.alpha) + Au[I];
    }
  for (int k = 0; k < p.mu; ++k) fas(o, lc, p, r);
  // prolongation of the update u^{l-1} - u* (no beta)
#pragma omp parallel for schedule(dynamic, 16)
  for (int t = o.ib[lc]; t < o.ib[lc] + o.ic[lc]; ++t)
    for (int off = 0; off < o.B3; ++off) {
      size_t ch[8];
      children_of(o, lc, t, off, ch);
      size_t I = o.idx(t, off);
      // an inactive coarse cell carries no correction (DESIGN reading 20: it is not a DOF; with
      // Alg. 3 it has no active child and u = u* = 0, in the GMG comparison mode a solid
      // coarse cell can have fluid children and a nonzero u*)
      if (o.c[I] == 0.0) continue;
      double corr = o.u[I] - o.ustar[I];
      for (int d = 0; d < 8; ++d)
        if (o.c[ch[d]] != 0.0) o.u[ch[d]] += corr;
    }
  if (o.check_eq14) eq14_check(o, lc);
  smooth(o, l, p.nu_post, false);                // post-smoothing (B,R)
}

// Alg. 2, standard mu-cycle with beta at prolongation.  Only meaningful on
// uniform trees (no leaves below the finest level); used as an equivalence check.
void mucycle_std(Oracle& o, int l, const MG& p, std::vector<double>& r) {
  if (l == 0) { coarsest(o, p); return; }
  smooth(o, l, p.nu_pre, true);
  residual(o, l, r);
  int lc = l - 1;
#pragma omp parallel for schedule(dynamic, 16)
  for (int t = o.ib[lc]; t < o.ib[lc] + o.ic[lc]; ++t)
    for (int off = 0; off < o.B3; ++off) {
      size_t ch[8];
      children_of(o, lc, t, off, ch);
      double rs = 0.0;
      for (int d = 0; d < 8; ++d)
        if (o.c[ch[d]] != 0.0) rs += r[ch[d]];
      size_t I = o.idx(t, off);
      o.b[I] = rs / p.alpha;  // R r
      o.u[I] = 0.0;
    }
  for (int k = 0; k < p.mu; ++k) mucycle_std(o, lc, p, r);
#pragma omp parallel for schedule(dynamic, 16)
  for (int t = o.ib[lc]; t < o.ib[lc] + o.ic[lc]; ++t)
    for (int off = 0; off < o.B3; ++off) {
      size_t ch[8];
      children_of(o, lc, t, off, ch);
      size_t I = o.idx(t, off);
      for (int d = 0; d < 8; ++d)
        if (o.c[ch[d]] != 0.0) o.u[ch[d]] += p.beta * o.u[I];
    }
  smooth(o, l, p.nu_post, false);
}

// GMG comparison mode: the coarse operators of the cycle "obtained directly
// from the grid, without explicit reference to the fine-level operator": every inner
// cell's record by Eq. 3 (kinds P:L318-335) at its own level, from its own kind
// and face weights and those of its same-level neighbours (an inner cell never borders a
// ghost, SURVEY c-1), instead of Alg. 3.  In fluid-only regions this equals the Galerkin
// record; next to solid cells it does not ("the terms related to i will
// vanish from A_II^{l-1}" under Galerkin, not here).  The leaf records — and so the composite
// operator the PCG solves — are unchanged; only the preconditioner's cycle uses these.
// kind_inner / w_inner: the inner cells' inputs (inner-tile order, natural cell order;
// w_inner [6][NI*B3] or NULL = 1).
int setup_gmg(Oracle& o, const uint8_t* kind_inner, const float* w_inner) {
  if (!o.setup) { g_err = "setup_gmg needs setup first"; return S_INVALID; }
  const size_t NL3 = (size_t)o.NL * o.B3, NI3 = (size_t)o.NI * o.B3;
  for (size_t i = 0; i < NI3; ++i)
    if (kind_inner[i] > 2) { g_err = "bad cell kind"; return S_INVALID; }
  o.gmg_c = o.c;
  for (int a = 0; a < 3; ++a) o.gmg_cm[a] = o.cm[a];
  auto kind_of = [&](size_t j) -> int { return j < NL3 ? o.kind[j] : kind_inner[j - NL3]; };
  auto w_of = [&](int f, size_t j) -> double {
    if (j < NL3) return o.wf(f, j);
    return w_inner ? (double)w_inner[(size_t)f * NI3 + (j - NL3)] : 1.0;
  };
  int err = S_OK;
#pragma omp parallel for schedule(dynamic, 16)
  for (int t = o.NL; t < o.T; ++t) {
    const int l = o.tlev(t);
    const double h = o.hcell(l);
    for (int off = 0; off < o.B3; ++off) {
      const size_t i = o.idx(t, off);
      const int k = kind_of(i);
      int64_t X, Y, Z;
      o.coords(t, off, &X, &Y, &Z);
      double c = 0.0, cm[3] = {0.0, 0.0, 0.0};
      if (k != K_NEUMANN) {
        for (int f = 0; f < 6; ++f) {
          const int a = f / 2, sg = (f & 1) ? 1 : -1;
          int64_t q[3] = {X, Y, Z};
          q[a] += sg;
          const Loc n = o.locate(l, q[0], q[1], q[2]);
          if (n.what == L_WALL) {
            if (k == K_FLUID && o.wall[f] == 1) c += w_of(f, i) * h;
          } else if (n.what == L_CELL) {
            const size_t j = o.idx(n.tile, n.off);
            if (kind_of(j) != K_NEUMANN) {
              if (k == K_FLUID) c += (sg < 0 ? w_of(f, i) : w_of(f ^ 1, j)) * h;
              if (sg < 0) cm[a] = -w_of(f, i) * h;
            }
          } else {
#pragma omp critical(orc_gmg_err)
            { err = S_NOT_GRADED; g_err = "inner cell next to a ghost or an uncovered position"; }
          }
        }
      }
      o.gmg_c[i] = c;  // a fluid cell with c == 0 is isolated and therefore inactive
      for (int a = 0; a < 3; ++a) o.gmg_cm[a][i] = cm[a];
    }
  }
  if (err) return err;
  o.gmg = true;
  o.M0.clear();
  o.c0_cells.clear();
  return S_OK;
}

// the cycle's coefficient set in place of c / cm for the duration of a preconditioner call
struct CycleCoefs {
  Oracle& o;
  explicit CycleCoefs(Oracle& oo) : o(oo) { swap(); }
  ~CycleCoefs() { swap(); }
  void swap() {
    if (!o.gmg) return;
    std::swap(o.c, o.gmg_c);
    for (int a = 0; a < 3; ++a) std::swap(o.cm[a], o.gmg_cm[a]);
  }
};

// M(r): u^l := 0 for all l; b^l[leaf(l)] := r; cycle from the finest level; z := u[leaves]
void precond(Oracle& o, const MG& p, const double* rin, double* z, bool fas_form) {
  CycleCoefs cyc(o);  // GMG mode: the grid-assembled coarse records (same leaf records)
  size_t NC = (size_t)o.T * o.B3, N = (size_t)o.NL * o.B3;
  std::fill(o.u.begin(), o.u.end(), 0.0);
  std::fill(o.b.begin(), o.b.end(), 0.0);
  std::fill(o.ustar.begin(), o.ustar.end(), 0.0);
  for (size_t i = 0; i < N; ++i) o.b[i] = o.c[i] != 0.0 ? rin[i] : 0.0;
  std::vector<double> r(NC, 0.0);
  if (fas_form) fas(o, o.L, p, r); else mucycle_std(o, o.L, p, r);
  for (size_t i = 0; i < N; ++i) z[i] = o.u[i];
}

double dot(const Oracle& o, const double* a, const double* b) {
  size_t N = (size_t)o.NL * o.B3;
  double s = 0.0;
  for (size_t i = 0; i < N; ++i)
    if (o.c[i] != 0.0) s += a[i] * b[i];
  return s;
}

void project_mean(const Oracle& o, double* r) {
  size_t N = (size_t)o.NL * o.B3;
  double s = 0.0;
  size_t n = 0;
  for (size_t i = 0; i < N; ++i)
    if (o.c[i] != 0.0) { s += r[i]; n++; }
  if (!n) return;
  double m = s / (double)n;
#pragma omp parallel for schedule(static)
  for (size_t i = 0; i < N; ++i)
    if (o.c[i] != 0.0) r[i] -= m;
}

bool pure_neumann(const Oracle& o) {
  for (int f = 0; f < 6; ++f) if (o.wall[f] == 1) return false;
  for (uint8_t k : o.kind) if (k == K_DIRICHLET) return false;
  return true;
}

// Alg. 1, readings SURVEY c-7 / c-8 #11-12.
int pcg(Oracle& o, const MG& p, int precond_kind, const double* bin, double* x, double rtol,
        int max_iters, int nullspace, int* iters_out, double* relres_out, double* bnorm_out,
        double* hist, int hcap) {
  size_t N = (size_t)o.NL * o.B3;
  bool ns = nullspace < 0 ? pure_neumann(o) : nullspace == 1;
  std::vector<double> r(N), z(N), pv(N), q(N);
  for (size_t i = 0; i < N; ++i) { x[i] = 0.0; r[i] = o.c[i] != 0.0 ? bin[i] : 0.0; }
  if (ns) project_mean(o, r.data());
  double bn = std::sqrt(dot(o, r.data(), r.data()));
  *bnorm_out = bn;
  *iters_out = 0;
  *relres_out = 0.0;
  if (bn == 0.0) return S_OK;
  auto M = [&](const double* rr, double* zz) {
    if (precond_kind == 0) { for (size_t i = 0; i < N; ++i) zz[i] = o.c[i] != 0.0 ? rr[i] : 0.0; }
    else precond(o, p, rr, zz, precond_kind == 1);
  };
  M(r.data(), z.data());
  pv = z;
  double rho = dot(o, r.data(), z.data());
  int k = 0;
  while (true) {
    apply_composite(o, pv.data(), q.data());
    double sigma = dot(o, pv.data(), q.data());
    if (!(sigma > 0.0)) { *iters_out = k; return S_BREAKDOWN; }
    double alpha = rho / sigma;
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < N; ++i) { x[i] += alpha * pv[i]; r[i] -= alpha * q[i]; }
    if (ns) project_mean(o, r.data());
    k++;
    double rn = std::sqrt(dot(o, r.data(), r.data()));
    if (k - 1 < hcap) hist[k - 1] = rn / bn;
    *iters_out = k;
    *relres_out = rn / bn;
    if (rn <= rtol * bn) return S_OK;
    if (k >= max_iters) return S_MAXITER;
    M(r.data(), z.data());
    double rho2 = dot(o, r.data(), z.data());
    double beta = rho2 / rho;
    rho = rho2;
#pragma omp parallel for schedule(static)
    for (size_t i = 0; i < N; ++i) pv[i] = z[i] + beta * pv[i];
  }
}

// -------------------------------------------------------------------------------------
// Projection operators on the composite octree ("apply the pressure gradient
// to project the velocity field and measure the divergence").  Face
// velocities u6[f][i]: the velocity component along +axis(f) on face f of leaf cell i
// (shared faces stored by both cells); fluid face area S = frac * h^2; the outward flux
// of face f is s_f u S with s_f = -1 on - faces, +1 on + faces.
// -------------------------------------------------------------------------------------
// Per-face decomposition of the composite operator's row i (Eq. 2 P:L295-297 per face,
// T-junction faces Eqs. 9-12): F_f = kd_f p_i + c_f v_f with kd_f the face's
// share of the geometric diagonal (the assembly's per-face term), c_f the face's coupling
// and v_f the composite neighbour value; sum_f F_f = (A p)_i.
void face_fluxes(const Oracle& o, int t, int off, const double* p, double F[6]) {
  const int l = o.tlev(t);
  const double h = o.hcell(l);
  const size_t i = o.idx(t, off);
  int64_t X, Y, Z;
  o.coords(t, off, &X, &Y, &Z);
  std::vector<size_t> subs;
  for (int f = 0; f < 6; ++f) {
    int a = f / 2, sg = (f & 1) ? 1 : -1;
    int64_t q[3] = {X, Y, Z};
    q[a] += sg;
    Loc n = o.locate(l, q[0], q[1], q[2]);
    double kd = 0.0, coef = sg < 0 ? o.cm[a][i] : coef_plus(o, l, a, n, q[0], q[1], q[2]), v = 0.0;
    if (n.what == L_WALL) {
      if (o.wall[f] == 1) kd = o.wf(f, i) * h;
    } else if (n.what == L_CELL && n.tile < o.NL) {
      size_t j = o.idx(n.tile, n.off);
      if (o.kind[j] != K_NEUMANN) kd = (sg < 0 ? o.wf(f, i) : o.wf(f ^ 1, j)) * h;
      v = o.c[j] != 0.0 ? p[j] : 0.0;
    } else if (n.what == L_CELL) {
      fine_subcells(o, l, n, f, subs);
      for (size_t sidx : subs)
        if (o.kind[sidx] != K_NEUMANN) kd += 0.5 * o.wf(f ^ 1, sidx) * (0.5 * h);
      v = child_mean(o, l, n, p);
    } else if (n.what == L_GHOST) {
      size_t C = o.idx(n.tile, n.off);
      if (o.kind[C] != K_NEUMANN) kd = o.wf(f, i) * h;
      if (o.c[C] != 0.0) v = p[i] + 0.5 * (p[C] - parent_mean(o, l, t, X, Y, Z, p));
    }
    F[f] = kd * p[i] + coef * v;
  }
}

// b_i = -(net outflow of u) over the faces of active leaf cell i; a coarse leaf's face
// toward finer cells takes the fine cells' entries (the finer side is authoritative).
void divergence(const Oracle& o, const float* frac, const double* u6, double* b) {
  const size_t N = (size_t)o.NL * o.B3;
  std::vector<size_t> subs;
  for (int t = 0; t < o.NL; ++t) {
    const int l = o.tlev(t);
    const double h = o.hcell(l);
    for (int off = 0; off < o.B3; ++off) {
      const size_t i = o.idx(t, off);
      b[i] = 0.0;
      if (o.c[i] == 0.0) continue;
      int64_t X, Y, Z;
      o.coords(t, off, &X, &Y, &Z);
      double out = 0.0;
      for (int f = 0; f < 6; ++f) {
        int a = f / 2, sg = (f & 1) ? 1 : -1;
        int64_t q[3] = {X, Y, Z};
        q[a] += sg;
        Loc n = o.locate(l, q[0], q[1], q[2]);
        if (n.what == L_CELL && n.tile >= o.NL) {
          fine_subcells(o, l, n, f, subs);
          const double hs = 0.5 * h;
          for (size_t sidx : subs)
            out += sg * u6[(size_t)(f ^ 1) * N + sidx] * (double)frac[(size_t)(f ^ 1) * N + sidx] * hs * hs;
        } else {
          out += sg * u6[(size_t)f * N + i] * (double)frac[(size_t)f * N + i] * h * h;
        }
      }
      b[i] = -out;
    }
  }
}

// u6 <- u6 - G p: on every face of an active leaf cell with fluid area S > 0, the normal
// velocity changes by F_f / S (outward), so that divergence(u - G p) = divergence(u) - A p.
void subtract_gradient(const Oracle& o, const float* frac, const double* p, double* u6) {
  const size_t N = (size_t)o.NL * o.B3;
  for (int t = 0; t < o.NL; ++t) {
    const double h = o.hcell(o.tlev(t));
    for (int off = 0; off < o.B3; ++off) {
      const size_t i = o.idx(t, off);
      if (o.c[i] == 0.0) continue;
      double F[6];
      face_fluxes(o, t, off, p, F);
      for (int f = 0; f < 6; ++f) {
        const double S = (double)frac[(size_t)f * N + i] * h * h;
        if (S > 0.0) u6[(size_t)f * N + i] += ((f & 1) ? 1.0 : -1.0) * F[f] / S;
      }
    }
  }
}

// Multigrid as a standalone solver ("can be used as standalone solvers"; P:L411
// "if multigrid is used as a standalone solver, beta should be set to 1"): the stationary
// iteration x_{k+1} = x_k + M(b - A x_k) from x_0 = 0, with the residual updated as
// r_{k+1} = r_k - A z_k and tested like Alg. 1 line 8 (||r_k|| <= rtol ||r_0||).
int mg_solve(Oracle& o, const MG& p, bool fas_form, const double* bin, double* x, double rtol, int max_iters,
             int nullspace, int* iters_out, double* relres_out, double* bnorm_out, double* hist, int hcap) {
  size_t N = (size_t)o.NL * o.B3;
  bool ns = nullspace < 0 ? pure_neumann(o) : nullspace == 1;
  std::vector<double> r(N), z(N), q(N);
  for (size_t i = 0; i < N; ++i) { x[i] = 0.0; r[i] = o.c[i] != 0.0 ? bin[i] : 0.0; }
  if (ns) project_mean(o, r.data());
  double bn = std::sqrt(dot(o, r.data(), r.data()));
  *bnorm_out = bn;
  *iters_out = 0;
  *relres_out = 0.0;
  if (bn == 0.0) return S_OK;
  int k = 0;
  while (true) {
    precond(o, p, r.data(), z.data(), fas_form);   // z = M(r)
    apply_composite(o, z.data(), q.data());        // q = A z
    for (size_t i = 0; i < N; ++i) {
      if (o.c[i] == 0.0) continue;
      x[i] += z[i];
      r[i] -= q[i];
    }
    if (ns) project_mean(o, r.data());
    k++;
    double rn = std::sqrt(dot(o, r.data(), r.data()));
    if (k - 1 < hcap) hist[k - 1] = rn / bn;
    *iters_out = k;
    *relres_out = rn / bn;
    if (rn <= rtol * bn) return S_OK;
    if (k >= max_iters) return S_MAXITER;
  }
}

// -------------------------------------------------------------------------------------
// Cut-cell geometry of the static tank scene ("signed distance
// values are evaluated at cell corners"; fluid face fractions by marching
// squares, ghost-fluid classification from the cell-centre SDF).  phi < 0 is solid.
// -------------------------------------------------------------------------------------
double sphere_phi(const double p[3], const double c[3], double r) {
  double dx = p[0] - c[0], dy = p[1] - c[1], dz = p[2] - c[2];
  return std::sqrt(dx * dx + dy * dy + dz * dz) - r;
}

// fluid (phi >= 0) area fraction of a unit square from its corner samples in cyclic order
// (0,0),(1,0),(1,1),(0,1): the polygon of fluid corners and linear edge crossings, area by
// the shoelace formula; the saddle (diagonal corners alike, neighbours opposite) with a
// solid face centre is two separate fluid corner triangles.
double face_fraction(const double phi[4], double phi_centre) {
  static const double P[4][2] = {{0, 0}, {1, 0}, {1, 1}, {0, 1}};
  bool fl[4];
  for (int k = 0; k < 4; ++k) fl[k] = phi[k] >= 0.0;
  const bool saddle = fl[0] == fl[2] && fl[1] == fl[3] && fl[0] != fl[1];
  if (saddle && phi_centre < 0.0) {
    double area = 0.0;
    for (int k = 0; k < 4; ++k) {
      if (!fl[k]) continue;
      int nx = (k + 1) % 4, pv = (k + 3) % 4;
      double a = phi[k] / (phi[k] - phi[nx]);
      double b = phi[k] / (phi[k] - phi[pv]);
      area += 0.5 * a * b;
    }
    return std::min(1.0, std::max(0.0, area));
  }
  double pts[8][2];
  int n = 0;
  for (int e = 0; e < 4; ++e) {
    int a = e, b = (e + 1) % 4;
    if (fl[a]) { pts[n][0] = P[a][0]; pts[n][1] = P[a][1]; ++n; }
    if (fl[a] != fl[b]) {
      double t = phi[a] / (phi[a] - phi[b]);
      pts[n][0] = P[a][0] + t * (P[b][0] - P[a][0]);
      pts[n][1] = P[a][1] + t * (P[b][1] - P[a][1]);
      ++n;
    }
  }
  double area = 0.0;
  for (int k = 0; k < n; ++k) {
    int k1 = (k + 1) % n;
    area += pts[k][0] * pts[k1][1] - pts[k1][0] * pts[k][1];
  }
  return std::min(1.0, std::max(0.0, 0.5 * std::fabs(area)));
}

// kind, face weights and right-hand side of every leaf cell of the tank scene: solid
// sphere obstacle (centre c, radius r; r <= 0: none) -> Neumann cells where phi(centre) <
// 0; face weight = fluid fraction of the face from its 4 corner samples; tank walls solid
// (w = 0) except the open top y = ext_y (w = 1); b = h^2 (w_y+ - w_y-) on fluid cells
// (unit downward velocity, volume-integrated divergence).  tiles: canonical leaf order.
void tank_fields(const int32_t* tiles, int64_t n, int B, const double* ext, const double* c, double r,
                 uint8_t* kind, float* w, float* bout) {
  const int64_t B3 = (int64_t)B * B * B, N = n * B3;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < n; ++t) {
    const int l = tiles[4 * t];
    const double h = std::ldexp(1.0, -l) / B;
    for (int64_t off = 0; off < B3; ++off) {
      const int64_t i = t * B3 + off;
      const int64_t X = (int64_t)tiles[4 * t + 1] * B + off % B;
      const int64_t Y = (int64_t)tiles[4 * t + 2] * B + (off / B) % B;
      const int64_t Z = (int64_t)tiles[4 * t + 3] * B + off / (B * B);
      const double cen[3] = {(X + 0.5) * h, (Y + 0.5) * h, (Z + 0.5) * h};
      const bool solid = r > 0.0 && sphere_phi(cen, c, r) < 0.0;
      kind[i] = solid ? K_NEUMANN : K_FLUID;
      double wf[6];
      for (int f = 0; f < 6; ++f) {
        const int a = f / 2, side = f % 2;
        const int o1 = a == 0 ? 1 : 0, o2 = a == 2 ? 1 : 2;
        double pc[3] = {cen[0], cen[1], cen[2]};
        pc[a] += (side - 0.5) * h;
        double frac = 1.0;
        if (r > 0.0) {
          static const int U[4] = {-1, 1, 1, -1}, V[4] = {-1, -1, 1, 1};
          double phi[4];
          for (int k = 0; k < 4; ++k) {
            double q[3] = {pc[0], pc[1], pc[2]};
            q[o1] += 0.5 * U[k] * h;
            q[o2] += 0.5 * V[k] * h;
            phi[k] = sphere_phi(q, c, r);
          }
          frac = face_fraction(phi, sphere_phi(pc, c, r));
        }
        const bool lo = pc[a] <= 0.0, hi = pc[a] >= ext[a];
        if (a == 1) {
          if (lo) frac = 0.0;
          if (hi) frac = 1.0;
        } else if (lo || hi) {
          frac = 0.0;
        }
        wf[f] = (double)(float)frac;
        w[(size_t)f * N + i] = (float)frac;
      }
      bout[i] = solid ? 0.0f : (float)(h * h * (wf[3] - wf[2]));
    }
  }
}

MG mg_from(const double* prm) {
  MG p;
  if (prm) {
    p.alpha = prm[0]; p.beta = prm[1]; p.mu = (int)prm[2]; p.nu_pre = (int)prm[3];
    p.nu_post = (int)prm[4]; p.nu_coarsest = (int)prm[5]; p.coarsest = (int)prm[6];
  }
  return p;
}

}  // namespace

// ======================================================================================
// C API (ctypes; see oracle/oracle.py)
// ======================================================================================
extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

void* orc_create(int B, const int32_t* ext, const int32_t* wall, const int32_t* tiles, int64_t n,
                 int32_t* status) {
  auto* o = new Oracle();
  if (B != 2 && B != 4 && B != 8) { g_err = "B must be 2, 4 or 8"; *status = S_INVALID; delete o; return nullptr; }
  o->B = B;
  o->B3 = B * B * B;
  for (int a = 0; a < 3; ++a) o->ext[a] = ext[a];
  for (int f = 0; f < 6; ++f) o->wall[f] = wall[f];
  int st = build(*o, tiles, n);
  *status = st;
  if (st) { delete o; return nullptr; }
  return o;
}

void orc_destroy(void* h) { delete (Oracle*)h; }

// out: [L, NL, NI, T, then for l = 0..L: leaf_begin, leaf_count, inner_begin, inner_count]
void orc_info(void* h, int64_t* out) {
  auto* o = (Oracle*)h;
  out[0] = o->L; out[1] = o->NL; out[2] = o->NI; out[3] = o->T;
  for (int l = 0; l <= o->L; ++l) {
    out[4 + 4 * l] = o->lb[l]; out[5 + 4 * l] = o->lc[l];
    out[6 + 4 * l] = o->ib[l]; out[7 + 4 * l] = o->ic[l];
  }
}

void orc_tables(void* h, int32_t* tiles, int32_t* nbr, int32_t* parent, int32_t* child) {
  auto* o = (Oracle*)h;
  for (int t = 0; t < o->T; ++t)
    for (int a = 0; a < 4; ++a) tiles[4 * t + a] = o->tile[t][a];
  std::memcpy(nbr, o->nbr.data(), sizeof(int32_t) * o->nbr.size());
  std::memcpy(parent, o->parent.data(), sizeof(int32_t) * o->parent.size());
  if (o->NI) std::memcpy(child, o->child.data(), sizeof(int32_t) * o->child.size());
}

int32_t orc_setup(void* h, const uint8_t* kind, const float* w, double alpha, int32_t literal) {
  return setup(*(Oracle*)h, kind, w, alpha, literal != 0);
}

// out: T*B3*4 doubles (c, cxm, cym, czm) per cell in all-tile order
void orc_coefs(void* h, double* out) {
  auto* o = (Oracle*)h;
  size_t NC = (size_t)o->T * o->B3;
  for (size_t i = 0; i < NC; ++i) {
    out[4 * i] = o->c[i];
    for (int a = 0; a < 3; ++a) out[4 * i + 1 + a] = o->cm[a][i];
  }
}

// GMG comparison mode: the inner cells' records assembled from their own kinds / weights
int32_t orc_setup_gmg(void* h, const uint8_t* kind_inner, const float* w_inner) {
  return setup_gmg(*(Oracle*)h, kind_inner, w_inner);
}

// the cycle's records (= orc_coefs unless GMG mode), same layout as orc_coefs
void orc_coefs_cycle(void* h, double* out) {
  auto* o = (Oracle*)h;
  CycleCoefs cyc(*o);
  size_t NC = (size_t)o->T * o->B3;
  for (size_t i = 0; i < NC; ++i) {
    out[4 * i] = o->c[i];
    for (int a = 0; a < 3; ++a) out[4 * i + 1 + a] = o->cm[a][i];
  }
}

// out: the diagonal c of the leaf cells (NL*B3 doubles; c == 0: inactive)
void orc_leaf_diag(void* h, double* out) {
  auto* o = (Oracle*)h;
  std::memcpy(out, o->c.data(), sizeof(double) * (size_t)o->NL * o->B3);
}

// ghost cell (level, X, Y, Z): its -face coefficients; returns 1 if such a ghost exists
int32_t orc_ghost_coef(void* h, int32_t l, int64_t X, int64_t Y, int64_t Z, double* out) {
  auto* o = (Oracle*)h;
  auto it = o->gcoef.find(gkey(l, X, Y, Z));
  if (it == o->gcoef.end()) return 0;
  for (int a = 0; a < 3; ++a) out[a] = it->second[a];
  return 1;
}

void orc_apply(void* h, const double* x, double* y) { apply_composite(*(Oracle*)h, x, y); }

// Eq. 14 check: enable / reset; read [max deviation, max |coarse value|]
void orc_set_check_eq14(void* h, int32_t on) {
  auto* o = (Oracle*)h;
  o->check_eq14 = on != 0;
  o->eq14_dev = 0.0;
  o->eq14_scale = 0.0;
}
void orc_eq14(void* h, double* out) {
  auto* o = (Oracle*)h;
  out[0] = o->eq14_dev;
  out[1] = o->eq14_scale;
}

void orc_apply_level(void* h, int32_t l, const double* u, double* y) {
  apply_level(*(Oracle*)h, l, u, y);
}

void orc_rbgs_pass(void* h, int32_t l, int32_t colour, double* u, const double* b) {
  rbgs_pass(*(Oracle*)h, l, colour, u, b);
}

// direct coarsest solve of level 0 alone (Alg. 4 line 4): u <- M0 b on the level-0 cells of
// the all-tile arrays (other entries untouched)
void orc_direct_coarsest(void* h, const double* b_all, double* u_all) {
  auto* o = (Oracle*)h;
  size_t NC = (size_t)o->T * o->B3;
  std::copy(b_all, b_all + NC, o->b.begin());
  std::copy(u_all, u_all + NC, o->u.begin());
  direct_coarsest(*o);
  std::copy(o->u.begin(), o->u.end(), u_all);
}

// prm: [alpha, beta, mu, nu_pre, nu_post, nu_coarsest, coarsest]; form: 1 = Alg. 4 (FAS), 0 = Alg. 2
void orc_vcycle(void* h, const double* prm, const double* r, double* z, int32_t form) {
  precond(*(Oracle*)h, mg_from(prm), r, z, form == 1);
}

// precond_kind: 0 identity, 1 FAS mu-cycle (Alg. 4), 2 standard mu-cycle (Alg. 2)
int32_t orc_pcg(void* h, const double* prm, int32_t precond_kind, const double* b, double* x,
                double rtol, int32_t max_iters, int32_t nullspace, int32_t* iters, double* relres,
                double* bnorm, double* hist, int32_t hcap) {
  int it = 0;
  int st = pcg(*(Oracle*)h, mg_from(prm), precond_kind, b, x, rtol, max_iters, nullspace, &it,
               relres, bnorm, hist, hcap);
  *iters = it;
  return st;
}

// form: 1 = Alg. 4 (FAS), 0 = Alg. 2
int32_t orc_mg_solve(void* h, const double* prm, int32_t form, const double* b, double* x, double rtol,
                     int32_t max_iters, int32_t nullspace, int32_t* iters, double* relres, double* bnorm,
                     double* hist, int32_t hcap) {
  int it = 0;
  int st = mg_solve(*(Oracle*)h, mg_from(prm), form == 1, b, x, rtol, max_iters, nullspace, &it, relres, bnorm,
                    hist, hcap);
  *iters = it;
  return st;
}

void orc_divergence(void* h, const float* frac, const double* u6, double* b) {
  divergence(*(Oracle*)h, frac, u6, b);
}

void orc_subtract_gradient(void* h, const float* frac, const double* p, double* u6) {
  subtract_gradient(*(Oracle*)h, frac, p, u6);
}

void orc_face_fluxes(void* h, int32_t t, int32_t off, const double* p, double* F) {
  face_fluxes(*(Oracle*)h, t, off, p, F);
}

double orc_face_fraction(const double* phi4, double phi_centre) { return face_fraction(phi4, phi_centre); }

void orc_tank_fields(const int32_t* tiles, int64_t n, int32_t B, const double* ext, const double* centre,
                     double radius, uint8_t* kind, float* w, float* b) {
  tank_fields(tiles, n, B, ext, centre, radius, kind, w, b);
}

}  // extern "C"
