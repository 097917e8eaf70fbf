// Row-per-thread tile stencils (sm_100a), shared by the RBGS colour pass (direct.cu), the
// residual-restriction (direct.cu) and the composite apply (kernels.cu).
//
// A thread owns one colour row of a tile: the four cells x = 2m + p (m = 0..3) of row (y, z)
// of colour c, p = (c + y + z) & 1, at the contiguous slots own = c*256 + 4*(y + 8z) + m of
// the colour-split order (octmg_internal.cuh).  The other colour's row at the same slots
// (oth = own ^ 256) holds every x-neighbour of the row but one (p = 0: element 3 of the x-
// tile's row; p = 1: element 0 of the x+ tile's row), its rows 4 / 32 slots away are the y /
// z neighbours (wrapped into the neighbour tile: +28 / -28, +224 / -224), so the 7-point
// stencil of the row is 11 float4 + 2 scalar loads (plus the row's own record).  Every load
// is issued unconditionally (walls read the tile itself and are zeroed), so all loads of a
// row are in flight at once.
//
// Irregular tiles (a T-junction face, or — in the composite leaf operator — a same-level
// inner neighbour) take the same row loads and then replace the values across those faces:
//   ghost face  (Eq. 12): g = u_i + (u_C - m_P)/2 from the coarse leaf cell C
//               (0 if C is inactive), the +face coupling from the tile's ghost coefficient
//               layer (reading 5), m_P the mean of the active cells of the cell's
//               2x2x2 parent block (reading 2), formed by warp shuffles;
//   inner face: the mean of the active children of the neighbour cell.
// Face order of every sum: x-, x+, y-, y+, z-, z+ (the oracle's).
#pragma once
#include "octmg_internal.cuh"

namespace octmg {
namespace rowk {

__device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ float e4(const float4& v, int m) {
  return m == 0 ? v.x : m == 1 ? v.y : m == 2 ? v.z : v.w;
}
__device__ __forceinline__ void s4(float4& v, int m, float x) {
  if (m == 0) v.x = x;
  else if (m == 1) v.y = x;
  else if (m == 2) v.z = x;
  else v.w = x;
}
__device__ __forceinline__ float4 msk4(const float4& v, const float4& c) {  // v where c != 0, else 0
  return make_float4(c.x != 0.0f ? v.x : 0.0f, c.y != 0.0f ? v.y : 0.0f, c.z != 0.0f ? v.z : 0.0f,
                     c.w != 0.0f ? v.w : 0.0f);
}

struct RowGeo {
  int y, z, p, own, oth;
  bool yl, yh, zl, zh;
};
__device__ __forceinline__ RowGeo row_geo(int colour, int row) {
  RowGeo g;
  g.y = row & 7;
  g.z = row >> 3;
  g.p = (colour + g.y + g.z) & 1;
  g.own = (colour << 8) + 4 * row;
  g.oth = g.own ^ 256;
  g.yl = g.y > 0; g.yh = g.y < 7; g.zl = g.z > 0; g.zh = g.z < 7;
  return g;
}

// the stencil neighbours of a row (values of one field, couplings of the +faces)
struct RowSt {
  float4 ox, ym, yp, zm, zp;  // other-colour rows: same / y- / y+ / z- / z+
  float xs;                   // the x-neighbour outside the row
  float4 cxo, cyp, czp;       // c_x- / c_y- / c_z- of the +x / +y / +z neighbours
  float xsc;                  // c_x- of the cell outside the row (the +x coupling when p = 1)
};

// TU(n): field pointer of tile n (n >= 0; called with the own tile index for n < 0).
// FLUX: the couplings across domain walls are zeroed too (the flux form multiplies them by
// a difference, not by the zero wall value)
template <class TU, bool FLUX = false>
__device__ __forceinline__ void row_load(RowSt& s, const TU& tu, const float* coef, int t, const int (&nb)[6],
                                         const RowGeo& g) {
  const float* ut = tu(t);
  const float* ct = coef + ((size_t)t << 11);
  auto tp = [&](int n) { return n >= 0 ? tu(n) : ut; };
  auto tc = [&](int n) { return n >= 0 ? coef + ((size_t)n << 11) : ct; };
  s.ox = ld4(ut + g.oth);
  s.cxo = ld4(ct + 512 + g.oth);
  const int nx = g.p ? nb[1] : nb[0];
  s.xs = __ldg(tp(nx) + g.oth + (g.p ? 0 : 3));
  s.xsc = __ldg(tc(nx) + 512 + g.oth);
  if (nx < 0) s.xs = 0.0f;
  s.ym = ld4((g.yl ? ut : tp(nb[2])) + g.oth + (g.yl ? -4 : 28));
  s.yp = ld4((g.yh ? ut : tp(nb[3])) + g.oth + (g.yh ? 4 : -28));
  s.zm = ld4((g.zl ? ut : tp(nb[4])) + g.oth + (g.zl ? -32 : 224));
  s.zp = ld4((g.zh ? ut : tp(nb[5])) + g.oth + (g.zh ? 32 : -224));
  s.cyp = ld4((g.yh ? ct : tc(nb[3])) + 1024 + g.oth + (g.yh ? 4 : -28));
  s.czp = ld4((g.zh ? ct : tc(nb[5])) + 1536 + g.oth + (g.zh ? 32 : -224));
  const float4 Z4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (!g.yl && nb[2] < 0) s.ym = Z4;
  if (!g.yh && nb[3] < 0) s.yp = Z4;
  if (!g.zl && nb[4] < 0) s.zm = Z4;
  if (!g.zh && nb[5] < 0) s.zp = Z4;
  if (FLUX) {
    if (nx < 0) s.xsc = 0.0f;
    if (!g.yh && nb[3] < 0) s.cyp = Z4;
    if (!g.zh && nb[5] < 0) s.czp = Z4;
  }
}

// Which stencil entries of the row hold a difference v_f - p_i instead of a value (flux form:
// the ghost and inner-neighbour faces, formed as differences to keep them exact)
struct RowRep {
  bool xs, ym, yp, zm, zp;
};

// Flux form of the leaf operator row: (A p)_i = d_i p_i + sum_f c_f (v_f - p_i), faces in the
// order x-, x+, y-, y+, z-, z+; d: the row sums (exact diagonal + couplings, setup.cu
// k_leaf_rowsum); pv: the cells' own values.  For a smooth p the differences are exact or
// nearly so, so the fp32 evaluation keeps the accuracy that c p + sum c_f v_f loses to
// cancellation (|A p| << |c||p| on the low modes the preconditioned CG leaves last).
__device__ __forceinline__ float4 row_sums_flux(const RowSt& s, const RowGeo& g, const RowRep& rp, const float4& qx,
                                                const float4& qy, const float4& qz, const float4& pv,
                                                const float4& d) {
  float r[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const float pi = e4(pv, m);
    const bool xm_out = !g.p && m == 0, xp_out = g.p && m == 3;  // entries outside the row (xs)
    const float vxm = g.p ? e4(s.ox, m) : (m == 0 ? s.xs : e4(s.ox, m - 1));
    const float vxp = g.p ? (m == 3 ? s.xs : e4(s.ox, m + 1)) : e4(s.ox, m);
    const float cxp = g.p ? (m == 3 ? s.xsc : e4(s.cxo, m + 1)) : e4(s.cxo, m);
    float sm = e4(d, m) * pi;
    sm = fmaf(e4(qx, m), (xm_out && rp.xs) ? vxm : vxm - pi, sm);
    sm = fmaf(cxp, (xp_out && rp.xs) ? vxp : vxp - pi, sm);
    sm = fmaf(e4(qy, m), rp.ym ? e4(s.ym, m) : e4(s.ym, m) - pi, sm);
    sm = fmaf(e4(s.cyp, m), rp.yp ? e4(s.yp, m) : e4(s.yp, m) - pi, sm);
    sm = fmaf(e4(qz, m), rp.zm ? e4(s.zm, m) : e4(s.zm, m) - pi, sm);
    sm = fmaf(e4(s.czp, m), rp.zp ? e4(s.zp, m) : e4(s.zp, m) - pi, sm);
    r[m] = sm;
  }
  return make_float4(r[0], r[1], r[2], r[3]);
}

// face sums of the row's 4 cells, starting from s0 (c*u, or 0), order x-, x+, y-, y+, z-, z+
__device__ __forceinline__ float4 row_sums(const RowSt& s, const RowGeo& g, const float4& qx, const float4& qy,
                                           const float4& qz, const float4& s0) {
  float r[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const float vxm = g.p ? e4(s.ox, m) : (m == 0 ? s.xs : e4(s.ox, m - 1));
    const float vxp = g.p ? (m == 3 ? s.xs : e4(s.ox, m + 1)) : e4(s.ox, m);
    const float cxp = g.p ? (m == 3 ? s.xsc : e4(s.cxo, m + 1)) : e4(s.cxo, m);
    float sm = e4(s0, m);
    sm = fmaf(e4(qx, m), vxm, sm);
    sm = fmaf(cxp, vxp, sm);
    sm = fmaf(e4(qy, m), e4(s.ym, m), sm);
    sm = fmaf(e4(s.cyp, m), e4(s.yp, m), sm);
    sm = fmaf(e4(qz, m), e4(s.zm, m), sm);
    sm = fmaf(e4(s.czp, m), e4(s.zp, m), sm);
    r[m] = sm;
  }
  return make_float4(r[0], r[1], r[2], r[3]);
}

// m_P of the four 2x2x2 blocks the row's cells lie in: per block, the x-pair sum of the
// row (own + other colour, both masked to the active cells) plus the rows y^1, z^1 by xor
// shuffles (lane distance LY / LZ) — the order of the pair-per-thread kernels (pair sum,
// then y, then z; each step commutative, so every lane of a block gets the same bits).
template <int LY, int LZ>
__device__ __forceinline__ float4 row_block_mean(const float4& own_m, const float4& own_c, const float4& oth_m,
                                                 const float4& oth_c) {
  const unsigned FULL = 0xffffffffu;
  float r[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    float su = e4(own_m, m) + e4(oth_m, m);
    int na = (e4(own_c, m) != 0.0f) + (e4(oth_c, m) != 0.0f);
    su += __shfl_xor_sync(FULL, su, LY);
    na += __shfl_xor_sync(FULL, na, LY);
    su += __shfl_xor_sync(FULL, su, LZ);
    na += __shfl_xor_sync(FULL, na, LZ);
    r[m] = na ? su / (float)na : 0.0f;
  }
  return make_float4(r[0], r[1], r[2], r[3]);
}

// Eq. 12 ghost values across the row's T-junction faces (and the ghost-layer couplings of
// the +faces).  ui: the cells' own values; mP: their block means; UC(C): the coarse-level
// field pointer of coarse leaf tile C; ZERO_UC: coarse values read as 0.
// FLUX: the entries become the differences g - u_i = (u_C - m_P)/2 (-u_i if C is inactive)
// and rp records them.
template <bool ZERO_UC, class UC, bool FLUX = false>
__device__ __forceinline__ void row_ghosts(RowSt& s, const RowGeo& g, int t, const int (&nb)[6], const int4& tv,
                                           const float* coef, const float* glayer_val, const int3& gl,
                                           const UC& uc_of, const float4& ui, const float4& mP,
                                           RowRep* rp = nullptr) {
  auto gval = [&](int m, int f) {
    const int ax = f >> 1, sg = (f & 1) ? 1 : -1;
    int c[3] = {tv.y * 8 + 2 * m + g.p, tv.z * 8 + g.y, tv.w * 8 + g.z};
    c[ax] += sg;
    const int C = -2 - nb[f];
    const int co = cslot((c[0] >> 1) & 7, (c[1] >> 1) & 7, (c[2] >> 1) & 7);
    const float cC = __ldg(coef + ((size_t)C << 11) + co);  // activity and value loaded together
    const float uc = ZERO_UC ? 0.0f : __ldg(uc_of(C) + co);
    if (FLUX) return cC != 0.0f ? 0.5f * (uc - e4(mP, m)) : -e4(ui, m);
    return cC != 0.0f ? e4(ui, m) + 0.5f * (uc - e4(mP, m)) : 0.0f;
  };
  auto glv = [&](int ax, int x) {  // gl: the tile's +x / +y / +z ghost-layer indices
    return __ldg(glayer_val + (size_t)(ax == 0 ? gl.x : (ax == 1 ? gl.y : gl.z)) * 64 +
                 (ax == 0 ? g.y + 8 * g.z : (ax == 1 ? x + 8 * g.z : x + 8 * g.y)));
  };
  const bool gx = (g.p == 0 && nb[0] <= -2) || (g.p == 1 && nb[1] <= -2);
  if (g.p == 0 && nb[0] <= -2) s.xs = gval(0, 0);
  if (g.p == 1 && nb[1] <= -2) { s.xs = gval(3, 1); s.xsc = glv(0, 7); }
  const bool gym = !g.yl && nb[2] <= -2, gyp = !g.yh && nb[3] <= -2;
  const bool gzm = !g.zl && nb[4] <= -2, gzp = !g.zh && nb[5] <= -2;
  if (gym) s.ym = make_float4(gval(0, 2), gval(1, 2), gval(2, 2), gval(3, 2));
  if (gyp) {
    s.yp = make_float4(gval(0, 3), gval(1, 3), gval(2, 3), gval(3, 3));
    s.cyp = make_float4(glv(1, g.p), glv(1, 2 + g.p), glv(1, 4 + g.p), glv(1, 6 + g.p));
  }
  if (gzm) s.zm = make_float4(gval(0, 4), gval(1, 4), gval(2, 4), gval(3, 4));
  if (gzp) {
    s.zp = make_float4(gval(0, 5), gval(1, 5), gval(2, 5), gval(3, 5));
    s.czp = make_float4(glv(2, g.p), glv(2, 2 + g.p), glv(2, 4 + g.p), glv(2, 6 + g.p));
  }
  if (FLUX) {
    rp->xs |= gx; rp->ym |= gym; rp->yp |= gyp; rp->zm |= gzm; rp->zp |= gzp;
  }
}

// Composite leaf operator: the value across a face toward a same-level inner tile is the
// mean of the active children of the neighbour cell, children in octant order
// dx + 2dy + 4dz, activity and value loaded together.  PV(tile, slot): the leaf value.
// FLUX: the entries become the mean of the differences v_child - p_i (-p_i without an
// active child) and rp records them; pi: the cells' own values.
template <class PV, bool FLUX = false>
__device__ __forceinline__ void row_inner(RowSt& s, const RowGeo& g, const int (&nb)[6], int NL, const int* child,
                                          const float* coef, const PV& pv, const float4& pi = float4{},
                                          RowRep* rp = nullptr) {
  auto ival = [&](int m, int f) {
    const int ax = f >> 1, sg = (f & 1) ? 1 : -1;
    int nc[3] = {2 * m + g.p, g.y, g.z};
    nc[ax] = (nc[ax] + sg) & 7;
    const int n = nb[f];
    const int ct = __ldg(child + 8 * (size_t)(n - NL) + (nc[0] >> 2) + 2 * (nc[1] >> 2) + 4 * (nc[2] >> 2));
    float sm = 0.0f;
    int k = 0;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      const int sl = cslot((2 * nc[0] + (d & 1)) & 7, (2 * nc[1] + ((d >> 1) & 1)) & 7, (2 * nc[2] + (d >> 2)) & 7);
      const float cc = __ldg(coef + ((size_t)ct << 11) + sl);
      float v = pv(ct, sl);
      if (FLUX) v -= e4(pi, m);
      if (cc != 0.0f) { sm += v; k++; }
    }
    if (FLUX) return k ? sm / (float)k : -e4(pi, m);
    return k ? sm / (float)k : 0.0f;
  };
  const bool ix = (g.p == 0 && nb[0] >= NL) || (g.p == 1 && nb[1] >= NL);
  const bool iym = !g.yl && nb[2] >= NL, iyp = !g.yh && nb[3] >= NL;
  const bool izm = !g.zl && nb[4] >= NL, izp = !g.zh && nb[5] >= NL;
  if (g.p == 0 && nb[0] >= NL) s.xs = ival(0, 0);
  if (g.p == 1 && nb[1] >= NL) s.xs = ival(3, 1);
  if (iym) s.ym = make_float4(ival(0, 2), ival(1, 2), ival(2, 2), ival(3, 2));
  if (iyp) s.yp = make_float4(ival(0, 3), ival(1, 3), ival(2, 3), ival(3, 3));
  if (izm) s.zm = make_float4(ival(0, 4), ival(1, 4), ival(2, 4), ival(3, 4));
  if (izp) s.zp = make_float4(ival(0, 5), ival(1, 5), ival(2, 5), ival(3, 5));
  if (FLUX) {
    rp->xs |= ix; rp->ym |= iym; rp->yp |= iyp; rp->zm |= izm; rp->zp |= izp;
  }
}

// the tile's +x / +y / +z ghost-layer indices (loaded early, with the tile origin, so the
// ghost couplings are one dependent load away instead of two)
__device__ __forceinline__ int3 load_gl(const int* glayer, int t) {
  return make_int3(__ldg(glayer + 3 * t), __ldg(glayer + 3 * t + 1), __ldg(glayer + 3 * t + 2));
}

__device__ __forceinline__ void load_nb(const int* nbr, int t, int (&nb)[6]) {
  const int2* np = reinterpret_cast<const int2*>(nbr + 6 * (size_t)t);
  const int2 n0 = __ldg(np), n1 = __ldg(np + 1), n2 = __ldg(np + 2);
  nb[0] = n0.x; nb[1] = n0.y; nb[2] = n1.x; nb[3] = n1.y; nb[4] = n2.x; nb[5] = n2.y;
}

}  // namespace rowk
}  // namespace octmg
