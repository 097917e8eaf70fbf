// Per-cell stencil helpers shared by the tile kernels (direct.cu) and the on-chip coarse
// sub-cycle (subcycle.cu).  Cell (x,y,z) of tile t at the tile's level; coefficient record
// float4 (c, c_x-, c_y-, c_z-); face order x-, x+, y-, y+, z-, z+ (the oracle's).
// NC: load path of the values (see ldv): 1 in the tile kernels (nothing they read is written
// before it is read), 0 / 2 inside the coarse-cycle kernels, which read what they wrote in
// earlier phases (0: one CTA, 2: several CTAs across grid barriers).
#pragma once
#include "octmg_internal.cuh"

namespace octmg {

enum { SM_PLAIN = 0, SM_ZERO1 = 1, SM_ZERO2 = 2, SM_PRO1 = 3, SM_PRO2 = 4, SM_RESTRICT = 5, SM_PLAIN_RZ = 6 };

// the i-th tile of a level launch: from the order array, or computed (no dependent load
// before the tile's own loads can issue)
__device__ __forceinline__ int level_tile(const SmoothArgs& a, int i) {
  if (a.order) return __ldg(a.order + i);
  return i < a.ord_nleaf ? a.ord_leaf0 + i : a.ord_inner0 + (i - a.ord_nleaf);
}

// NC: 1 = read-only path (__ldg), 2 = L2 only (__ldcg; data written by other CTAs earlier
// in the same launch, across a grid barrier), 0 = plain load (same-CTA data)
template <int NC>
__device__ __forceinline__ float ldv(const float* p) {
  if (NC == 1) return __ldg(p);
  if (NC == 2) return __ldcg(p);
  return *p;
}

__device__ __forceinline__ int loff(int x, int y, int z) { return cslot(x, y, z); }  // slot order
__device__ __forceinline__ float comp(const float4& v, int a) { return a == 0 ? v.y : (a == 1 ? v.z : v.w); }
__device__ __forceinline__ int pcell_of(int4 tv, int x, int y, int z) {
  return loff(((tv.y & 1) << 2) + (x >> 1), ((tv.z & 1) << 2) + (y >> 1), ((tv.w & 1) << 2) + (z >> 1));
}

// face term sum (x-, x+, y-, y+, z-, z+ order, the oracle's) for cell (x,y,z) of tile t at
// its level, values from u; ghosts use ui (the cell's snapshot value) and mP (mean of the
// active cells of its parent block) — only evaluated if the tile has a ghost face.
// ZERO_OWN: cells of `colour` read as 0 (first black pass of a cycle).
template <bool ZERO_OWN, int NC = 1>
__device__ __forceinline__ float face_sum(const SmoothArgs& a, int t, int x, int y, int z, const float4& q,
                                          float ui, float mP, int colour, float s0, const float* su = nullptr,
                                          const float (*scm)[TB3] = nullptr, const int* nbp = nullptr,
                                          const int4* tvp = nullptr) {
  const size_t base = (size_t)t * TB3;
  const float* ut = tptr(a.u, t, a.NL);
  const int c[3] = {x, y, z};
  // every face neighbour is in the other colour half at a fixed slot offset (in the tile or
  // wrapped into the neighbour tile), see face_sum_regular in direct.cu
  const int nbase = loff(x, y, z) ^ 256;
  const int nown = ((x + y + z) & 1) ^ 1;  // colour of every face neighbour
  const int p = x & 1;
  float s = s0;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1, sg = (f & 1) ? 1 : -1;
    const bool inside = c[ax] + sg >= 0 && c[ax] + sg < 8;
    const int dlt = f == 0 ? (inside ? p - 1 : 3) : f == 1 ? (inside ? p : -3) : f == 2 ? (inside ? -4 : 28)
                  : f == 3 ? (inside ? 4 : -28) : f == 4 ? (inside ? -32 : 224) : (inside ? 32 : -224);
    const int no = nbase + dlt;
    float v = 0.0f, cf = (f & 1) ? 0.0f : comp(q, ax);
    if (inside) {
      v = su ? su[no] : ldv<NC>(ut + no);  // su: this tile's values staged in shared memory
      if (ZERO_OWN && nown == colour) v = 0.0f;
      if (f & 1) cf = scm ? scm[ax][no] : __ldg(a.coef + cidx(base + no, 1 + ax));  // scm: staged SoA
    } else {
      const int n = nbp ? nbp[f] : __ldg(a.nbr + 6 * t + f);  // nbp: the caller's prefetched entries
      if (n >= 0) {
        v = ldv<NC>(tptr(a.u, n, a.NL) + no);
        if (ZERO_OWN && nown == colour) v = 0.0f;
        if (f & 1) cf = __ldg(a.coef + cidx((size_t)n * TB3 + no, 1 + ax));
      } else if (n <= -2) {
        if (f & 1)
          cf = __ldg(a.glayer_val + (size_t)__ldg(a.glayer + 3 * t + ax) * 64 +
                     (ax == 0 ? y + 8 * z : (ax == 1 ? x + 8 * z : x + 8 * y)));
        const int C = -2 - n;
        const int4 tv = tvp ? *tvp : __ldg(a.tile + t);
        int g[3] = {tv.y * 8 + c[0], tv.z * 8 + c[1], tv.w * 8 + c[2]};
        g[ax] += sg;
        const int co = loff((g[0] >> 1) & 7, (g[1] >> 1) & 7, (g[2] >> 1) & 7);
        // the coarse leaf's activity and value are loaded together (no dependent load)
        const float cC = __ldg(a.coef + cidx((size_t)C * TB3 + co, 0));
        const float uc = ZERO_OWN ? 0.0f : ldv<NC>(tptr(a.uc, C, a.NL) + co);
        if (cC != 0.0f) v = ui + 0.5f * (uc - mP);
      }
    }
    s = fmaf(cf, v, s);
  }
  return s;
}

__device__ __forceinline__ bool has_ghost(const SmoothArgs& a, int t) {
  bool g = false;
#pragma unroll
  for (int f = 0; f < 6; ++f) g |= __ldg(a.nbr + 6 * t + f) <= -2;
  return g;
}

// mean of the active cells of the 2x2x2 block holding (x,y,z) (pass-start values), summed
// as ((x-pair at dy0,dz0 + x-pair at dy1,dz0) + (dy0,dz1 + dy1,dz1)) — the order of the
// row kernels' shuffle sums (rowtile.cuh row_block_mean), so every kernel forms the same m_P
template <bool ZERO_OWN, int NC = 1>
__device__ __forceinline__ float block_mean(const SmoothArgs& a, int t, int x, int y, int z, int colour) {
  const size_t base = (size_t)t * TB3;
  const float* ut = tptr(a.u, t, a.NL);
  float pr[2][2];
  int nn = 0;
  // the block's cells: q0 + 4 dy + 32 dz in the half of colour (dx + dy + dz) & 1 (the
  // block corner (x&~1, y&~1, z&~1) has even coordinates, hence colour 0)
  const int q0 = (x >> 1) + 4 * (y & ~1) + 32 * (z & ~1);
#pragma unroll
  for (int dz = 0; dz < 2; ++dz)
#pragma unroll
    for (int dy = 0; dy < 2; ++dy) {
      float v[2];
#pragma unroll
      for (int dx = 0; dx < 2; ++dx) {
        const int cb = (dx + dy + dz) & 1;
        const int bo = (cb << 8) + q0 + 4 * dy + 32 * dz;
        const float cc = __ldg(a.coef + cidx(base + bo, 0));
        float bv = ldv<NC>(ut + bo);  // loaded with the activity (no load behind a branch)
        if (ZERO_OWN && cb == colour) bv = 0.0f;
        v[dx] = cc != 0.0f ? bv : 0.0f;
        nn += cc != 0.0f;
      }
      pr[dz][dy] = v[0] + v[1];
    }
  const float sm = (pr[0][0] + pr[0][1]) + (pr[1][0] + pr[1][1]);
  return nn ? sm / (float)nn : 0.0f;
}


}  // namespace octmg

