// 7-point face sums of an x-pair of cells on tiles with no ghost face (every tile of a
// uniform level; most tiles of an adaptive one).  Thread layout of the tile kernels: lane j
// of a 256-thread tile CTA owns cells (x0, y, z), (x0+1, y, z) with x0 = 2*(j&3), so the
// four lanes of an x-row are consecutive lanes of one warp.  In the colour-split slot order
// the two cells of a pair have the same index q = x0/2 + 4y + 32z in opposite colour halves
// (slots sA and sA ^ 256), so every field is read as two fully coalesced scalar loads per
// warp.  The x-neighbours inside the row come from the adjacent lanes by shuffles, the row
// ends from the x-neighbour tiles.  Every load is issued unconditionally (a wall face reads
// the tile itself and is zeroed) so all loads of the pair are in flight at once.  Face
// order of the sums: x-, x+, y-, y+, z-, z+ (the oracle's, the +face coupling
// taken from the neighbour's -face entry).
#pragma once
#include "octmg_internal.cuh"

namespace octmg {

// the two cells of the pair starting at slot sA of a tile-contiguous array
__device__ __forceinline__ float2 ldpair(const float* p, int sA) { return make_float2(__ldg(p + sA), __ldg(p + (sA ^ 256))); }

// val2(tile, sA) -> float2 of the values of the pair at slots sA, sA ^ 256 of `tile`;
// val1(tile, s) -> one value.  cxm/cym/czm: the pair's own -face coefficients; s0: the
// starting sums (the diagonal terms c*u, as the general paths start).  Returns the sums.
template <class V2, class V1>
__device__ __forceinline__ float2 row2_faces(const float* coef, int t, const int (&nb)[6], int x2, int y, int z,
                                             const float2 v, const float2 cxm, const float2 cym, const float2 czm,
                                             const float2 s0, const V2& val2, const V1& val1) {
  const unsigned FULL = 0xffffffffu;
  const int x0 = 2 * x2;
  // x-neighbours inside the row (lanes j-1, j+1 of the same row)
  float left = __shfl_up_sync(FULL, v.y, 1);
  float right = __shfl_down_sync(FULL, v.x, 1);
  float cxr = __shfl_down_sync(FULL, cxm.x, 1);  // c_x- of cell x0+2 = +x coupling of x0+1
  // row ends: every lane issues both edge loads (the four lanes of a row hit the same
  // sectors), so no load waits behind a divergent branch
  const int nl = nb[0], nr = nb[1];
  const int sl = cslot(7, y, z), sr = cslot(0, y, z);
  const float wl = val1(nl >= 0 ? nl : t, sl);
  const float wr = val1(nr >= 0 ? nr : t, sr);
  const float cr = __ldg(coef + ((size_t)(nr >= 0 ? nr : t) << 11) + 512 + sr);
  if (x2 == 0) left = nl >= 0 ? wl : 0.0f;
  if (x2 == 3) {
    right = nr >= 0 ? wr : 0.0f;
    cxr = nr >= 0 ? cr : 0.0f;
  }
  // the pairs of the y- / y+ / z- / z+ rows: other colour half, q -+ 4 / -+ 32 (wrapped into
  // the neighbour tile: +28 / -28 / +224 / -224)
  const int ob = cslot(x0, y, z) ^ 256;
  const int oym = ob + (y > 0 ? -4 : 28), oyp = ob + (y < 7 ? 4 : -28);
  const int ozm = ob + (z > 0 ? -32 : 224), ozp = ob + (z < 7 ? 32 : -224);
  const int nym = y > 0 ? t : nb[2], nyp = y < 7 ? t : nb[3];
  const int nzm = z > 0 ? t : nb[4], nzp = z < 7 ? t : nb[5];
  float2 vym = val2(nym >= 0 ? nym : t, oym), vyp = val2(nyp >= 0 ? nyp : t, oyp);
  float2 vzm = val2(nzm >= 0 ? nzm : t, ozm), vzp = val2(nzp >= 0 ? nzp : t, ozp);
  const float2 cyp = ldpair(coef + ((size_t)(nyp >= 0 ? nyp : t) << 11) + 1024, oyp);
  const float2 czp = ldpair(coef + ((size_t)(nzp >= 0 ? nzp : t) << 11) + 1536, ozp);
  const float2 Z2 = make_float2(0.0f, 0.0f);
  if (nym < 0) vym = Z2;
  if (nyp < 0) vyp = Z2;
  if (nzm < 0) vzm = Z2;
  if (nzp < 0) vzp = Z2;
  float a0 = fmaf(cxm.x, left, s0.x);
  a0 = fmaf(cxm.y, v.y, a0);
  a0 = fmaf(cym.x, vym.x, a0);
  a0 = fmaf(cyp.x, vyp.x, a0);
  a0 = fmaf(czm.x, vzm.x, a0);
  a0 = fmaf(czp.x, vzp.x, a0);
  float a1 = fmaf(cxm.y, v.x, s0.y);
  a1 = fmaf(cxr, right, a1);
  a1 = fmaf(cym.y, vym.y, a1);
  a1 = fmaf(cyp.y, vyp.y, a1);
  a1 = fmaf(czm.y, vzm.y, a1);
  a1 = fmaf(czp.y, vzp.y, a1);
  return make_float2(a0, a1);
}

}  // namespace octmg
