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

// The tile read across each face of a thread's pair (the own tile inside the tile and at
// walls; x faces: the row-end tiles, read by every lane) and whether the face is a wall.
struct RowTiles {
  int tf[6];
  bool wall[6];
};
__device__ __forceinline__ RowTiles row_tiles(int t, const int (&nb)[6], int y, int z) {
  RowTiles r;
  const bool in[6] = {false, false, y > 0, y < 7, z > 0, z < 7};
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    r.wall[f] = !in[f] && nb[f] < 0;
    r.tf[f] = in[f] || nb[f] < 0 ? t : nb[f];
  }
  return r;
}

// Face sums of the pair.  vals.pair(f, s) / vals.one(f, s): values at slot s of the tile
// across face f (row_tiles); v: the pair's own values; cxm/cym/czm: its -face
// coefficients; cxr/cyp/czp planes: the c_x- / c_y- / c_z- planes of the tiles across the
// x+ (row end) / y+ / z+ faces; s0: the starting sums (the diagonal terms c*u, as the
// general paths start).
template <class V>
__device__ __forceinline__ float2 row2_faces(const V& vals, const RowTiles& rt, int x2, int y, int z, const float2 v,
                                             const float2 cxm, const float2 cym, const float2 czm, const float2 s0,
                                             const float* cx_plane, const float* cy_plane, const float* cz_plane) {
  const unsigned FULL = 0xffffffffu;
  const int x0 = 2 * x2;
  // x-neighbours inside the row (lanes j-1, j+1 of the same row)
  float left = __shfl_up_sync(FULL, v.y, 1);
  float right = __shfl_down_sync(FULL, v.x, 1);
  float cxr = __shfl_down_sync(FULL, cxm.x, 1);  // c_x- of cell x0+2 = +x coupling of x0+1
  // row ends (every lane issues both loads; the four lanes of a row hit the same sectors)
  const int sl = cslot(7, y, z), sr = cslot(0, y, z);
  const float wl = vals.one(0, sl);
  const float wr = vals.one(1, sr);
  const float cr = __ldg(cx_plane + sr);
  if (x2 == 0) left = rt.wall[0] ? 0.0f : wl;
  if (x2 == 3) {
    right = rt.wall[1] ? 0.0f : wr;
    cxr = rt.wall[1] ? 0.0f : cr;
  }
  // the pairs of the y- / y+ / z- / z+ rows: other colour half, q -+ 4 / -+ 32 (wrapped into
  // the neighbour tile: +28 / -28 / +224 / -224)
  const int ob = cslot(x0, y, z) ^ 256;
  const int oym = ob + (y > 0 ? -4 : 28), oyp = ob + (y < 7 ? 4 : -28);
  const int ozm = ob + (z > 0 ? -32 : 224), ozp = ob + (z < 7 ? 32 : -224);
  float2 vym = vals.pair(2, oym), vyp = vals.pair(3, oyp);
  float2 vzm = vals.pair(4, ozm), vzp = vals.pair(5, ozp);
  const float2 cyp = ldpair(cy_plane, oyp);
  const float2 czp = ldpair(cz_plane, ozp);
  const float2 Z2 = make_float2(0.0f, 0.0f);
  if (rt.wall[2]) vym = Z2;
  if (rt.wall[3]) vyp = Z2;
  if (rt.wall[4]) vzm = Z2;
  if (rt.wall[5]) vzp = Z2;
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

// values of one field (a tile-contiguous leaf/inner pair) across the faces
struct FldVals {
  const float* p[6];
  __device__ __forceinline__ float2 pair(int f, int s) const { return ldpair(p[f], s); }
  __device__ __forceinline__ float one(int f, int s) const { return __ldg(p[f] + s); }
};
// z + beta p_old across the faces (leaf vectors; tiles addressed by index to keep the
// register footprint small)
struct DirVals {
  const float* z;
  const float* po;  // null: beta = 0
  int tf[6];
  float beta;
  __device__ __forceinline__ float2 pair(int f, int s) const {
    const size_t b = (size_t)tf[f] << 9;
    float2 v = ldpair(z + b, s);
    if (po) {
      const float2 w = ldpair(po + b, s);
      v.x = fmaf(beta, w.x, v.x);
      v.y = fmaf(beta, w.y, v.y);
    }
    return v;
  }
  __device__ __forceinline__ float one(int f, int s) const {
    const size_t b = (size_t)tf[f] << 9;
    float v = __ldg(z + b + s);
    if (po) v = fmaf(beta, __ldg(po + b + s), v);
    return v;
  }
};

}  // namespace octmg
