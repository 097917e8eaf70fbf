// Cell-level neighbour lookup on the tile octree shared by the coefficient assembly
// (setup.cu) and the projection operators (projection.cu): what lies across face f of
// cell (x,y,z) of tile t (same-level leaf / inner cell, domain wall, or ghost whose coarse
// leaf cell is given), the per-face weight w = beta * frac of a leaf cell, and the fine
// sub-cells of an inner neighbour touching a face.
#pragma once
#include "octmg_internal.cuh"

namespace octmg {
namespace nbr_detail {

enum { NB_WALL = 0, NB_LEAF = 1, NB_INNER = 2, NB_GHOST = 3 };
enum { KF = 0, KD = 1, KN = 2 };

struct NbRef {
  int what, tile, off;
};

__device__ __forceinline__ int loff(int x, int y, int z) { return cslot(x, y, z); }  // slot order

// neighbour of cell (x,y,z) of tile t (tile coords tv) across face f
__device__ __forceinline__ NbRef nb_ref(const int* nbr, int4 tv, int t, int NL, int x, int y, int z, int f) {
  int a = f >> 1, s = (f & 1) ? 1 : -1;
  int c[3] = {x, y, z};
  c[a] += s;
  if (c[a] >= 0 && c[a] < 8) return {t < NL ? NB_LEAF : NB_INNER, t, loff(c[0], c[1], c[2])};
  int n = nbr[6 * t + f];
  if (n == -1) return {NB_WALL, -1, -1};
  if (n >= 0) {
    c[a] &= 7;
    return {n < NL ? NB_LEAF : NB_INNER, n, loff(c[0], c[1], c[2])};
  }
  // ghost: the level-(l-1) leaf cell containing the fine neighbour position
  int g[3] = {tv.y * 8 + x, tv.z * 8 + y, tv.w * 8 + z};
  g[a] += s;
  return {NB_GHOST, -2 - n, loff((g[0] >> 1) & 7, (g[1] >> 1) & 7, (g[2] >> 1) & 7)};
}

struct WIn {
  const float* beta;  // [6][N] or null
  const float* frac;  // [6][N] or null
  size_t N;
  __device__ __forceinline__ float w(int f, size_t i) const {
    float v = 1.0f;
    if (beta) v = beta[(size_t)f * N + i];
    if (frac) v = beta ? v * frac[(size_t)f * N + i] : frac[(size_t)f * N + i];
    return v;
  }
};

// the 4 fine sub-cells (leaf cells at level l+1) of the inner cell nb that touch the
// fine-to-coarse face f of our cell; order dz, dy, dx as in the oracle
__device__ __forceinline__ void fine_subs(const int* child, int NL, const NbRef& nb, int f, size_t out[4]) {
  int xn, yn, zn;
  slot_xyz(nb.off, xn, yn, zn);
  int ct = child[8 * (nb.tile - NL) + (xn >> 2) + 2 * (yn >> 2) + 4 * (zn >> 2)];
  int a = f >> 1;
  int facing = (f & 1) ? 0 : 1;
  int k = 0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        int d[3] = {dx, dy, dz};
        if (d[a] != facing) continue;
        out[k++] = (size_t)ct * TB3 + loff((2 * xn + dx) & 7, (2 * yn + dy) & 7, (2 * zn + dz) & 7);
      }
}


}  // namespace nbr_detail
using namespace nbr_detail;
}  // namespace octmg
