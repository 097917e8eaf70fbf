// Projection operators on the composite octree ("apply the
// pressure gradient to project the velocity field and measure the divergence"; SPEC
// S:L170-178).  Face velocities u6[f][i]: the component along +axis(f) on face f of leaf
// cell i (both cells of a shared face hold a copy); fluid area S = frac h^2; the outward
// flux of face f is s_f u S, s_f = -1 on - faces and +1 on + faces.
//
//  * divergence: b_i = -sum_f s_f u S over the faces of every active leaf cell; a coarse
//    leaf's face toward finer cells sums the fine cells' entries (finer side authoritative).
//  * gradient subtraction: per face the composite operator's flux F_f = kd_f p_i + c_f v_f
//    (kd_f: the face's share of the geometric diagonal, recomputed from kind and w as the
//    assembly does; c_f, v_f: the operator's coupling and neighbour value, Eq. 12 ghosts at
//    T-junctions) and u += s_f F_f / S, so that div(u - G p) = div(u) - A p.
// One thread per cell, one CTA per leaf tile.
#include <algorithm>

#include "nbref.cuh"

namespace octmg {

namespace {

__device__ __forceinline__ float cplane(const float* coef, size_t i, int k) { return __ldg(coef + cidx(i, k)); }

struct ProjArgs {
  const int4* tile;
  const int* nbr;
  const int* child;
  const int* glayer;
  const float* coef;
  const float* glayer_val;
  const uint8_t* kind;
  WIn w;
  const float* frac;  // [6][N] or null (= 1)
  const float* p;
  const float* u6;
  float* u6w;
  float* b;
  int NL;
  uint8_t wall[6];
};

__device__ __forceinline__ float fr(const ProjArgs& a, int f, size_t i) {
  return a.frac ? a.frac[(size_t)f * a.w.N + i] : 1.0f;
}

__global__ __launch_bounds__(512) void k_divergence(ProjArgs a) {
  const int t = blockIdx.x;
  const int off = threadIdx.x;
  int x, y, z;
    slot_xyz(off, x, y, z);
  const size_t i = (size_t)t * TB3 + off;
  const int4 tv = a.tile[t];
  const float h = ldexpf(1.0f, -tv.x) * 0.125f;
  float out = 0.0f;
  if (cplane(a.coef, i, 0) != 0.0f) {
    for (int f = 0; f < 6; ++f) {
      const float sg = (f & 1) ? 1.0f : -1.0f;
      NbRef nb = nb_ref(a.nbr, tv, t, a.NL, x, y, z, f);
      if (nb.what == NB_INNER) {  // finer cells across: their entries of the shared face
        size_t sub[4];
        fine_subs(a.child, a.NL, nb, f, sub);
        const float hs = 0.5f * h;
        for (int k = 0; k < 4; ++k)
          out += sg * a.u6[(size_t)(f ^ 1) * a.w.N + sub[k]] * fr(a, f ^ 1, sub[k]) * (hs * hs);
      } else {
        out += sg * a.u6[(size_t)f * a.w.N + i] * fr(a, f, i) * (h * h);
      }
    }
  }
  a.b[i] = -out;
}

// mean of the active cells of the 2x2x2 block holding (x,y,z) of leaf tile t (values p)
__device__ __forceinline__ float block_mean_p(const ProjArgs& a, int t, int x, int y, int z) {
  float s = 0.0f;
  int n = 0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const size_t j = (size_t)t * TB3 + loff((x & ~1) + dx, (y & ~1) + dy, (z & ~1) + dz);
        if (cplane(a.coef, j, 0) != 0.0f) { s += a.p[j]; n++; }
      }
  return n ? s / (float)n : 0.0f;
}

__global__ __launch_bounds__(512) void k_subtract_gradient(ProjArgs a) {
  const int t = blockIdx.x;
  const int off = threadIdx.x;
  int x, y, z;
    slot_xyz(off, x, y, z);
  const size_t i = (size_t)t * TB3 + off;
  if (cplane(a.coef, i, 0) == 0.0f) return;  // inactive cell: its faces are left unchanged
  const int4 tv = a.tile[t];
  const float h = ldexpf(1.0f, -tv.x) * 0.125f;
  const float pi = a.p[i];
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1;
    const float sg = (f & 1) ? 1.0f : -1.0f;
    NbRef nb = nb_ref(a.nbr, tv, t, a.NL, x, y, z, f);
    float kd = 0.0f, cf = 0.0f, v = 0.0f;
    if (!(f & 1)) cf = cplane(a.coef, i, 1 + ax);
    if (nb.what == NB_WALL) {
      if (a.wall[f]) kd = a.w.w(f, i) * h;
    } else if (nb.what == NB_LEAF) {
      const size_t j = (size_t)nb.tile * TB3 + nb.off;
      if (a.kind[j] != KN) kd = ((f & 1) ? a.w.w(f ^ 1, j) : a.w.w(f, i)) * h;
      if (f & 1) cf = cplane(a.coef, j, 1 + ax);
      v = cplane(a.coef, j, 0) != 0.0f ? a.p[j] : 0.0f;
    } else if (nb.what == NB_INNER) {  // coarse side of a T-junction
      size_t sub[4];
      fine_subs(a.child, a.NL, nb, f, sub);
      for (int k = 0; k < 4; ++k)
        if (a.kind[sub[k]] != KN) kd += 0.5f * a.w.w(f ^ 1, sub[k]) * (0.5f * h);
      const size_t n = (size_t)nb.tile * TB3 + nb.off;
      if (f & 1) cf = cplane(a.coef, n, 1 + ax);
      // inner neighbour value: mean of its active children (all leaves)
      int xn, yn, zn;
      slot_xyz(nb.off, xn, yn, zn);
      const int ct = a.child[8 * (nb.tile - a.NL) + (xn >> 2) + 2 * (yn >> 2) + 4 * (zn >> 2)];
      float s = 0.0f;
      int c = 0;
      for (int dz = 0; dz < 2; ++dz)
        for (int dy = 0; dy < 2; ++dy)
          for (int dx = 0; dx < 2; ++dx) {
            const size_t q = (size_t)ct * TB3 + loff((2 * xn + dx) & 7, (2 * yn + dy) & 7, (2 * zn + dz) & 7);
            if (cplane(a.coef, q, 0) != 0.0f) { s += a.p[q]; c++; }
          }
      v = c ? s / (float)c : 0.0f;
    } else {  // ghost (fine side of a T-junction), Eq. 12
      const size_t C = (size_t)nb.tile * TB3 + nb.off;
      if (a.kind[C] != KN) kd = a.w.w(f, i) * h;
      if (f & 1) {
        const int layer = a.glayer[3 * t + ax];
        cf = layer >= 0 ? a.glayer_val[(size_t)layer * 64 + (ax == 0 ? y + 8 * z : (ax == 1 ? x + 8 * z : x + 8 * y))]
                        : 0.0f;
      }
      if (cplane(a.coef, C, 0) != 0.0f) v = pi + 0.5f * (a.p[C] - block_mean_p(a, t, x, y, z));
    }
    const float F = fmaf(cf, v, kd * pi);
    const float S = fr(a, f, i) * (h * h);
    if (S > 0.0f) a.u6w[(size_t)f * a.w.N + i] = a.u6[(size_t)f * a.w.N + i] + sg * (F / S);
  }
}

ProjArgs proj_args(const Hier& h) {
  const Tree& T = *h.tree;
  ProjArgs a;
  a.tile = T.tile;
  a.nbr = T.nbr;
  a.child = T.child;
  a.glayer = T.glayer;
  a.coef = h.coef;
  a.glayer_val = h.glayer_val;
  a.kind = nullptr;
  a.w = WIn{nullptr, nullptr, (size_t)T.NL * TB3};
  a.frac = nullptr;
  a.p = nullptr;
  a.u6 = nullptr;
  a.u6w = nullptr;
  a.b = nullptr;
  a.NL = T.NL;
  for (int f = 0; f < 6; ++f) a.wall[f] = T.wall[f];
  return a;
}

}  // namespace

// The caller's arrays are in natural cell order; the kernels work in slot order on
// temporaries (the projection is not on the solver's hot path).
template <class T>
static octmg_status tmp(T** p, size_t n, cudaStream_t s) {
  return cudaMallocAsync((void**)p, sizeof(T) * std::max<size_t>(n, 1), s) == cudaSuccess ? OCTMG_OK
                                                                                     : cuda_status(cudaErrorMemoryAllocation, "projection temporaries");
}

octmg_status divergence(const Hier& h, const float* frac, const float* u6, float* b, cudaStream_t s) {
  const int64_t N = (int64_t)h.tree->NL * TB3;
  float *fr_s = nullptr, *u_s = nullptr, *b_s = nullptr;
  if (frac) {
    OCTMG_TRY(tmp(&fr_s, 6 * (size_t)N, s));
    launch_permute_f32(frac, fr_s, N, 6, true, s);
  }
  OCTMG_TRY(tmp(&u_s, 6 * (size_t)N, s));
  OCTMG_TRY(tmp(&b_s, (size_t)N, s));
  launch_permute_f32(u6, u_s, N, 6, true, s);
  ProjArgs a = proj_args(h);
  a.frac = fr_s;
  a.u6 = u_s;
  a.b = b_s;
  if (h.tree->NL) k_divergence<<<h.tree->NL, TB3, 0, s>>>(a);
  launch_permute_f32(b_s, b, N, 1, false, s);
  if (fr_s) cudaFreeAsync(fr_s, s);
  cudaFreeAsync(u_s, s);
  cudaFreeAsync(b_s, s);
  OCTMG_CUDA(cudaGetLastError());
  return OCTMG_OK;
}

octmg_status subtract_gradient(const Hier& h, const uint8_t* kind, const float* fbeta, const float* frac,
                               const float* p, float* u6, cudaStream_t s) {
  const int64_t N = (int64_t)h.tree->NL * TB3;
  uint8_t* k_s = nullptr;
  float *be_s = nullptr, *fr_s = nullptr, *p_s = nullptr, *u_s = nullptr;
  OCTMG_TRY(tmp(&k_s, (size_t)N, s));
  launch_permute_u8(kind, k_s, N, true, s);
  if (fbeta) {
    OCTMG_TRY(tmp(&be_s, 6 * (size_t)N, s));
    launch_permute_f32(fbeta, be_s, N, 6, true, s);
  }
  if (frac) {
    OCTMG_TRY(tmp(&fr_s, 6 * (size_t)N, s));
    launch_permute_f32(frac, fr_s, N, 6, true, s);
  }
  OCTMG_TRY(tmp(&p_s, (size_t)N, s));
  OCTMG_TRY(tmp(&u_s, 6 * (size_t)N, s));
  launch_permute_f32(p, p_s, N, 1, true, s);
  launch_permute_f32(u6, u_s, N, 6, true, s);
  ProjArgs a = proj_args(h);
  a.kind = k_s;
  a.w = WIn{be_s, fr_s, (size_t)N};
  a.frac = fr_s;
  a.p = p_s;
  a.u6 = u_s;
  a.u6w = u_s;  // in place: each thread reads and writes only its own cell's six entries
  if (h.tree->NL) k_subtract_gradient<<<h.tree->NL, TB3, 0, s>>>(a);
  launch_permute_f32(u_s, u6, N, 6, false, s);
  cudaFreeAsync(k_s, s);
  if (be_s) cudaFreeAsync(be_s, s);
  if (fr_s) cudaFreeAsync(fr_s, s);
  cudaFreeAsync(p_s, s);
  cudaFreeAsync(u_s, s);
  OCTMG_CUDA(cudaGetLastError());
  return OCTMG_OK;
}

}  // namespace octmg
