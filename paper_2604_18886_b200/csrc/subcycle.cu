// The tile-layout coarse sub-cycle (sm_100a): the whole FAS-style mu-cycle below a level
// (Alg. 4) in ONE launch of one 1024-thread CTA, phases separated by
// __syncthreads, for the smallest levels (<= 16 tiles each) of trees whose coarse levels hold
// leaves (the complete levels below the coarsest leaf level take the dense shared-memory /
// cluster kernels of coarse_dense.cu instead).  Round 1 also had a cooperative-grid version
// and an 8-CTA cluster version of these phases (measured slower; removed in round 2).
//
// Every phase has the same per-cell arithmetic as the tile kernels (stencil.cuh).  Mapping:
// a tile's cells are handled by 256 consecutive threads of one CTA (colour passes: one
// colour cell per thread and tile), so the in-place colour pass needs only a CTA barrier
// between its reads and writes (it reads other tiles' cells of the other colour only).
// Loads of mutable data: plain in the one-CTA kernel (M = 0), L2-only (__ldcg, M = 2) in
// the grid kernel, where other CTAs wrote them before a grid barrier.
#include <cstdlib>

#include "stencil.cuh"

namespace octmg {

namespace {

constexpr int SUB_THREADS = 1024;
constexpr int SUB_MAXL = 4;
constexpr int SUB_MAX_PER_THREAD = 4;   // colour cells per thread of the one-CTA kernel
constexpr int GRID_MAXL = 10;           // level-table size of the arguments

struct SubArgs {
  SmoothArgs a;
  int L;                 // finest level of the tree
  int K;                 // top level of this (sub-)cycle
  int fas_first;         // form the FAS rhs of level K's inner rows first
  int mu, nu_pre, nu_post, nu_coarsest;
  const int* order_all;  // tiles of each level in rank order
  int lvl_off[GRID_MAXL + 1], lvl_n[GRID_MAXL + 1];
  int ib[GRID_MAXL + 1], ic[GRID_MAXL + 1];
};

__device__ __forceinline__ int ph_tid() { return threadIdx.x; }
__device__ __forceinline__ int ph_nthreads() { return SUB_THREADS; }

// Face sum of a cell of a tile with no ghost face (as face_sum_regular in direct.cu, with
// the sub-cycle's load path M for the values): every neighbour is in the other colour half
// at a fixed slot offset, in this tile or wrapped into the face-neighbour tile.
template <int M>
__device__ __forceinline__ float face_sum_reg(const SmoothArgs& a, int t, const int (&nb)[6], int sl, int x, int y,
                                              int z, const float4& q, float s0 = 0.0f) {
  const int base = sl ^ 256;
  const int p = x & 1;
  const bool in[6] = {x > 0, x < 7, y > 0, y < 7, z > 0, z < 7};
  const int dlt[6] = {in[0] ? p - 1 : 3, in[1] ? p : -3, in[2] ? -4 : 28, in[3] ? 4 : -28, in[4] ? -32 : 224,
                      in[5] ? 32 : -224};
  float s = s0;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1;
    const bool wall = !in[f] && nb[f] < 0;
    const int tn = in[f] || wall ? t : nb[f];
    const int no = base + dlt[f];
    float v = ldv<M>(tptr(a.u, tn, a.NL) + no);
    const float cf = (f & 1) ? __ldg(a.coef + ((size_t)tn << 11) + ((1 + ax) << 9) + no) : comp(q, ax);
    if (wall) v = 0.0f;
    s = fmaf(cf, v, s);
  }
  return s;
}

template <int M>
__device__ __noinline__ void sc_pass(const SubArgs& A, int l, int colour, int mode, unsigned& epoch) {
  constexpr int MAXK = SUB_MAX_PER_THREAD;
  const SmoothArgs& a = A.a;
  const int* ord = A.order_all + A.lvl_off[l];
  const int ncell = A.lvl_n[l] * 256;
  float unew[MAXK];
  float* dst[MAXK];
  int k = 0;
  for (int s = ph_tid(); s < ncell && k < MAXK; s += ph_nthreads(), ++k) {
    const int t = __ldg(ord + (s >> 8));
    const int j = s & 255;
    const int y = (j >> 2) & 7, z = j >> 5;
    const int x = 2 * (j & 3) + ((colour + y + z) & 1);
    const int off = loff(x, y, z);
    float* ut = tptr(a.u, t, a.NL);
    const float4 q = ldcoef(a.coef, (size_t)t * TB3 + off);
    const float b = ldv<M>(tptr(a.b, t, a.NL) + off);
    dst[k] = nullptr;
    unew[k] = 0.0f;
    if (q.x != 0.0f) {
      if (mode == SM_ZERO1) {
        unew[k] = b / q.x;
      } else {
        const bool z2 = mode == SM_ZERO2;
        int nb[6];
#pragma unroll
        for (int f = 0; f < 6; ++f) nb[f] = __ldg(a.nbr + 6 * t + f);
        bool ghost = false;
#pragma unroll
        for (int f = 0; f < 6; ++f) ghost |= nb[f] <= -2;
        float fs;
        if (!ghost) {  // (face neighbours have the other colour: ZERO2 reads them as PLAIN does)
          fs = face_sum_reg<M>(a, t, nb, off, x, y, z, q);  // slot-offset stencil, no ghosts
        } else {
          float ui = 0.0f, mP = 0.0f;
          if (ghost) {
            ui = z2 ? 0.0f : ldv<M>(ut + off);
            mP = z2 ? block_mean<true, M>(a, t, x, y, z, colour) : block_mean<false, M>(a, t, x, y, z, colour);
          }
          fs = z2 ? face_sum<true, M>(a, t, x, y, z, q, ui, mP, colour, 0.0f)
                  : face_sum<false, M>(a, t, x, y, z, q, ui, mP, colour, 0.0f);
        }
        unew[k] = (b - fs) / q.x;
      }
      dst[k] = ut + off;
    } else if (mode == SM_ZERO1 || mode == SM_ZERO2) {
      dst[k] = ut + off;
    }
  }
  __syncthreads();  // all pass-start reads of each tile (one CTA per tile) before the writes
  for (int i = 0; i < k; ++i)
    if (dst[i]) *dst[i] = unew[i];
  __syncthreads();
}

template <int M>
__device__ void sc_passes(const SubArgs& A, int l, int iters, bool red_first, int m1, int m2, unsigned& epoch) {
  for (int k = 0; k < iters; ++k) {
    sc_pass<M>(A, l, red_first ? 0 : 1, k == 0 ? m1 : SM_PLAIN, epoch);
    sc_pass<M>(A, l, red_first ? 1 : 0, k == 0 ? m2 : SM_PLAIN, epoch);
  }
}

// residual + restriction + Avg of level l into level l-1 (k_restrict_direct's arithmetic);
// groups of 256 threads own one tile at a time
template <int M>
__device__ __noinline__ void sc_restrict(const SubArgs& A, int l, unsigned& epoch) {
  const SmoothArgs& a = A.a;
  const int* ord = A.order_all + A.lvl_off[l];
  const int n = A.lvl_n[l];
  const int ngrp = ph_nthreads() / 256;
  for (int t0 = 0; t0 < n; t0 += ngrp) {
    const int ti = t0 + ph_tid() / 256;
    if (ti < n) {  // uniform per 256-thread group, so the shuffles below are converged
      const int t = __ldg(ord + ti);
      const int j = threadIdx.x & 255;
      const int x2 = j & 3;
      const int y = ((j >> 2) & 1) | (((j >> 4) & 3) << 1);
      const int z = ((j >> 3) & 1) | ((j >> 6) << 1);
      const int x0 = 2 * x2;
      const size_t base = (size_t)t * TB3;
      const int off0 = loff(x0, y, z);
      const int off1 = loff(x0 + 1, y, z);
      const float4 q0 = ldcoef(a.coef, base + off0), q1 = ldcoef(a.coef, base + off1);
      const float* ut = tptr(a.u, t, a.NL);
      const float* bt = tptr(a.b, t, a.NL);
      const float u0 = ldv<M>(ut + off0), u1 = ldv<M>(ut + off1);
      const float b0 = ldv<M>(bt + off0), b1 = ldv<M>(bt + off1);
      float su = (q0.x != 0.0f ? u0 : 0.0f) + (q1.x != 0.0f ? u1 : 0.0f);
      int na = (q0.x != 0.0f) + (q1.x != 0.0f);
      su += __shfl_xor_sync(0xffffffffu, su, 4);
      na += __shfl_xor_sync(0xffffffffu, na, 4);
      su += __shfl_xor_sync(0xffffffffu, su, 8);
      na += __shfl_xor_sync(0xffffffffu, na, 8);
      const float mP = na ? su / (float)na : 0.0f;
      float r0 = 0.0f, r1 = 0.0f;
      int nb[6];
#pragma unroll
      for (int f = 0; f < 6; ++f) nb[f] = __ldg(a.nbr + 6 * t + f);
      bool ghost = false;
#pragma unroll
      for (int f = 0; f < 6; ++f) ghost |= nb[f] <= -2;
      if (!ghost) {
        if (q0.x != 0.0f) r0 = b0 - face_sum_reg<M>(a, t, nb, off0, x0, y, z, q0, q0.x * u0);
        if (q1.x != 0.0f) r1 = b1 - face_sum_reg<M>(a, t, nb, off1, x0 + 1, y, z, q1, q1.x * u1);
      } else {
        if (q0.x != 0.0f) r0 = b0 - face_sum<false, M>(a, t, x0, y, z, q0, u0, mP, 0, q0.x * u0);
        if (q1.x != 0.0f) r1 = b1 - face_sum<false, M>(a, t, x0 + 1, y, z, q1, u1, mP, 0, q1.x * u1);
      }
      float rs = r0 + r1;
      rs += __shfl_xor_sync(0xffffffffu, rs, 4);
      rs += __shfl_xor_sync(0xffffffffu, rs, 8);
      if (((j >> 2) & 3) == 0) {
        const int4 tv = __ldg(a.tile + t);
        const int P = __ldg(a.parent + t);
        const size_t pi = (size_t)(P - a.NL) * TB3 + pcell_of(tv, x0, y, z);
        a.u.inner[pi] = a.std_form ? 0.0f : mP;  // Alg. 2: zero coarse guess, u* = 0
        a.ustar_w[pi] = a.std_form ? 0.0f : mP;
        a.b.inner[pi] = a.beta * (rs / a.alpha);
      }
    }
  }
  __syncthreads();
}

// b_I = beta R r (in b) + (A^l u*)_I on the inner rows of level l (Alg. 4 line 10)
template <int M>
__device__ __noinline__ void sc_fasrhs(const SubArgs& A, int l, unsigned& epoch) {
  const SmoothArgs& a = A.a;
  const int ncell = A.ic[l] * TB3;
  for (int s = ph_tid(); s < ncell; s += ph_nthreads()) {
    const int t = A.ib[l] + (s >> 9);
    const int off = s & 511;
    int x, y, z;
    slot_xyz(off, x, y, z);
    const float4 q = ldcoef(a.coef, (size_t)t * TB3 + off);
    float* bi = a.b.inner + (size_t)(t - a.NL) * TB3 + off;
    if (q.x != 0.0f) {
      const float u = ldv<M>(tptr(a.u, t, a.NL) + off);
      *bi = ldv<M>(bi) + face_sum<false, M>(a, t, x, y, z, q, 0.0f, 0.0f, 0, q.x * u);  // no ghosts
    } else {
      *bi = 0.0f;
    }
  }
  __syncthreads();
}

// u += P (u^{l-1} - u*) on the active cells of level l (Alg. 4 line 15)
template <int M>
__device__ __noinline__ void sc_prolong(const SubArgs& A, int l, unsigned& epoch) {
  const SmoothArgs& a = A.a;
  const int* ord = A.order_all + A.lvl_off[l];
  const int ncell = A.lvl_n[l] * TB3;
  for (int s = ph_tid(); s < ncell; s += ph_nthreads()) {
    const int t = __ldg(ord + (s >> 9));
    const int off = s & 511;
    if (ldcoef(a.coef, (size_t)t * TB3 + off).x == 0.0f) continue;
    const int4 tv = __ldg(a.tile + t);
    const int P = __ldg(a.parent + t);
    int ox, oy, oz;
    slot_xyz(off, ox, oy, oz);
    const int pc = pcell_of(tv, ox, oy, oz);
    float* up = tptr(a.u, t, a.NL) + off;
    if (a.pro_active_only && __ldg(a.coef + ((size_t)P << 11) + pc) == 0.0f) continue;  // (GMG mode)
    *up = ldv<M>(up) + a.pro_scale * (ldv<M>(tptr(a.uc, P, a.NL) + pc) - ldv<M>(a.ustar + (size_t)(P - a.NL) * TB3 + pc));
  }
  __syncthreads();
}

// direct coarsest solve u^0 = M0 b^0 (Alg. 4 line 4; coarsest.cu): every CTA stages
// b^0 in shared memory, then one warp per row over all warps of the phase
template <int M>
__device__ __noinline__ void sc_direct(const SubArgs& A, unsigned& epoch) {
  __shared__ __align__(16) float sb[C0_MAX_CELLS];
  const SmoothArgs& a = A.a;
  const int n = a.c0n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) sb[j] = ldv<M>(tptr(a.b, a.c0tile[j >> 9], a.NL) + (j & 511));
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int i = ph_tid() >> 5; i < n; i += ph_nthreads() >> 5) {
    const float4* row = reinterpret_cast<const float4*>(a.c0M + (size_t)i * n);
    float s = 0.0f;
    for (int q = lane; q < n / 4; q += 32) {
      const float4 m = __ldg(row + q);
      const float4 v = *reinterpret_cast<const float4*>(sb + 4 * q);
      s = fmaf(m.x, v.x, s);
      s = fmaf(m.y, v.y, s);
      s = fmaf(m.z, v.z, s);
      s = fmaf(m.w, v.w, s);
    }
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      const int t = a.c0tile[i >> 9], sl = i & 511;
      if (__ldg(a.coef + cidx((size_t)t * TB3 + sl, 0)) != 0.0f) tptr(a.u, t, a.NL)[sl] = s;
    }
  }
  __syncthreads();
}

// smoothing at the coarsest level: nu_b/2 x (R,B) then nu_b/2 x (B,R), or the
// direct solve
template <int M>
__device__ void sc_coarsest(const SubArgs& A, bool finest, unsigned& epoch) {
  if (A.a.c0n > 0) {
    sc_direct<M>(A, epoch);
    return;
  }
  const int h1 = A.nu_coarsest / 2;
  sc_passes<M>(A, 0, h1, true, finest ? SM_ZERO1 : SM_PLAIN, finest ? SM_ZERO2 : SM_PLAIN, epoch);
  const bool zz = finest && h1 == 0;
  sc_passes<M>(A, 0, A.nu_coarsest - h1, false, zz ? SM_ZERO1 : SM_PLAIN, zz ? SM_ZERO2 : SM_PLAIN, epoch);
}

// Alg. 4 from level `top` down, iteratively (explicit per-level count of the mu coarse
// calls made; every thread runs the same control flow)
template <int M>
__device__ void sc_cycle(const SubArgs& A, int top, bool fas_first, unsigned& epoch) {
  int done[GRID_MAXL + 1];
  int l = top;
  bool ff = fas_first;
  bool entering = true;
  while (true) {
    if (entering) {
      if (l < A.L && ff && A.ic[l] > 0 && !A.a.std_form) sc_fasrhs<M>(A, l, epoch);
      const bool finest = l == A.L;
      if (l == 0) {
        sc_coarsest<M>(A, finest, epoch);
      } else {
        sc_passes<M>(A, l, A.nu_pre, true, finest ? SM_ZERO1 : SM_PLAIN, finest ? SM_ZERO2 : SM_PLAIN, epoch);
        sc_restrict<M>(A, l, epoch);
        done[l] = 0;
        l -= 1;
        ff = true;
        continue;  // enter the first coarse call
      }
      entering = false;  // level l finished
    }
    if (l == top) break;
    const int p = l + 1;
    if (++done[p] < A.mu) {  // next coarse call starts from the previous one's u^{l}
      l = p - 1;
      ff = false;
      entering = true;
      continue;
    }
    sc_prolong<M>(A, p, epoch);
    sc_passes<M>(A, p, A.nu_post, false, SM_PLAIN, SM_PLAIN, epoch);
    l = p;  // level p finished
  }
}

__global__ __launch_bounds__(SUB_THREADS, 1) void k_subcycle(SubArgs A) {
  unsigned e = 0;
  sc_cycle<0>(A, A.K, A.fas_first != 0, e);
}

SubArgs make_args(const SmoothArgs& base, int L, int K, int fas_first, const octmg_mg_params& prm,
                  const int* order_all, const int* lvl_off, const int* lvl_n, const int* ib, const int* ic) {
  SubArgs A;
  A.a = base;
  A.L = L;
  A.K = K;
  A.fas_first = fas_first;
  A.mu = prm.mu;
  A.nu_pre = prm.nu_pre;
  A.nu_post = prm.nu_post;
  A.nu_coarsest = prm.nu_coarsest;
  A.order_all = order_all;
  for (int l = 0; l <= GRID_MAXL; ++l) {
    A.lvl_off[l] = l <= K ? lvl_off[l] : 0;
    A.lvl_n[l] = l <= K ? lvl_n[l] : 0;
    A.ib[l] = l <= K ? ib[l] : 0;
    A.ic[l] = l <= K ? ic[l] : 0;
  }
  return A;
}

}  // namespace

int subcycle_max_tiles() { return SUB_THREADS * SUB_MAX_PER_THREAD / 256; }
int subcycle_max_level() { return SUB_MAXL; }

void launch_subcycle(const SmoothArgs& base, int L, int K, int fas_first, const octmg_mg_params& prm,
                     const int* order_all, const int* lvl_off, const int* lvl_n, const int* ib, const int* ic,
                     cudaStream_t s) {
  SubArgs A = make_args(base, L, K, fas_first, prm, order_all, lvl_off, lvl_n, ib, ic);
  k_subcycle<<<1, SUB_THREADS, 0, s>>>(A);
}

}  // namespace octmg
