// Coarse-cycle kernels (sm_100a): the whole FAS-style mu-cycle below a level (Alg. 4,
// P:L723-756) in ONE launch instead of ~11 launches per level visit.
//
//  * k_subcycle: one CTA of 1024 threads, phases separated by __syncthreads; for the
//    smallest levels (<= 16 tiles each, 8K cells), whose data stays in L1/L2.
//    k_subcycle_cluster (OCTMG_SUBCYCLE_CTAS=8): the same spread over one thread-block
//    cluster of 8 CTAs with the hardware cluster barrier (<= 128 tiles per level).
//  * k_coarse_grid: a persistent cooperative grid (one 1024-thread CTA per SM, co-resident
//    by cooperative launch) for the levels below the finest ones (up to a few thousand
//    tiles each, L2-resident): every phase is spread over all CTAs and ends with a grid
//    barrier; when the recursion reaches the sub-cycle level, CTA 0 runs the rest of the
//    cycle alone (the k_subcycle phases) while the other CTAs wait at the next barrier.
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
constexpr int GRID_MAX_PER_THREAD = 8;  // colour cells per thread of the grid kernel
constexpr int GRID_MAXL = 10;
constexpr int SUB_CLUSTER = 8;          // CTAs of the sub-cycle cluster (portable maximum)

struct SubArgs {
  SmoothArgs a;
  int L;                 // finest level of the tree
  int K;                 // top level of this (sub-)cycle
  int sK;                // grid kernel: levels <= sK run in CTA 0 alone (-1: none)
  int fas_first;         // form the FAS rhs of level K's inner rows first
  int mu, nu_pre, nu_post, nu_coarsest;
  const int* order_all;  // tiles of each level in rank order
  int lvl_off[GRID_MAXL + 1], lvl_n[GRID_MAXL + 1];
  int ib[GRID_MAXL + 1], ic[GRID_MAXL + 1];
  unsigned* bar;         // grid barrier counter (zeroed before the launch)
};

// Phase modes: PM 0 = one CTA (__syncthreads), 1 = cooperative grid (global barrier),
// 2 = one thread-block cluster (hardware cluster barrier).  Phase extent: all threads of the
// launch (PM 1, 2: the grid is one cluster / the co-resident grid) or of this CTA.
template <int PM>
__device__ __forceinline__ int ph_tid() { return PM ? blockIdx.x * SUB_THREADS + threadIdx.x : threadIdx.x; }
template <int PM>
__device__ __forceinline__ int ph_nthreads() { return PM ? gridDim.x * SUB_THREADS : SUB_THREADS; }

// cluster barrier with release/acquire semantics at cluster scope: writes of every CTA of
// the cluster before it are visible to every CTA after it
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// grid barrier: monotonic arrival counter, barrier k waits for k * gridDim arrivals
__device__ __forceinline__ void grid_barrier(const SubArgs& A, unsigned& epoch) {
  __syncthreads();
  epoch += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(A.bar, 1u);
    const volatile unsigned* vb = A.bar;
    while (*vb < epoch) {
    }
    __threadfence();
  }
  __syncthreads();
}

template <int PM>
__device__ __forceinline__ void phase_end(const SubArgs& A, unsigned& epoch) {
  if (PM == 1) grid_barrier(A, epoch);
  else if (PM == 2) cluster_barrier();
  else __syncthreads();
}

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

template <int PM, int M>
__device__ __noinline__ void sc_pass(const SubArgs& A, int l, int colour, int mode, unsigned& epoch) {
  constexpr int MAXK = PM == 1 ? GRID_MAX_PER_THREAD : SUB_MAX_PER_THREAD;
  const SmoothArgs& a = A.a;
  const int* ord = A.order_all + A.lvl_off[l];
  const int ncell = A.lvl_n[l] * 256;
  float unew[MAXK];
  float* dst[MAXK];
  int k = 0;
  for (int s = ph_tid<PM>(); s < ncell && k < MAXK; s += ph_nthreads<PM>(), ++k) {
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
  phase_end<PM>(A, epoch);
}

template <int PM, int M>
__device__ void sc_passes(const SubArgs& A, int l, int iters, bool red_first, int m1, int m2, unsigned& epoch) {
  for (int k = 0; k < iters; ++k) {
    sc_pass<PM, M>(A, l, red_first ? 0 : 1, k == 0 ? m1 : SM_PLAIN, epoch);
    sc_pass<PM, M>(A, l, red_first ? 1 : 0, k == 0 ? m2 : SM_PLAIN, epoch);
  }
}

// residual + restriction + Avg of level l into level l-1 (k_restrict_direct's arithmetic);
// groups of 256 threads own one tile at a time
template <int PM, int M>
__device__ __noinline__ void sc_restrict(const SubArgs& A, int l, unsigned& epoch) {
  const SmoothArgs& a = A.a;
  const int* ord = A.order_all + A.lvl_off[l];
  const int n = A.lvl_n[l];
  const int ngrp = ph_nthreads<PM>() / 256;
  for (int t0 = 0; t0 < n; t0 += ngrp) {
    const int ti = t0 + ph_tid<PM>() / 256;
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
  phase_end<PM>(A, epoch);
}

// b_I = beta R r (in b) + (A^l u*)_I on the inner rows of level l (Alg. 4 line 10)
template <int PM, int M>
__device__ __noinline__ void sc_fasrhs(const SubArgs& A, int l, unsigned& epoch) {
  const SmoothArgs& a = A.a;
  const int ncell = A.ic[l] * TB3;
  for (int s = ph_tid<PM>(); s < ncell; s += ph_nthreads<PM>()) {
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
  phase_end<PM>(A, epoch);
}

// u += P (u^{l-1} - u*) on the active cells of level l (Alg. 4 line 15)
template <int PM, int M>
__device__ __noinline__ void sc_prolong(const SubArgs& A, int l, unsigned& epoch) {
  const SmoothArgs& a = A.a;
  const int* ord = A.order_all + A.lvl_off[l];
  const int ncell = A.lvl_n[l] * TB3;
  for (int s = ph_tid<PM>(); s < ncell; s += ph_nthreads<PM>()) {
    const int t = __ldg(ord + (s >> 9));
    const int off = s & 511;
    if (ldcoef(a.coef, (size_t)t * TB3 + off).x == 0.0f) continue;
    const int4 tv = __ldg(a.tile + t);
    const int P = __ldg(a.parent + t);
    int ox, oy, oz;
    slot_xyz(off, ox, oy, oz);
    const int pc = pcell_of(tv, ox, oy, oz);
    float* up = tptr(a.u, t, a.NL) + off;
    *up = ldv<M>(up) + a.pro_scale * (ldv<M>(tptr(a.uc, P, a.NL) + pc) - ldv<M>(a.ustar + (size_t)(P - a.NL) * TB3 + pc));
  }
  phase_end<PM>(A, epoch);
}

// direct coarsest solve u^0 = M0 b^0 (Alg. 4 line 4; coarsest.cu): every CTA stages
// b^0 in shared memory, then one warp per row over all warps of the phase
template <int PM, int M>
__device__ __noinline__ void sc_direct(const SubArgs& A, unsigned& epoch) {
  __shared__ __align__(16) float sb[C0_MAX_CELLS];
  const SmoothArgs& a = A.a;
  const int n = a.c0n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) sb[j] = ldv<M>(tptr(a.b, a.c0tile[j >> 9], a.NL) + (j & 511));
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int i = ph_tid<PM>() >> 5; i < n; i += ph_nthreads<PM>() >> 5) {
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
  phase_end<PM>(A, epoch);
}

// smoothing at the coarsest level: nu_b/2 x (R,B) then nu_b/2 x (B,R), or the
// direct solve
template <int PM, int M>
__device__ void sc_coarsest(const SubArgs& A, bool finest, unsigned& epoch) {
  if (A.a.c0n > 0) {
    sc_direct<PM, M>(A, epoch);
    return;
  }
  const int h1 = A.nu_coarsest / 2;
  sc_passes<PM, M>(A, 0, h1, true, finest ? SM_ZERO1 : SM_PLAIN, finest ? SM_ZERO2 : SM_PLAIN, epoch);
  const bool zz = finest && h1 == 0;
  sc_passes<PM, M>(A, 0, A.nu_coarsest - h1, false, zz ? SM_ZERO1 : SM_PLAIN, zz ? SM_ZERO2 : SM_PLAIN, epoch);
}

// Alg. 4 from level `top` down, iteratively (explicit per-level count of the mu coarse
// calls made; every thread runs the same control flow).  PM 1: levels <= A.sK run in CTA 0
// alone (the one-CTA version of this function) while the other CTAs wait at a barrier.
template <int PM, int M>
__device__ void sc_cycle(const SubArgs& A, int top, bool fas_first, unsigned& epoch) {
  int done[GRID_MAXL + 1];
  int l = top;
  bool ff = fas_first;
  bool entering = true;
  while (true) {
    if (entering) {
      bool leaf_work = true;
      if constexpr (PM == 1) {
        if (l <= A.sK) {
          if (blockIdx.x == 0) {
            unsigned dummy = 0;
            sc_cycle<0, M>(A, l, ff, dummy);
          }
          grid_barrier(A, epoch);
          leaf_work = false;
        }
      }
      if (leaf_work) {
        if (l < A.L && ff && A.ic[l] > 0 && !A.a.std_form) sc_fasrhs<PM, M>(A, l, epoch);
        const bool finest = l == A.L;
        if (l == 0) {
          sc_coarsest<PM, M>(A, finest, epoch);
        } else {
          sc_passes<PM, M>(A, l, A.nu_pre, true, finest ? SM_ZERO1 : SM_PLAIN, finest ? SM_ZERO2 : SM_PLAIN,
                             epoch);
          sc_restrict<PM, M>(A, l, epoch);
          done[l] = 0;
          l -= 1;
          ff = true;
          continue;  // enter the first coarse call
        }
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
    sc_prolong<PM, M>(A, p, epoch);
    sc_passes<PM, M>(A, p, A.nu_post, false, SM_PLAIN, SM_PLAIN, epoch);
    l = p;  // level p finished
  }
}

__global__ __launch_bounds__(SUB_THREADS, 1) void k_subcycle(SubArgs A) {
  unsigned e = 0;
  sc_cycle<0, 0>(A, A.K, A.fas_first != 0, e);
}

// the sub-cycle spread over one cluster of SUB_CLUSTER CTAs (one per SM).  M = 2: mutable
// data read through L2; M = 0: plain (L1-cached) loads, relying on the cluster barrier's
// release/acquire semantics at cluster scope for visibility of the other CTAs' writes
template <int M>
__global__ __launch_bounds__(SUB_THREADS, 1) void k_subcycle_cluster(SubArgs A) {
  unsigned e = 0;
  sc_cycle<2, M>(A, A.K, A.fas_first != 0, e);
}

__global__ __launch_bounds__(SUB_THREADS, 1) void k_coarse_grid(SubArgs A) {
  unsigned e = 0;
  sc_cycle<1, 2>(A, A.K, A.fas_first != 0, e);
}

SubArgs make_args(const SmoothArgs& base, int L, int K, int sK, int fas_first, const octmg_mg_params& prm,
                  const int* order_all, const int* lvl_off, const int* lvl_n, const int* ib, const int* ic) {
  SubArgs A;
  A.a = base;
  A.L = L;
  A.K = K;
  A.sK = sK;
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
  A.bar = nullptr;
  return A;
}

}  // namespace

// CTAs of the sub-cycle: 1 (default) or a cluster of SUB_CLUSTER (OCTMG_SUBCYCLE_CTAS=8;
// measured slower: every phase then reads through L2)
int subcycle_ctas() {
  const char* e = getenv("OCTMG_SUBCYCLE_CTAS");
  return (e && atoi(e) > 1) ? SUB_CLUSTER : 1;
}
int subcycle_max_tiles(int ctas) { return ctas * SUB_THREADS * SUB_MAX_PER_THREAD / 256; }
int subcycle_max_level() { return SUB_MAXL; }
int coarse_grid_max_level() { return GRID_MAXL; }

// tiles per level the grid kernel takes: GRID_MAX_PER_THREAD colour cells per thread
int coarse_grid_max_tiles(int nblocks) { return nblocks * SUB_THREADS * GRID_MAX_PER_THREAD / 256; }

int coarse_grid_blocks() {
  static int nb = -1;
  if (nb < 0) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_coarse_grid, SUB_THREADS, 0);
    nb = per >= 1 ? sms : 0;
  }
  return nb;
}

void launch_subcycle(const SmoothArgs& base, int L, int K, int fas_first, const octmg_mg_params& prm,
                     const int* order_all, const int* lvl_off, const int* lvl_n, const int* ib, const int* ic,
                     int ctas, cudaStream_t s) {
  SubArgs A = make_args(base, L, K, -1, fas_first, prm, order_all, lvl_off, lvl_n, ib, ic);
  if (ctas <= 1) {
    k_subcycle<<<1, SUB_THREADS, 0, s>>>(A);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(SUB_CLUSTER);
  cfg.blockDim = dim3(SUB_THREADS);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = SUB_CLUSTER;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const char* ld = getenv("OCTMG_SUBCYCLE_LD");
  if (ld && atoi(ld) == 2) cudaLaunchKernelEx(&cfg, k_subcycle_cluster<2>, A);
  else cudaLaunchKernelEx(&cfg, k_subcycle_cluster<0>, A);
}

cudaError_t launch_coarse_grid(const SmoothArgs& base, int L, int K, int sK, int fas_first,
                               const octmg_mg_params& prm, const int* order_all, const int* lvl_off,
                               const int* lvl_n, const int* ib, const int* ic, unsigned* bar, cudaStream_t s) {
  SubArgs A = make_args(base, L, K, sK, fas_first, prm, order_all, lvl_off, lvl_n, ib, ic);
  A.bar = bar;
  cudaError_t e = cudaMemsetAsync(bar, 0, sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  // cooperative launch: every CTA co-resident (the grid barrier relies on it)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(coarse_grid_blocks());
  cfg.blockDim = dim3(SUB_THREADS);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_coarse_grid, A);
}

}  // namespace octmg
