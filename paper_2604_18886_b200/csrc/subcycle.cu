// On-chip coarse sub-cycle (sm_100a): the whole FAS-style mu-cycle below a small level K
// (Alg. 4) runs inside ONE CTA of 1024 threads, phase by phase with
// __syncthreads between phases, instead of ~30 tiny kernel launches per visit.  The levels
// it covers hold <= 16 tiles each (8K cells), so every phase is a few L1/L2 round trips;
// their data stays in L1/L2.  Same per-cell arithmetic as the tile kernels (stencil.cuh),
// with coherent loads (NC = false) because the CTA reads what it wrote in earlier phases.
#include "stencil.cuh"

namespace octmg {

namespace {

constexpr int SUB_THREADS = 1024;
constexpr int SUB_MAXL = 4;
constexpr int SUB_MAX_PER_THREAD = 4;  // colour cells per thread (16 tiles * 256 / 1024)

struct SubArgs {
  SmoothArgs a;
  int L;                 // finest level of the tree
  int K;                 // top level of this sub-cycle
  int fas_first;         // form the FAS rhs of level K's inner rows first
  int mu, nu_pre, nu_post, nu_coarsest;
  const int* order_all;  // tiles of each level in rank order
  int lvl_off[SUB_MAXL + 1], lvl_n[SUB_MAXL + 1];
  int ib[SUB_MAXL + 1], ic[SUB_MAXL + 1];
};

__device__ void sc_pass(const SubArgs& A, int l, int colour, int mode) {
  const SmoothArgs& a = A.a;
  const int* ord = A.order_all + A.lvl_off[l];
  const int ncell = A.lvl_n[l] * 256;
  float unew[SUB_MAX_PER_THREAD];
  float* dst[SUB_MAX_PER_THREAD];
  int k = 0;
  for (int s = threadIdx.x; s < ncell; s += SUB_THREADS, ++k) {
    const int t = ord[s >> 8];
    const int j = s & 255;
    const int y = (j >> 2) & 7, z = j >> 5;
    const int x = 2 * (j & 3) + ((colour + y + z) & 1);
    const int off = loff(x, y, z);
    float* ut = tptr(a.u, t, a.NL);
    const float4 q = __ldg(a.coef + (size_t)t * TB3 + off);
    const float b = ldv<false>(tptr(a.b, t, a.NL) + off);
    dst[k] = nullptr;
    unew[k] = 0.0f;
    if (q.x != 0.0f) {
      if (mode == SM_ZERO1) {
        unew[k] = b / q.x;
      } else {
        const bool z2 = mode == SM_ZERO2;
        float ui = 0.0f, mP = 0.0f;
        if (has_ghost(a, t)) {
          ui = z2 ? 0.0f : ldv<false>(ut + off);
          mP = z2 ? block_mean<true, false>(a, t, x, y, z, colour) : block_mean<false, false>(a, t, x, y, z, colour);
        }
        const float fs = z2 ? face_sum<true, false>(a, t, x, y, z, q, ui, mP, colour, 0.0f)
                            : face_sum<false, false>(a, t, x, y, z, q, ui, mP, colour, 0.0f);
        unew[k] = (b - fs) / q.x;
      }
      dst[k] = ut + off;
    } else if (mode == SM_ZERO1 || mode == SM_ZERO2) {
      dst[k] = ut + off;
    }
  }
  __syncthreads();  // all pass-start reads before the in-place writes
  for (int i = 0; i < k; ++i)
    if (dst[i]) *dst[i] = unew[i];
  __syncthreads();
}

__device__ void sc_passes(const SubArgs& A, int l, int iters, bool red_first, int m1, int m2) {
  for (int k = 0; k < iters; ++k) {
    sc_pass(A, l, red_first ? 0 : 1, k == 0 ? m1 : SM_PLAIN);
    sc_pass(A, l, red_first ? 1 : 0, k == 0 ? m2 : SM_PLAIN);
  }
}

// residual + restriction + Avg of level l into level l-1 (k_restrict_direct's arithmetic)
__device__ void sc_restrict(const SubArgs& A, int l) {
  const SmoothArgs& a = A.a;
  const int* ord = A.order_all + A.lvl_off[l];
  const int n = A.lvl_n[l];
  for (int t0 = 0; t0 < n; t0 += SUB_THREADS / 256) {
    const int ti = t0 + (threadIdx.x >> 8);
    if (ti < n) {  // uniform per 256-thread group, so the shuffles below are converged
      const int t = ord[ti];
      const int j = threadIdx.x & 255;
      const int x2 = j & 3;
      const int y = ((j >> 2) & 1) | (((j >> 4) & 3) << 1);
      const int z = ((j >> 3) & 1) | ((j >> 6) << 1);
      const int x0 = 2 * x2;
      const size_t base = (size_t)t * TB3;
      const int off0 = loff(x0, y, z);
      const float4 q0 = __ldg(a.coef + base + off0), q1 = __ldg(a.coef + base + off0 + 1);
      const float* ut = tptr(a.u, t, a.NL);
      const float* bt = tptr(a.b, t, a.NL);
      const float u0 = ut[off0], u1 = ut[off0 + 1];
      const float b0 = bt[off0], b1 = bt[off0 + 1];
      float su = (q0.x != 0.0f ? u0 : 0.0f) + (q1.x != 0.0f ? u1 : 0.0f);
      int na = (q0.x != 0.0f) + (q1.x != 0.0f);
      su += __shfl_xor_sync(0xffffffffu, su, 4);
      na += __shfl_xor_sync(0xffffffffu, na, 4);
      su += __shfl_xor_sync(0xffffffffu, su, 8);
      na += __shfl_xor_sync(0xffffffffu, na, 8);
      const float mP = na ? su / (float)na : 0.0f;
      float r0 = 0.0f, r1 = 0.0f;
      if (q0.x != 0.0f) r0 = b0 - face_sum<false, false>(a, t, x0, y, z, q0, u0, mP, 0, q0.x * u0);
      if (q1.x != 0.0f) r1 = b1 - face_sum<false, false>(a, t, x0 + 1, y, z, q1, u1, mP, 0, q1.x * u1);
      float rs = r0 + r1;
      rs += __shfl_xor_sync(0xffffffffu, rs, 4);
      rs += __shfl_xor_sync(0xffffffffu, rs, 8);
      if (((j >> 2) & 3) == 0) {
        const int4 tv = __ldg(a.tile + t);
        const int P = __ldg(a.parent + t);
        const size_t pi = (size_t)(P - a.NL) * TB3 + pcell_of(tv, x0, y, z);
        a.u.inner[pi] = mP;
        a.ustar_w[pi] = mP;
        a.b.inner[pi] = a.beta * (rs / a.alpha);
      }
    }
  }
  __syncthreads();
}

// b_I = beta R r (in b) + (A^l u*)_I on the inner rows of level l (Alg. 4 line 10)
__device__ void sc_fasrhs(const SubArgs& A, int l) {
  const SmoothArgs& a = A.a;
  const int ncell = A.ic[l] * TB3;
  for (int s = threadIdx.x; s < ncell; s += SUB_THREADS) {
    const int t = A.ib[l] + (s >> 9);
    const int off = s & 511;
    const int x = off & 7, y = (off >> 3) & 7, z = off >> 6;
    const float4 q = __ldg(a.coef + (size_t)t * TB3 + off);
    float* bi = a.b.inner + (size_t)(t - a.NL) * TB3 + off;
    if (q.x != 0.0f) {
      const float u = tptr(a.u, t, a.NL)[off];
      *bi = *bi + face_sum<false, false>(a, t, x, y, z, q, 0.0f, 0.0f, 0, q.x * u);  // no ghosts
    } else {
      *bi = 0.0f;
    }
  }
  __syncthreads();
}

// u += P (u^{l-1} - u*) on the active cells of level l (Alg. 4 line 15)
__device__ void sc_prolong(const SubArgs& A, int l) {
  const SmoothArgs& a = A.a;
  const int* ord = A.order_all + A.lvl_off[l];
  const int ncell = A.lvl_n[l] * TB3;
  for (int s = threadIdx.x; s < ncell; s += SUB_THREADS) {
    const int t = ord[s >> 9];
    const int off = s & 511;
    if (__ldg(a.coef + (size_t)t * TB3 + off).x == 0.0f) continue;
    const int4 tv = __ldg(a.tile + t);
    const int P = __ldg(a.parent + t);
    const int pc = pcell_of(tv, off & 7, (off >> 3) & 7, off >> 6);
    tptr(a.u, t, a.NL)[off] += tptr(a.uc, P, a.NL)[pc] - a.ustar[(size_t)(P - a.NL) * TB3 + pc];
  }
  __syncthreads();
}

// compile-time level recursion (no device call stack): sc_fas<l> calls sc_fas<l-1>
template <int l>
__device__ void sc_fas(const SubArgs& A, bool fas_first);

template <int l>
__device__ __forceinline__ void sc_fas_level(const SubArgs& A, bool fas_first) {
  if (l < A.L && fas_first && A.ic[l] > 0) sc_fasrhs(A, l);
  const bool finest = l == A.L;
  if constexpr (l == 0) {
    const int h1 = A.nu_coarsest / 2;
    sc_passes(A, 0, h1, true, finest ? SM_ZERO1 : SM_PLAIN, finest ? SM_ZERO2 : SM_PLAIN);
    const bool zz = finest && h1 == 0;
    sc_passes(A, 0, A.nu_coarsest - h1, false, zz ? SM_ZERO1 : SM_PLAIN, zz ? SM_ZERO2 : SM_PLAIN);
  } else {
    sc_passes(A, l, A.nu_pre, true, finest ? SM_ZERO1 : SM_PLAIN, finest ? SM_ZERO2 : SM_PLAIN);
    sc_restrict(A, l);
    for (int k = 0; k < A.mu; ++k) sc_fas<l - 1>(A, k == 0);
    sc_prolong(A, l);
    sc_passes(A, l, A.nu_post, false, SM_PLAIN, SM_PLAIN);
  }
}

template <int l>
__device__ void sc_fas(const SubArgs& A, bool fas_first) {
  sc_fas_level<l>(A, fas_first);
}

__global__ __launch_bounds__(SUB_THREADS, 1) void k_subcycle(SubArgs A) {
  const bool ff = A.fas_first != 0;
  switch (A.K) {
    case 0: sc_fas<0>(A, ff); break;
    case 1: sc_fas<1>(A, ff); break;
    case 2: sc_fas<2>(A, ff); break;
    case 3: sc_fas<3>(A, ff); break;
    default: sc_fas<4>(A, ff); break;
  }
}

}  // namespace

int subcycle_max_tiles() { return SUB_THREADS * SUB_MAX_PER_THREAD / 256; }
int subcycle_max_level() { return SUB_MAXL; }

void launch_subcycle(const SmoothArgs& base, int L, int K, int fas_first, const octmg_mg_params& prm,
                     const int* order_all, const int* lvl_off, const int* lvl_n, const int* ib, const int* ic,
                     cudaStream_t s) {
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
  for (int l = 0; l <= SUB_MAXL; ++l) {
    A.lvl_off[l] = l <= K ? lvl_off[l] : 0;
    A.lvl_n[l] = l <= K ? lvl_n[l] : 0;
    A.ib[l] = l <= K ? ib[l] : 0;
    A.ic[l] = l <= K ? ic[l] : 0;
  }
  k_subcycle<<<1, SUB_THREADS, 0, s>>>(A);
}

}  // namespace octmg
