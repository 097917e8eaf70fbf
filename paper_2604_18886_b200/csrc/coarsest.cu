// Direct solve at the coarsest level (Alg. 4 line 4: "Smooth(nu_b, u^0, b^0) — or
// direct solve"; reading 9b), sm_100a.
//
// Setup (once per hierarchy, fp64): the level-0 operator A0 over the cells of C_0 (a plain
// 7-point matrix: level 0 has no ghosts, and the record form makes it symmetric), its
// connected components over the active cells (label propagation), the floating ones (every
// row sum |sum_j A0_ij| <= 1e-5 A0_ii: no Dirichlet coupling, A0 1_C = 0), the
// regularised R = A0 + sum_floating (s_C/|C|) 1_C 1_C^T, R^{-1} by Gauss-Jordan elimination
// with partial pivoting (one pivot kernel + one grid-wide elimination kernel per step), and
// M0 = R^{-1} P (P: mean removal over each floating component) rounded to fp32 — the exact
// solution operator on components coupled to Dirichlet data, the minimum-norm one on
// floating components.  Per visit: u^0 = M0 b^0, one warp per row, b^0 staged in shared
// memory (k_coarse_direct; the on-chip sub-cycle has its own copy of this step).
#include "stencil.cuh"

namespace octmg {

namespace {

struct C0Map {
  const int* c0tile;
  int lb0, lc0, ib0;
  __device__ __forceinline__ int pos(int t) const { return t >= ib0 ? lc0 + (t - ib0) : t - lb0; }
};

// dense A0 (row i = cell k*512 + slot of level-0 tile c0tile[k]) and the coupling graph
__global__ void k_c0_assemble(const float* coef, const int* nbr, C0Map m, int n, double* A, int* nb6) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int t = m.c0tile[i >> 9], sl = i & 511;
  int x, y, z;
  slot_xyz(sl, x, y, z);
  double* row = A + (size_t)i * n;
  const float ci = coef[cidx((size_t)t * TB3 + sl, 0)];
  for (int f = 0; f < 6; ++f) nb6[6 * i + f] = -1;
  if (ci == 0.0f) return;  // inactive row: zero (the level operator outputs 0)
  row[i] = (double)ci;
  const int c[3] = {x, y, z};
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1, sg = (f & 1) ? 1 : -1;
    int q[3] = {c[0], c[1], c[2]};
    q[ax] += sg;
    int tn = t;
    if (q[ax] < 0 || q[ax] > 7) {
      tn = nbr[6 * t + f];
      if (tn < 0) continue;  // domain wall (level 0 has no ghosts)
      q[ax] &= 7;
    }
    const int sn = cslot(q[0], q[1], q[2]);
    const int j = m.pos(tn) * TB3 + sn;
    if (coef[cidx((size_t)tn * TB3 + sn, 0)] == 0.0f) continue;  // inactive neighbour: value 0
    // -face: own record; +face: the neighbour's -face entry
    const float cf = (f & 1) ? coef[cidx((size_t)tn * TB3 + sn, 1 + ax)] : coef[cidx((size_t)t * TB3 + sl, 1 + ax)];
    row[j] += (double)cf;
    if (cf != 0.0f) nb6[6 * i + f] = j;
  }
}

// components (min-label propagation), row-sum floating test, per-component size and diagonal
// sum (one thread, cell order: deterministic)
__global__ __launch_bounds__(1024) void k_c0_components(const double* A, const int* nb6, int n, int* comp,
                                                         int* csize, double* csum, int* floating) {
  __shared__ int lab[C0_MAX_CELLS];
  __shared__ int changed;
  for (int i = threadIdx.x; i < n; i += blockDim.x) lab[i] = A[(size_t)i * n + i] != 0.0 ? i : -1;
  __syncthreads();
  while (true) {
    if (threadIdx.x == 0) changed = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (lab[i] < 0) continue;
      int mn = lab[i];
      for (int f = 0; f < 6; ++f) {
        const int j = nb6[6 * i + f];
        if (j >= 0) mn = min(mn, lab[j]);
      }
      if (mn < lab[i]) {
        lab[i] = mn;
        changed = 1;
      }
    }
    __syncthreads();
    if (!changed) break;
    __syncthreads();
  }
  // row sums (each thread its rows, column order)
  __shared__ unsigned char coupled[C0_MAX_CELLS];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    coupled[i] = 0;
    if (lab[i] < 0) continue;
    double rs = 0.0;
    for (int j = 0; j < n; ++j) rs += A[(size_t)i * n + j];
    coupled[i] = fabs(rs) > 1e-5 * A[(size_t)i * n + i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 0; i < n; ++i) {
      csize[i] = 0;
      csum[i] = 0.0;
      floating[i] = 1;
    }
    for (int i = 0; i < n; ++i) {
      comp[i] = lab[i];
      if (lab[i] < 0) continue;
      csize[lab[i]]++;
      csum[lab[i]] += A[(size_t)i * n + i];
      if (coupled[i]) floating[lab[i]] = 0;
    }
  }
}

// [R | I]: R = A0 on the active block + the floating components' rank-one terms; identity
// rows / columns for inactive cells
__global__ void k_c0_regularize(const double* A, const int* comp, const int* csize, const double* csum,
                                const int* floating, int n, double* R) {
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)n * n) return;
  const int i = (int)(e / n), j = (int)(e % n);
  double v;
  const int ci = comp[i], cj = comp[j];
  if (ci < 0 || cj < 0) {
    v = i == j ? 1.0 : 0.0;
  } else {
    v = A[e];
    if (ci == cj && floating[ci]) v += (csum[ci] / csize[ci]) / csize[ci];
  }
  R[(size_t)i * 2 * n + j] = v;
  R[(size_t)i * 2 * n + n + j] = i == j ? 1.0 : 0.0;
}

// Gauss-Jordan step k: partial pivot (largest |R_ik|, i >= k, first on ties), row swap,
// normalisation of row k, and the multipliers f_i = R_ik of the other rows
__global__ __launch_bounds__(1024) void k_gj_pivot(double* R, int n, int k, double* f) {
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  const int w = 2 * n;
  double best = -1.0;
  int bidx = n;
  for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double v = fabs(R[(size_t)i * w + k]);
    if (v > best) { best = v; bidx = i; }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double o = bv[threadIdx.x + s];
      const int oi = bi[threadIdx.x + s];
      if (o > bv[threadIdx.x] || (o == bv[threadIdx.x] && oi < bi[threadIdx.x])) {
        bv[threadIdx.x] = o;
        bi[threadIdx.x] = oi;
      }
    }
    __syncthreads();
  }
  const int piv = bi[0];
  if (piv != k)
    for (int j = threadIdx.x; j < w; j += blockDim.x) {
      const double a = R[(size_t)k * w + j];
      R[(size_t)k * w + j] = R[(size_t)piv * w + j];
      R[(size_t)piv * w + j] = a;
    }
  __syncthreads();
  const double d = R[(size_t)k * w + k];
  __syncthreads();
  for (int j = threadIdx.x; j < w; j += blockDim.x) R[(size_t)k * w + j] /= d;
  for (int i = threadIdx.x; i < n; i += blockDim.x) f[i] = i == k ? 0.0 : R[(size_t)i * w + k];
}

__global__ void k_gj_elim(double* R, int n, int k, const double* f) {
  const int w = 2 * n;
  const size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (size_t)n * w) return;
  const int i = (int)(e / w), j = (int)(e % w);
  if (i == k) return;
  const double fi = f[i];
  if (fi != 0.0) R[e] -= fi * R[(size_t)k * w + j];
}

// M0 = R^{-1} P, zero rows / columns for inactive cells; one CTA per row, the per-component
// sums of the row by one thread in column order (deterministic)
__global__ __launch_bounds__(256) void k_c0_final(const double* R, const int* comp, const int* csize,
                                                  const int* floating, int n, float* M0) {
  __shared__ double acc[C0_MAX_CELLS];
  const int i = blockIdx.x;
  const int w = 2 * n;
  const double* ri = R + (size_t)i * w + n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) acc[j] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int j = 0; j < n; ++j)
      if (comp[j] >= 0 && floating[comp[j]]) acc[comp[j]] += ri[j];
  __syncthreads();
  const bool act = comp[i] >= 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double v = 0.0;
    const int cj = comp[j];
    if (act && cj >= 0) {
      v = ri[j];
      if (floating[cj]) v -= acc[cj] / csize[cj];
    }
    M0[(size_t)i * n + j] = (float)v;
  }
}

// u^0 = M0 b^0: b^0 staged in shared memory, one warp per row (float4 columns), lanes summed
// by xor shuffles; only active cells are written
__global__ __launch_bounds__(256) void k_coarse_direct(SmoothArgs a) {
  __shared__ __align__(16) float sb[C0_MAX_CELLS];
  const int n = a.c0n;
  for (int j = threadIdx.x; j < n; j += blockDim.x) sb[j] = __ldg(tptr(a.b, a.c0tile[j >> 9], a.NL) + (j & 511));
  __syncthreads();
  const int i = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= n) return;
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

}  // namespace

void launch_coarse_direct(const SmoothArgs& a, cudaStream_t s) {
  if (a.c0n > 0) k_coarse_direct<<<(a.c0n + 7) / 8, 256, 0, s>>>(a);
}

octmg_status build_coarse_direct(Hier& h, cudaStream_t s) {
  const Tree& T = *h.tree;
  const int ntiles = T.lc[0] + T.ic[0];
  const int n = ntiles * TB3;
  if (n > C0_MAX_CELLS) {
    set_error("direct coarsest solve: level 0 has " + std::to_string(n) + " cells (at most " +
              std::to_string(C0_MAX_CELLS) + ")");
    return OCTMG_E_INVALID;
  }
  std::vector<int> tiles;
  for (int t = T.lb[0]; t < T.lb[0] + T.lc[0]; ++t) tiles.push_back(t);
  for (int t = T.ib[0]; t < T.ib[0] + T.ic[0]; ++t) tiles.push_back(t);
  h.c0tile = (int*)dev_malloc(sizeof(int) * tiles.size());
  h.c0M = (float*)dev_malloc(sizeof(float) * (size_t)n * n);
  if (!h.c0tile || !h.c0M) { set_error("device allocation failed (direct coarsest solve)"); return OCTMG_E_OOM; }
  h.allocs.push_back(h.c0tile);
  h.allocs.push_back(h.c0M);
  OCTMG_CUDA(cudaMemcpyAsync(h.c0tile, tiles.data(), sizeof(int) * tiles.size(), cudaMemcpyHostToDevice, s));
  // scratch (freed below)
  const size_t nn = (size_t)n * n;
  double* A = (double*)dev_malloc(sizeof(double) * nn);
  double* R = (double*)dev_malloc(sizeof(double) * 2 * nn);
  double* f = (double*)dev_malloc(sizeof(double) * n);
  double* csum = (double*)dev_malloc(sizeof(double) * n);
  int* ints = (int*)dev_malloc(sizeof(int) * (size_t)n * 9);
  auto release = [&]() {
    cudaStreamSynchronize(s);
    dev_free(A); dev_free(R); dev_free(f); dev_free(csum); dev_free(ints);
  };
  if (!A || !R || !f || !csum || !ints) {
    release();
    set_error("device allocation failed (direct coarsest solve scratch)");
    return OCTMG_E_OOM;
  }
  int* nb6 = ints;
  int* comp = ints + 6 * (size_t)n;
  int* csize = comp + n;
  int* floating = csize + n;
  C0Map m{h.c0tile, T.lb[0], T.lc[0], T.ib[0]};
  cudaMemsetAsync(A, 0, sizeof(double) * nn, s);
  k_c0_assemble<<<(n + 127) / 128, 128, 0, s>>>(h.ccoef, T.nbr, m, n, A, nb6);
  k_c0_components<<<1, 1024, 0, s>>>(A, nb6, n, comp, csize, csum, floating);
  k_c0_regularize<<<(unsigned)((nn + 255) / 256), 256, 0, s>>>(A, comp, csize, csum, floating, n, R);
  const unsigned eg = (unsigned)((2 * nn + 255) / 256);
  for (int k = 0; k < n; ++k) {
    k_gj_pivot<<<1, 1024, 0, s>>>(R, n, k, f);
    k_gj_elim<<<eg, 256, 0, s>>>(R, n, k, f);
  }
  k_c0_final<<<n, 256, 0, s>>>(R, comp, csize, floating, n, h.c0M);
  cudaError_t e = cudaGetLastError();
  release();
  if (e != cudaSuccess) return cuda_status(e, "direct coarsest solve setup");
  h.c0n = n;
  return OCTMG_OK;
}

}  // namespace octmg
