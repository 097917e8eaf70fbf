// PCG kernels (sm_100a): the composite leaf operator q = A p with the fp64 p.q reduction,
// and the vector updates / dots.  One 128-thread CTA per 8^3 tile for the operator, one
// colour row of 4 cells per thread (rowtile.cuh); the operator is evaluated in flux form
// with the exact row sums of setup.cu (k_leaf_rowsum); the +face coupling comes from the
// neighbour record or the ghost layer.
#include <algorithm>

#include "octmg_internal.cuh"
#include "rowtile.cuh"

namespace octmg {

namespace {


__device__ __forceinline__ double block_reduce_d(double v, double* sred) {
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) sred[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += sred[k];
  return s;  // valid in thread 0
}

// deterministic last-block reduction: returns true in thread 0 of the last block, with the
// ordered sum of all partials in *total
__device__ __forceinline__ bool last_block_sum(double mine, double* partial, unsigned* counter, int nparts,
                                               double* total, double* sred) {
  __shared__ bool is_last;
  if (threadIdx.x == 0) {
    partial[blockIdx.x] = mine;
    __threadfence();
    unsigned prev = atomicAdd(counter, 1u);
    is_last = prev == (unsigned)nparts - 1;
  }
  __syncthreads();
  if (!is_last) return false;
  __threadfence();
  double s = 0.0;
  for (int k = threadIdx.x; k < nparts; k += blockDim.x) s += ((volatile double*)partial)[k];
  // fixed-order tree over threads
  __syncthreads();
  double tot = block_reduce_d(s, sred);
  if (threadIdx.x == 0) { *total = tot; *counter = 0u; }
  return threadIdx.x == 0;
}

// q = A p (composite leaf operator; p precomputed by k_pupdate, split PCG form)
// and the per-tile fp64 partial of p.q (Alg. 1 lines 9-10; fp64 dots P:L1233).  One
// colour row per thread (rowtile.cuh): thread j of a 128-thread tile CTA owns row j >> 1 of
// colour j & 1 (the two colours of a row in adjacent lanes, so a warp's float4 loads are two
// contiguous 256-B half-rows).  Tiles with a T-junction face or a same-level inner neighbour
// (IRR, CTA-uniform) take the same row loads and substitute the Eq. 12 ghost entries (m_P
// by shuffles over the rows y^1, z^1 = lanes j^2, j^16) and the inner neighbours'
// active-children means.  Flux form (A p)_i = d_i p_i + sum_f c_f (v_f - p_i) with the exact
// row sums d (setup.cu k_leaf_rowsum, rowk::row_sums_flux); the ghost and inner entries are
// formed directly as differences.  Algorithmic bytes: read p and the 4 record planes, write
// q = 24 B per leaf cell (+4 B on tiles with a nonzero row sum).
// LEAN: a hierarchy without same-level inner neighbours of leaf tiles and without nonzero row
// sums (every uniform tree): no pbar select per neighbour pointer, no row-sum load
template <bool DOT, bool IRR, bool LEAN = false>
__device__ __forceinline__ void apply_row_body(const ApplyArgs& a, int t, const int (&nb)[6], double* sred) {
  using namespace rowk;
  const RowGeo g = row_geo(threadIdx.x & 1, threadIdx.x >> 1);
  const float* pz = a.z;
  const float* ct = a.coef + ((size_t)t << 11);
  const int dk = LEAN ? -1 : __ldg(a.dtile + t);
  const float4 pc = ld4(pz + ((size_t)t << 9) + g.own);
  const float4 c0 = ld4(ct + g.own), cxm = ld4(ct + 512 + g.own), cym = ld4(ct + 1024 + g.own),
               czm = ld4(ct + 1536 + g.own);
  const int NL = a.NL;
  // values of tile n: a leaf's p, or for a same-level inner neighbour the means of its
  // active children precomputed on the face layer the row reads (k_inner_face_means)
  const float* pb = a.pbar;
  auto tu = [pz, pb, NL](int n) -> const float* {
    return (LEAN || n < NL) ? pz + ((size_t)n << 9) : pb + ((size_t)(n - NL) << 9);
  };
  RowSt s;
  row_load<decltype(tu), true>(s, tu, a.coef, t, nb, g);
  const float4 d = dk >= 0 ? ld4(a.dval + ((size_t)dk << 9) + g.own) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  const float4 pv = msk4(pc, c0);
  RowRep rp{false, false, false, false, false};
  if (IRR) {
    const float4 co = ld4(ct + g.oth);
    const float4 mP = row_block_mean<2, 16>(pv, c0, msk4(s.ox, co), co);
    // (the tile origin and ghost-layer indices loaded here, not up front: measured better for
    // the out-of-line irregular body, whose registers are short)
    row_ghosts<false, decltype(tu), true>(s, g, t, nb, __ldg(a.tile + t), a.coef, a.glayer_val,
                                          rowk::load_gl(a.glayer, t), tu, pv, mP, &rp);
  }
  const float4 f = row_sums_flux(s, g, rp, cxm, cym, czm, pv, d);
  const float4 r = make_float4(c0.x != 0.0f ? f.x : 0.0f, c0.y != 0.0f ? f.y : 0.0f, c0.z != 0.0f ? f.z : 0.0f,
                               c0.w != 0.0f ? f.w : 0.0f);
  *reinterpret_cast<float4*>(a.q + ((size_t)t << 9) + g.own) = r;
  if (DOT) {
    // fp64 partials per warp (4 per tile, no CTA barrier: the warps of an irregular tile finish
    // independently) of p.q and of sum q (the null-space projection's mean shift, fused into
    // k_update); k_chunk_sums / k_finish_sigma sum them in tile order (deterministic)
    double dd = (double)pv.x * (double)r.x + (double)pv.y * (double)r.y + (double)pv.z * (double)r.z +
                (double)pv.w * (double)r.w;
    for (int o = 16; o; o >>= 1) dd += __shfl_down_sync(0xffffffffu, dd, o);
    const size_t w = 4 * (size_t)blockIdx.x + (threadIdx.x >> 5);
    if ((threadIdx.x & 31) == 0) a.partial[w] = dd;
    if (a.sumq) {  // (uniform: PCG with the null-space projection)
      double dq = ((double)r.x + (double)r.y) + ((double)r.z + (double)r.w);
      for (int o = 16; o; o >>= 1) dq += __shfl_down_sync(0xffffffffu, dq, o);
      if ((threadIdx.x & 31) == 0) a.partial[4 * (size_t)gridDim.x + w] = dq;
    }
  }
}

// the irregular-tile body out of line (its registers do not lower the regular path's occupancy)
template <bool DOT>
__device__ __noinline__ void apply_row_irr(const ApplyArgs& a, int t, int n0, int n1, int n2, int n3, int n4, int n5,
                                           double* sred) {
  const int nb[6] = {n0, n1, n2, n3, n4, n5};
  apply_row_body<DOT, true>(a, t, nb, sred);
}

// INL: the irregular body inlined, at 6 CTAs/SM (80 registers) instead of out of line at 8
// (measured on configs 3 / 5: inlined at 7 or 8 CTAs/SM, 72 / 64 registers with spills, slower)
template <bool DOT, bool INL, bool LEAN = false>
__global__ __launch_bounds__(128, INL ? 6 : 8) void k_apply_v6(const __grid_constant__ ApplyArgs a) {
  __shared__ double sred[4];
  const int t = a.tiles ? a.tiles[blockIdx.x] : (int)blockIdx.x;
  int nb[6];
  rowk::load_nb(a.nbr, t, nb);
  if (LEAN) {  // (a tree without T-junction tiles: no irregular body, no call frame)
    apply_row_body<DOT, false, true>(a, t, nb, sred);
    return;
  }
  bool irr = false;
#pragma unroll
  for (int f = 0; f < 6; ++f) irr |= nb[f] <= -2;  // ghost faces (inner neighbours read pbar)
  if (irr) {  // CTA-uniform
    if (INL) apply_row_body<DOT, true>(a, t, nb, sred);
    else apply_row_irr<DOT>(a, t, nb[0], nb[1], nb[2], nb[3], nb[4], nb[5], sred);
    return;
  }
  apply_row_body<DOT, false>(a, t, nb, sred);
}

// The composite operator's value across a face toward a same-level inner tile is the mean of
// the active children of the neighbour cell.  One CTA of 64 threads per listed
// (inner tile, face) layer: each thread one cell of the layer, its 8 children (octant
// dx + 2dy + 4dz, activity and value loaded together) — all loads independent, unlike the
// same computation inside the apply's rows.  p is zero on inactive cells.
__global__ __launch_bounds__(64) void k_inner_face_means(const int2* ifaces, const int* child, const float* coef,
                                                        const float* p, float* pbar, int NL) {
  const int2 it = __ldg(ifaces + blockIdx.x);
  const int n = it.x, f = it.y, ax = f >> 1;
  const int c2 = threadIdx.x;
  int c[3];
  c[ax] = (f & 1) ? 7 : 0;
  c[ax == 0 ? 1 : 0] = c2 & 7;
  c[ax == 2 ? 1 : 2] = c2 >> 3;
  const int ct = __ldg(child + 8 * (size_t)(n - NL) + (c[0] >> 2) + 2 * (c[1] >> 2) + 4 * (c[2] >> 2));
  float sm = 0.0f;
  int k = 0;
#pragma unroll
  for (int d = 0; d < 8; ++d) {
    const int sl = cslot((2 * c[0] + (d & 1)) & 7, (2 * c[1] + ((d >> 1) & 1)) & 7, (2 * c[2] + (d >> 2)) & 7);
    const float cc = __ldg(coef + ((size_t)ct << 11) + sl);
    const float v = __ldg(p + ((size_t)ct << 9) + sl);
    if (cc != 0.0f) { sm += v; k++; }
  }
  pbar[((size_t)(n - NL) << 9) + cslot(c[0], c[1], c[2])] = k ? sm / (float)k : 0.0f;
}

// first stage of the p.q sum: block b adds the contiguous chunk b of the per-warp partials
// in a fixed order (deterministic), so the final single-CTA stage reads a few hundred values
__global__ __launch_bounds__(256) void k_chunk_sums(const double* partial, int64_t n, int64_t chunk, double* out) {
  __shared__ double sred[8];
  partial += blockIdx.y * n;  // y = 0: the p.q partials, 1: the sum-q partials
  out += blockIdx.y * gridDim.x;
  const int64_t lo = blockIdx.x * chunk, hi = min(n, lo + chunk);
  double s0 = 0.0, s1 = 0.0;
  int64_t k = lo + threadIdx.x;
  for (; k + 256 < hi; k += 512) {
    s0 += partial[k];
    s1 += partial[k + 256];
  }
  for (; k < hi; k += 256) s0 += partial[k];
  const double bs = block_reduce_d(s0 + s1, sred);
  if (threadIdx.x == 0) out[blockIdx.x] = bs;
}

// sigma = p.q and sum q from the partials (fixed order => deterministic): block 0 the first
// n values (p.q chunks) into sum_pq, block 1 the next n (q chunks) into sum_q
__global__ __launch_bounds__(1024) void k_finish_sigma(const double* partial, int n, Scalars* sc) {
  __shared__ double sred[32];
  partial += (size_t)blockIdx.x * n;
  // four independent accumulators per thread keep several loads in flight (fixed order)
  const int bd = blockDim.x;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = threadIdx.x;
  for (; k + 3 * bd < n; k += 4 * bd) {
    s0 += partial[k];
    s1 += partial[k + bd];
    s2 += partial[k + 2 * bd];
    s3 += partial[k + 3 * bd];
  }
  for (; k < n; k += bd) s0 += partial[k];
  double s = (s0 + s1) + (s2 + s3);
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += sred[w];
    if (blockIdx.x == 0) sc->sum_pq = tot;
    else sc->sum_q = tot;
  }
}

// ------------------------------------------------------------------------------------
// PCG vector kernels over this part's owned leaf cells (float4 index ranges); fixed grid and
// fixed-order last-block reductions => deterministic.  They write raw local sums into the
// Scalars; multi-part jobs sum those across parts before any consumer reads them.
// ------------------------------------------------------------------------------------
// activity nibble of the 4 cells of float4 index i (bit k = cell 4i+k active; mask bit per cell)
__device__ __forceinline__ unsigned act4(const uint32_t* act, int64_t i) { return (act[i >> 3] >> ((i & 7) * 4)) & 0xFu; }

// (the inner loop is unrolled 4x so that several iterations' loads are in flight at once)
#define FOR_RANGES(R, i)                                                                          \
  for (int rr_ = 0; rr_ < (R).n; ++rr_)                                                           \
    _Pragma("unroll 4")                                                                           \
    for (int64_t i = (R).begin[rr_] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;             \
         i < (R).begin[rr_] + (R).len[rr_]; i += (int64_t)gridDim.x * blockDim.x)

// natural-order rows (8 cells x + 8y + 64z of one tile row) of the ranges: q-th row of range rr
// starts at cell 4 begin + 8 q; its red / black halves are the slot-order float4s at
// tile + 4 row and tile + 256 + 4 row (row = y + 8z); cell x = 2m + p of the red half
// (p = (y + z) & 1) is natural x, of the black half 2m + 1 - p
#define FOR_ROWS(R, c0)                                                                           \
  for (int rr_ = 0; rr_ < (R).n; ++rr_)                                                           \
    for (int64_t q_ = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, c0 = 0;                     \
         q_ < (R).len[rr_] / 2 && ((c0 = 4 * (R).begin[rr_] + 8 * q_), true); q_ += (int64_t)gridDim.x * blockDim.x)

// two ordered sums (s2, s1) over the grid; the last block stores them at sc fields f2, f1
__device__ __forceinline__ void reduce2(double s2, double s1, double* partial, unsigned* counter, Scalars* sc,
                                        int f2, int f1, double* sred) {
  double b2 = block_reduce_d(s2, sred);
  __syncthreads();
  double b1 = block_reduce_d(s1, sred);
  double tot;
  if (threadIdx.x == 0) partial[gridDim.x + blockIdx.x] = b1;
  if (last_block_sum(b2, partial, counter, gridDim.x, &tot, sred)) {
    double t1 = 0.0;
    for (int k = 0; k < (int)gridDim.x; ++k) t1 += ((volatile double*)partial)[gridDim.x + k];
    reinterpret_cast<double*>(sc)[f2] = tot;
    if (f1 >= 0) reinterpret_cast<double*>(sc)[f1] = t1;
  }
}

// r = b on active cells (0 elsewhere), x = 0; sums ||r||^2, sum r (Alg. 1 lines 3-4).
// r and x are internal (slot order), b the caller's vector (natural order).
__global__ __launch_bounds__(256) void k_init(const float* b, const uint32_t* act, float* r, float* x, Ranges R,
                                              double* partial, unsigned* counter, Scalars* sc) {
  __shared__ double sred[8];
  double s2 = 0.0, s1 = 0.0;
  FOR_ROWS(R, c0) {
    // b is in the caller's natural cell order: one natural row (two 128-bit loads) gives the
    // red and the black colour row of the slot order
    const int64_t tb = c0 & ~(int64_t)511;
    const int row = (int)((c0 & 511) >> 3), y = row & 7, z = row >> 3, p = (y + z) & 1;
    const float4 n0 = __ldg(reinterpret_cast<const float4*>(b + c0)), n1 = __ldg(reinterpret_cast<const float4*>(b + c0 + 4));
    const float nv[8] = {n0.x, n0.y, n0.z, n0.w, n1.x, n1.y, n1.z, n1.w};
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t i = (tb + (c << 8) + 4 * row) >> 2;  // float4 index of the colour row
      const int pc = c ? 1 - p : p;
      float m[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) m[k] = nv[2 * k + pc];
      const unsigned am = act4(act, i);
      for (int k = 0; k < 4; ++k) {
        if (!((am >> k) & 1u)) m[k] = 0.0f;
        s2 += (double)m[k] * m[k];
        s1 += (double)m[k];
      }
      reinterpret_cast<float4*>(r)[i] = make_float4(m[0], m[1], m[2], m[3]);
      reinterpret_cast<float4*>(x)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->flags = 0;
  reduce2(s2, s1, partial, counter, sc, SF_RR, SF_R, sred);
}

// x += alpha p, r -= alpha q with alpha = (r,z)/(p,Ap) (Alg. 1 lines 9-11); sums ||r||^2,
// sum r.  The last block flags a breakdown and records rho = (r, z) for the next beta.
// alpha_fixed != 0: that step length instead (standalone multigrid: x += z, r -= A z)
// act (PCG with the null-space projection): the projection of the new r fused in,
// r -= m on the active cells with m = mean_active(r - alpha q) = (sum r - alpha sum q) / n
// formed from the sums of the projected r (previous update / initial projection) and of q
// (the apply) — the k_project pass and its 8 B/leaf are gone from the loop
__global__ __launch_bounds__(256) void k_update(float* __restrict__ x, float* __restrict__ r,
                                                const float* __restrict__ p, const float* __restrict__ q, Ranges R,
                                                double* partial, unsigned* counter, Scalars* sc, float alpha_fixed,
                                                const uint32_t* __restrict__ act) {
  __shared__ double sred[8];
  const double pq = sc->sum_pq, rz = sc->sum_rz;
  const bool ok = alpha_fixed != 0.0f || (pq > 0.0 && isfinite(pq) && isfinite(rz));
  const float alpha = alpha_fixed != 0.0f ? alpha_fixed : (ok ? (float)(rz / pq) : 0.0f);
  const float m = act ? (float)((sc->sum_r - (double)alpha * sc->sum_q) / sc->n_active) : 0.0f;
  double s2 = 0.0, s1 = 0.0;
  FOR_RANGES(R, i) {
    float4 xv = reinterpret_cast<float4*>(x)[i];
    float4 rv = reinterpret_cast<float4*>(r)[i];
    float4 pv = __ldg(reinterpret_cast<const float4*>(p) + i);
    float4 qv = __ldg(reinterpret_cast<const float4*>(q) + i);
    xv.x = fmaf(alpha, pv.x, xv.x); xv.y = fmaf(alpha, pv.y, xv.y);
    xv.z = fmaf(alpha, pv.z, xv.z); xv.w = fmaf(alpha, pv.w, xv.w);
    rv.x = fmaf(-alpha, qv.x, rv.x); rv.y = fmaf(-alpha, qv.y, rv.y);
    rv.z = fmaf(-alpha, qv.z, rv.z); rv.w = fmaf(-alpha, qv.w, rv.w);
    if (act) {
      const unsigned am = act4(act, i);
      if (am & 1u) rv.x -= m;
      if (am & 2u) rv.y -= m;
      if (am & 4u) rv.z -= m;
      if (am & 8u) rv.w -= m;
    }
    reinterpret_cast<float4*>(x)[i] = xv;
    reinterpret_cast<float4*>(r)[i] = rv;
    s2 += (double)rv.x * rv.x + (double)rv.y * rv.y + (double)rv.z * rv.z + (double)rv.w * rv.w;
    s1 += (double)rv.x + (double)rv.y + (double)rv.z + (double)rv.w;
  }
  double b2 = block_reduce_d(s2, sred);
  __syncthreads();
  double b1 = block_reduce_d(s1, sred);
  double tot;
  if (threadIdx.x == 0) partial[gridDim.x + blockIdx.x] = b1;
  if (last_block_sum(b2, partial, counter, gridDim.x, &tot, sred)) {
    double t1 = 0.0;
    for (int k = 0; k < (int)gridDim.x; ++k) t1 += ((volatile double*)partial)[gridDim.x + k];
    sc->sum_rr = tot;
    sc->sum_r = t1;
    sc->rho = rz;
    if (!ok) sc->flags |= 1;
  }
}

// null-space projection r -= mean_active(r), mean over all parts; ||r||^2
__global__ __launch_bounds__(256) void k_project(float* __restrict__ r, const uint32_t* __restrict__ act, Ranges R,
                                                 double* partial,
                                                 unsigned* counter, Scalars* sc) {
  __shared__ double sred[8];
  const float m = (float)(sc->sum_r / sc->n_active);
  double s2 = 0.0, s1 = 0.0;
  FOR_RANGES(R, i) {
    float4 v = reinterpret_cast<float4*>(r)[i];
    float e[4] = {v.x, v.y, v.z, v.w};
    const unsigned am = act4(act, i);
    for (int k = 0; k < 4; ++k) {
      if ((am >> k) & 1u) e[k] -= m;
      s2 += (double)e[k] * e[k];
      s1 += (double)e[k];
    }
    reinterpret_cast<float4*>(r)[i] = make_float4(e[0], e[1], e[2], e[3]);
  }
  // ||r||^2 and the sum of the projected r (the next fused projection's starting mean)
  reduce2(s2, s1, partial, counter, sc, SF_RR, SF_R, sred);
}

// (r, z) (Alg. 1 line 12)
__global__ __launch_bounds__(256) void k_dot_rz(const float* __restrict__ r, const float* __restrict__ z, Ranges R,
                                                double* partial,
                                                unsigned* counter, Scalars* sc) {
  __shared__ double sred[8];
  double s = 0.0;
  FOR_RANGES(R, i) {
    float4 a = __ldg(reinterpret_cast<const float4*>(r) + i);
    float4 b = __ldg(reinterpret_cast<const float4*>(z) + i);
    s += (double)a.x * b.x + (double)a.y * b.y + (double)a.z * b.z + (double)a.w * b.w;
  }
  double bs = block_reduce_d(s, sred);
  double tot;
  if (last_block_sum(bs, partial, counter, gridDim.x, &tot, sred)) {
    sc->sum_rz = tot;
    sc->beta_f = (float)(tot / sc->rho);  // (multi-part jobs recompute it after the allreduce)
  }
}

// p = z + beta p_old in place (Alg. 1 line 13; beta = 0 on the first iteration), over the
// owned leaf cells.  z and p_old are zero on inactive cells, so p is too.
__global__ __launch_bounds__(256) void k_pupdate(const float* __restrict__ z, float* __restrict__ p, Ranges R,
                                                 const Scalars* sc, int use_beta) {
  const float beta = use_beta ? sc->beta_f : 0.0f;
  FOR_RANGES(R, i) {
    const float4 zv = __ldg(reinterpret_cast<const float4*>(z) + i);
    float4 pv = make_float4(0.f, 0.f, 0.f, 0.f);
    if (use_beta) pv = reinterpret_cast<const float4*>(p)[i];
    pv.x = fmaf(beta, pv.x, zv.x);
    pv.y = fmaf(beta, pv.y, zv.y);
    pv.z = fmaf(beta, pv.z, zv.z);
    pv.w = fmaf(beta, pv.w, zv.w);
    reinterpret_cast<float4*>(p)[i] = pv;
  }
}

// the stopping test of the device-side PCG loop (Alg. 1 line 8): records ||r_k|| / ||r_0||,
// and sets the while-node's condition to "continue" unless converged, broken down,
// non-finite or at max_iters
__global__ void k_pcg_check(Scalars* sc, LoopState* ls, cudaGraphConditionalHandle h) {
  const double rr = sc->sum_rr;
  const int k = ++ls->k;
  const double rel = sqrt(rr) / ls->bn;
  if (k - 1 < LOOP_HCAP) ls->hist[k - 1] = rel;
  ls->rel = rel;
  int st = 0;
  if (sc->flags & 1) st = 9;
  else if (!isfinite(rr)) st = 8;
  const bool conv = st == 0 && rel <= ls->rtol;
  if (!conv && st == 0 && k >= ls->max_iters) st = 10;
  ls->status = st;
  ls->converged = conv ? 1 : 0;
  cudaGraphSetConditional(h, (conv || st) ? 0u : 1u);
}

__global__ void k_set_beta(Scalars* sc) { sc->beta_f = (float)(sc->sum_rz / sc->rho); }

__global__ void k_copy_ranges(const float* src, float* dst, Ranges R) {
  FOR_RANGES(R, i) reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
}

// dst (slot order) = src (caller's natural order) on the active cells, 0 elsewhere
__global__ void k_mask_copy(const float* src, const uint32_t* act, float* dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = ((act[i >> 5] >> (i & 31)) & 1u) ? src[(i & ~(int64_t)511) + slot_nat((int)(i & 511))] : 0.0f;
}

// dst (caller's natural order) = src (slot order) on the cells of the ranges: per natural row,
// the red and black colour rows interleaved into two 128-bit stores
__global__ void k_copy_to_nat(const float* src, float* dst, Ranges R) {
  FOR_ROWS(R, c0) {
    const int64_t tb = c0 & ~(int64_t)511;
    const int row = (int)((c0 & 511) >> 3), y = row & 7, z = row >> 3, p = (y + z) & 1;
    const float4 vr = reinterpret_cast<const float4*>(src)[(tb + 4 * row) >> 2];
    const float4 vb = reinterpret_cast<const float4*>(src)[(tb + 256 + 4 * row) >> 2];
    // natural x = 2m + p holds red m, 2m + 1 - p black m
    const float4 a = p ? make_float4(vb.x, vr.x, vb.y, vr.y) : make_float4(vr.x, vb.x, vr.y, vb.y);
    const float4 c = p ? make_float4(vb.z, vr.z, vb.w, vr.w) : make_float4(vr.z, vb.z, vr.w, vb.w);
    *reinterpret_cast<float4*>(dst + c0) = a;
    *reinterpret_cast<float4*>(dst + c0 + 4) = c;
  }
}

// per-cell arrays of nf fields (field stride n) between natural and slot order
template <class T>
__global__ void k_permute(const T* src, T* dst, int64_t n, int nf, int to_slots) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = (i & ~(int64_t)511) + slot_nat((int)(i & 511));
    for (int f = 0; f < nf; ++f) {
      if (to_slots) dst[(size_t)f * n + i] = src[(size_t)f * n + j];
      else dst[(size_t)f * n + j] = src[(size_t)f * n + i];
    }
  }
}

// activity bitmask of the leaf cells (bit i%32 of word i/32: c_i != 0)
__global__ void k_build_mask(const float* coef, int64_t nwords, uint32_t* act) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < nwords; w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t m = 0;
    for (int k = 0; k < 32; ++k) m |= (coef[cidx(32 * w + k, 0)] != 0.0f ? 1u : 0u) << k;
    act[w] = m;
  }
}

}  // namespace

// (r, z) from the fused last pass's partials (2 per tile) and beta = (r, z) / rho
__global__ __launch_bounds__(1024) void k_finish_rz(const double* partial, int n, Scalars* sc) {
  __shared__ double sred[32];
  const int bd = blockDim.x;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int k = threadIdx.x;
  for (; k + 3 * bd < n; k += 4 * bd) {
    s0 += partial[k];
    s1 += partial[k + bd];
    s2 += partial[k + 2 * bd];
    s3 += partial[k + 3 * bd];
  }
  for (; k < n; k += bd) s0 += partial[k];
  double s = (s0 + s1) + (s2 + s3);
  for (int o = 16; o; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += sred[w];
    sc->sum_rz = tot;
    sc->beta_f = (float)(tot / sc->rho);  // (multi-part jobs recompute it after the allreduce)
  }
}

void launch_rz_finish(const double* partial, int64_t n, double* scratch, Scalars* sc, cudaStream_t s) {
  const int G = (int)std::min<int64_t>(296, (n + 4095) / 4096);
  const int64_t chunk = (n + G - 1) / G;
  k_chunk_sums<<<G, 256, 0, s>>>(partial, n, chunk, scratch);
  k_finish_rz<<<1, 1024, 0, s>>>(scratch, G, sc);
}

void launch_apply(const ApplyArgs& a, cudaStream_t s) {
  if (a.n_ifaces > 0) k_inner_face_means<<<a.n_ifaces, 64, 0, s>>>(a.ifaces, a.child, a.coef, a.z, a.pbar, a.NL);
  if (a.ntiles == 0) {
    if (a.partial) cudaMemsetAsync(&a.sc->sum_pq, 0, sizeof(double), s);
    return;
  }
  // the irregular (T-junction) body inlined at 6 CTAs/SM (80 registers) on trees with
  // T-junction tiles; out of line at 8 CTAs/SM otherwise (its call frame spills to local
  // memory: 100M L2 sectors of local traffic per config-3 apply under ncu, config 5 apply
  // 45.2 -> 38.6 ms per solve inlined); OCTMG_APPLY_IRR=inline / call forces one form
  int env = -2;  // (read per call: the variant tests switch it within one process)
  if (env == -2) {
    const char* e = getenv("OCTMG_APPLY_IRR");
    env = !e ? -1 : (e[0] == 'i' ? 1 : 0);
  }
  const bool inl = env >= 0 ? env == 1 : a.irr_inline != 0;
  // trees without T-junction tiles, inner neighbours of leaf tiles or row sums: the lean body
  // (no pbar select, no row-sum load, no out-of-line call frame; 62 registers: config 2
  // apply 0.76 -> 0.67 ms per solve)
  const char* le = getenv("OCTMG_APPLY_LEAN");  // 0: the general body everywhere
  const bool lean = !inl && !a.irr_inline && a.n_ifaces == 0 && a.lean && !(le && le[0] == '0');
  if (a.partial) {
    if (inl) k_apply_v6<true, true><<<a.ntiles, 128, 0, s>>>(a);
    else if (lean) k_apply_v6<true, false, true><<<a.ntiles, 128, 0, s>>>(a);
    else k_apply_v6<true, false><<<a.ntiles, 128, 0, s>>>(a);
    // 4 warp partials per tile of p.q, then of sum q; summed in two fixed-order stages
    const int64_t n = 4 * (int64_t)a.ntiles;
    const int G = (int)std::min<int64_t>(296, (n + 4095) / 4096);
    const int64_t chunk = (n + G - 1) / G;
    const int ny = a.sumq ? 2 : 1;
    k_chunk_sums<<<dim3(G, ny), 256, 0, s>>>(a.partial, n, chunk, a.partial + 2 * n);
    k_finish_sigma<<<ny, 1024, 0, s>>>(a.partial + 2 * n, G, a.sc);
  } else {
    if (inl) k_apply_v6<false, true><<<a.ntiles, 128, 0, s>>>(a);
    else if (lean) k_apply_v6<false, false, true><<<a.ntiles, 128, 0, s>>>(a);
    else k_apply_v6<false, false><<<a.ntiles, 128, 0, s>>>(a);
  }
}

void launch_init(const float* b, const uint32_t* act, float* r, float* x, const Ranges& R, double* partial,
                 unsigned* counter, Scalars* sc, cudaStream_t s, int grid) {
  k_init<<<grid, 256, 0, s>>>(b, act, r, x, R, partial, counter, sc);
}
void launch_update(float* x, float* r, const float* p, const float* q, const Ranges& R, double* partial,
                   unsigned* counter, Scalars* sc, cudaStream_t s, int grid, float alpha_fixed,
                   const uint32_t* act_proj) {
  k_update<<<grid, 256, 0, s>>>(x, r, p, q, R, partial, counter, sc, alpha_fixed, act_proj);
}
void launch_project(float* r, const uint32_t* act, const Ranges& R, double* partial, unsigned* counter, Scalars* sc,
                    cudaStream_t s, int grid) {
  k_project<<<grid, 256, 0, s>>>(r, act, R, partial, counter, sc);
}
void launch_dot_rz(const float* r, const float* z, const Ranges& R, double* partial, unsigned* counter, Scalars* sc,
                   cudaStream_t s, int grid) {
  k_dot_rz<<<grid, 256, 0, s>>>(r, z, R, partial, counter, sc);
}
__global__ void k_set_rho_inf(Scalars* sc) { sc->rho = INFINITY; }
__global__ void k_copy_words(const unsigned* src, unsigned* dst, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = src[i];
}
void launch_set_rho_inf(Scalars* sc, cudaStream_t s) { k_set_rho_inf<<<1, 1, 0, s>>>(sc); }
void launch_copy_words(const void* src, void* dst, size_t nbytes, cudaStream_t s) {
  k_copy_words<<<1, 256, 0, s>>>((const unsigned*)src, (unsigned*)dst, (int)(nbytes / 4));
}
void launch_set_beta(Scalars* sc, cudaStream_t s) { k_set_beta<<<1, 1, 0, s>>>(sc); }
void launch_pcg_check(Scalars* sc, LoopState* ls, unsigned long long handle, cudaStream_t s) {
  k_pcg_check<<<1, 1, 0, s>>>(sc, ls, (cudaGraphConditionalHandle)handle);
}
void launch_pupdate(const float* z, float* p, const Ranges& R, const Scalars* sc, bool use_beta, cudaStream_t s,
                    int grid) {
  k_pupdate<<<grid, 256, 0, s>>>(z, p, R, sc, use_beta ? 1 : 0);
}

void launch_copy_ranges(const float* src, float* dst, const Ranges& R, cudaStream_t s) {
  k_copy_ranges<<<592, 256, 0, s>>>(src, dst, R);
}
void launch_copy_to_nat(const float* src, float* dst, const Ranges& R, cudaStream_t s) {
  k_copy_to_nat<<<592, 256, 0, s>>>(src, dst, R);
}
void launch_permute_f32(const float* src, float* dst, int64_t n, int nf, bool to_slots, cudaStream_t s) {
  k_permute<float><<<592, 256, 0, s>>>(src, dst, n, nf, to_slots ? 1 : 0);
}
void launch_permute_u8(const uint8_t* src, uint8_t* dst, int64_t n, bool to_slots, cudaStream_t s) {
  k_permute<uint8_t><<<592, 256, 0, s>>>(src, dst, n, 1, to_slots ? 1 : 0);
}
void launch_mask_copy(const float* src, const uint32_t* act, float* dst, int64_t n, cudaStream_t s) {
  k_mask_copy<<<592, 256, 0, s>>>(src, act, dst, n);
}
void launch_build_mask(const float* coef, int64_t n, uint32_t* act, cudaStream_t s) {
  k_build_mask<<<592, 256, 0, s>>>(coef, n / 32, act);
}

}  // namespace octmg
