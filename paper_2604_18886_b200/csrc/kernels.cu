// Hot-path kernels (sm_100a).  One CTA per 8^3 tile: the tile's values are
// staged in shared memory with a one-cell halo ("10x10x10 working region");
// ghost values are reconstructed on the fly at halo load (Eq. 12);
// coefficient records are float4 (c, c_x-, c_y-, c_z-) read with 128-bit loads and the
// +face coefficients come from the neighbour record or the ghost layer.
#include "octmg_internal.cuh"

namespace octmg {

namespace {

constexpr int NT = 256;  // threads per tile CTA; thread -> cells (2*x2, y, z), (2*x2+1, y, z)

__device__ __forceinline__ int su_idx(int x, int y, int z) { return (z + 1) * 100 + (y + 1) * 10 + (x + 1); }
__device__ __forceinline__ int scx_idx(int x, int y, int z) { return (z * 8 + y) * 9 + x; }   // x in 0..8
__device__ __forceinline__ int scy_idx(int x, int y, int z) { return (z * 9 + y) * 8 + x; }   // y in 0..8
__device__ __forceinline__ int scz_idx(int x, int y, int z) { return (z * 8 + y) * 8 + x; }   // z in 0..8
__device__ __forceinline__ int loff(int x, int y, int z) { return x + 8 * y + 64 * z; }
__device__ __forceinline__ float comp(const float4& v, int a) { return a == 0 ? v.y : (a == 1 ? v.z : v.w); }

struct TileSmem {
  float u[1000];
  float cx[576];
  float cy[576];
  float cz[576];
  float c[512];
  int nb[6];
  int4 tv;
  int4 ntv[6];     // neighbour tile coords (prolongation parity)
  int npar[6];     // neighbour tile parents
  int par;
};

// own boundary cell adjacent to halo item (f, p, q) and the source cell in the neighbour
__device__ __forceinline__ void face_cells(int f, int p, int q, int own[3], int src[3], int halo[3]) {
  int a = f >> 1, s = f & 1;
  int o[3];
  if (a == 0) { o[0] = s ? 7 : 0; o[1] = p; o[2] = q; }
  else if (a == 1) { o[0] = p; o[1] = s ? 7 : 0; o[2] = q; }
  else { o[0] = p; o[1] = q; o[2] = s ? 7 : 0; }
  for (int k = 0; k < 3; ++k) { own[k] = o[k]; src[k] = o[k]; halo[k] = o[k]; }
  src[a] = s ? 0 : 7;
  halo[a] = s ? 8 : -1;
}

// mean of the active cells of the 2x2x2 block (parent's children) holding own cell o
__device__ __forceinline__ float block_mean(const TileSmem& S, const int o[3]) {
  int bx = o[0] & ~1, by = o[1] & ~1, bz = o[2] & ~1;
  float s = 0.0f;
  int n = 0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        int off = loff(bx + dx, by + dy, bz + dz);
        if (S.c[off] != 0.0f) { s += S.u[su_idx(bx + dx, by + dy, bz + dz)]; n++; }
      }
  return n ? s / (float)n : 0.0f;
}

__device__ __forceinline__ void set_plus_coef(TileSmem& S, int a, const int halo[3], float v) {
  if (a == 0) S.cx[scx_idx(8, halo[1], halo[2])] = v;
  else if (a == 1) S.cy[scy_idx(halo[0], 8, halo[2])] = v;
  else S.cz[scz_idx(halo[0], halo[1], 8)] = v;
}

__device__ __forceinline__ float rowsum(const TileSmem& S, int x, int y, int z, float c) {
  // c*u first, then faces x-, x+, y-, y+, z-, z+ (the oracle's order)
  int iu = su_idx(x, y, z);
  float s = c * S.u[iu];
  s = fmaf(S.cx[scx_idx(x, y, z)], S.u[iu - 1], s);
  s = fmaf(S.cx[scx_idx(x + 1, y, z)], S.u[iu + 1], s);
  s = fmaf(S.cy[scy_idx(x, y, z)], S.u[iu - 10], s);
  s = fmaf(S.cy[scy_idx(x, y + 1, z)], S.u[iu + 10], s);
  s = fmaf(S.cz[scz_idx(x, y, z)], S.u[iu - 100], s);
  s = fmaf(S.cz[scz_idx(x, y, z + 1)], S.u[iu + 100], s);
  return s;
}


// ------------------------------------------------------------------------------------
// Composite operator (PCG q = A p with p = z + beta p fused, and the p.q dot)
// ------------------------------------------------------------------------------------
__device__ __forceinline__ float dir_val(const ApplyArgs& a, float beta, size_t i) {
  float v = a.z[i];
  if (a.pold) v = fmaf(beta, a.pold[i], v);
  return v;
}

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

template <bool DOT>
__global__ __launch_bounds__(NT) void k_apply(ApplyArgs a) {
  __shared__ TileSmem S;
  __shared__ double sred[NT / 32];
  const int t = blockIdx.x;
  const int tid = threadIdx.x;
  const float beta = (a.use_beta && a.pold) ? (float)a.sc->beta : 0.0f;
  if (tid < 6) S.nb[tid] = a.nbr[6 * t + tid];
  if (tid == 6) S.tv = a.tile[t];
  const int x2 = tid & 3, y = (tid >> 2) & 7, z = tid >> 5, x0 = 2 * x2;
  const int off0 = loff(x0, y, z);
  const size_t base = (size_t)t * TB3;
  float4 q0 = a.coef[base + off0], q1 = a.coef[base + off0 + 1];
  float p0v, p1v;
  {
    float2 zz = *reinterpret_cast<const float2*>(a.z + base + off0);
    p0v = zz.x; p1v = zz.y;
    if (a.pold) {
      float2 pp = *reinterpret_cast<const float2*>(a.pold + base + off0);
      p0v = fmaf(beta, pp.x, p0v);
      p1v = fmaf(beta, pp.y, p1v);
    }
    if (q0.x == 0.0f) p0v = 0.0f;
    if (q1.x == 0.0f) p1v = 0.0f;
  }
  if (a.pnew) *reinterpret_cast<float2*>(a.pnew + base + off0) = make_float2(p0v, p1v);
  S.u[su_idx(x0, y, z)] = p0v;
  S.u[su_idx(x0 + 1, y, z)] = p1v;
  S.c[off0] = q0.x;
  S.c[off0 + 1] = q1.x;
  S.cx[scx_idx(x0, y, z)] = q0.y;
  S.cx[scx_idx(x0 + 1, y, z)] = q1.y;
  S.cy[scy_idx(x0, y, z)] = q0.z;
  S.cy[scy_idx(x0 + 1, y, z)] = q1.z;
  S.cz[scz_idx(x0, y, z)] = q0.w;
  S.cz[scz_idx(x0 + 1, y, z)] = q1.w;
  __syncthreads();
  for (int w = tid; w < 384; w += NT) {
    int f = w >> 6, p = w & 7, q = (w >> 3) & 7;
    int own[3], src[3], halo[3];
    face_cells(f, p, q, own, src, halo);
    int ax = f >> 1;
    int n = S.nb[f];
    float v = 0.0f, cplus = 0.0f;
    if (n >= 0) {
      int so = loff(src[0], src[1], src[2]);
      float4 r = a.coef[(size_t)n * TB3 + so];
      cplus = comp(r, ax);
      if (n < a.NL) {
        if (r.x != 0.0f) v = dir_val(a, beta, (size_t)n * TB3 + so);
      } else {
        // inner same-level neighbour: mean of its active children (all leaves)
        int ct = a.child[8 * (n - a.NL) + (src[0] >> 2) + 2 * (src[1] >> 2) + 4 * (src[2] >> 2)];
        float s = 0.0f;
        int k = 0;
        for (int dz = 0; dz < 2; ++dz)
          for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
              size_t ci = (size_t)ct * TB3 +
                          loff((2 * src[0] + dx) & 7, (2 * src[1] + dy) & 7, (2 * src[2] + dz) & 7);
              if (a.coef[ci].x != 0.0f) { s += dir_val(a, beta, ci); k++; }
            }
        v = k ? s / (float)k : 0.0f;
      }
    } else if (n <= -2) {
      int C = -2 - n;
      int g0 = S.tv.y * 8 + halo[0], g1 = S.tv.z * 8 + halo[1], g2 = S.tv.w * 8 + halo[2];
      size_t ci = (size_t)C * TB3 + loff((g0 >> 1) & 7, (g1 >> 1) & 7, (g2 >> 1) & 7);
      if (a.coef[ci].x != 0.0f) {
        float pc = dir_val(a, beta, ci);
        v = S.u[su_idx(own[0], own[1], own[2])] + 0.5f * (pc - block_mean(S, own));
      }
      if (f & 1) cplus = a.glayer_val[(size_t)a.glayer[3 * t + ax] * 64 + p + 8 * q];
    }
    S.u[su_idx(halo[0], halo[1], halo[2])] = v;
    if (f & 1) set_plus_coef(S, ax, halo, cplus);
  }
  __syncthreads();
  float r0 = q0.x != 0.0f ? rowsum(S, x0, y, z, q0.x) : 0.0f;
  float r1 = q1.x != 0.0f ? rowsum(S, x0 + 1, y, z, q1.x) : 0.0f;
  *reinterpret_cast<float2*>(a.q + base + off0) = make_float2(r0, r1);
  if (DOT) {
    double d = (double)p0v * (double)r0 + (double)p1v * (double)r1;
    double tot;
    double bs = block_reduce_d(d, sred);
    if (last_block_sum(bs, a.partial, a.counter, gridDim.x, &tot, sred)) {
      Scalars* sc = a.sc;
      sc->sigma = tot;
      if (!(tot > 0.0) || !isfinite(tot)) { sc->flags |= 1; sc->alpha = 0.0; }
      else sc->alpha = sc->rho / tot;
    }
  }
}

// ------------------------------------------------------------------------------------
// PCG vector kernels (grid-stride over float4, fixed grid => deterministic partials)
// ------------------------------------------------------------------------------------
__device__ __forceinline__ bool active_of(const float4* coef, int64_t i) { return coef[i].x != 0.0f; }

__global__ __launch_bounds__(256) void k_init(const float* b, const float4* coef, float* r, float* x, int64_t n4,
                                              double* partial, unsigned* counter, Scalars* sc) {
  __shared__ double sred[8];
  double s2 = 0.0, s1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = reinterpret_cast<const float4*>(b)[i];
    float m[4] = {v.x, v.y, v.z, v.w};
    for (int k = 0; k < 4; ++k) {
      if (!active_of(coef, 4 * i + k)) m[k] = 0.0f;
      s2 += (double)m[k] * m[k];
      s1 += (double)m[k];
    }
    reinterpret_cast<float4*>(r)[i] = make_float4(m[0], m[1], m[2], m[3]);
    reinterpret_cast<float4*>(x)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  double b2 = block_reduce_d(s2, sred);
  __syncthreads();
  double b1 = block_reduce_d(s1, sred);
  double tot;
  // two sums: partial layout [0, grid) = s2, [grid, 2 grid) = s1
  if (threadIdx.x == 0) partial[gridDim.x + blockIdx.x] = b1;
  if (last_block_sum(b2, partial, counter, gridDim.x, &tot, sred)) {
    double t1 = 0.0;
    for (int k = 0; k < (int)gridDim.x; ++k) t1 += ((volatile double*)partial)[gridDim.x + k];
    sc->rr = tot;
    sc->rsum = t1;
    sc->flags = isfinite(tot) ? 0 : 2;
  }
}

__global__ __launch_bounds__(256) void k_update(float* x, float* r, const float* p, const float* q, int64_t n4,
                                                double* partial, unsigned* counter, Scalars* sc) {
  __shared__ double sred[8];
  const float alpha = (sc->flags & 1) ? 0.0f : (float)sc->alpha;
  double s2 = 0.0, s1 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 xv = reinterpret_cast<float4*>(x)[i];
    float4 rv = reinterpret_cast<float4*>(r)[i];
    float4 pv = reinterpret_cast<const float4*>(p)[i];
    float4 qv = reinterpret_cast<const float4*>(q)[i];
    xv.x = fmaf(alpha, pv.x, xv.x); xv.y = fmaf(alpha, pv.y, xv.y);
    xv.z = fmaf(alpha, pv.z, xv.z); xv.w = fmaf(alpha, pv.w, xv.w);
    rv.x = fmaf(-alpha, qv.x, rv.x); rv.y = fmaf(-alpha, qv.y, rv.y);
    rv.z = fmaf(-alpha, qv.z, rv.z); rv.w = fmaf(-alpha, qv.w, rv.w);
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
    sc->rr = tot;
    sc->rsum = t1;
    if (!isfinite(tot)) sc->flags |= 2;
  }
}

// null-space projection r -= mean_active(r), recomputes ||r||^2
__global__ __launch_bounds__(256) void k_project(float* r, const float4* coef, int64_t n4, double* partial,
                                                 unsigned* counter, Scalars* sc) {
  __shared__ double sred[8];
  const float m = (float)(sc->rsum / sc->n_active);
  double s2 = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = reinterpret_cast<float4*>(r)[i];
    float e[4] = {v.x, v.y, v.z, v.w};
    for (int k = 0; k < 4; ++k) {
      if (active_of(coef, 4 * i + k)) e[k] -= m;
      s2 += (double)e[k] * e[k];
    }
    reinterpret_cast<float4*>(r)[i] = make_float4(e[0], e[1], e[2], e[3]);
  }
  double b2 = block_reduce_d(s2, sred);
  double tot;
  if (last_block_sum(b2, partial, counter, gridDim.x, &tot, sred)) {
    sc->rr = tot;
    sc->mean = m;
  }
}

__global__ __launch_bounds__(256) void k_dot_rz(const float* r, const float* z, int64_t n4, double* partial,
                                                unsigned* counter, Scalars* sc, int first) {
  __shared__ double sred[8];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 a = reinterpret_cast<const float4*>(r)[i];
    float4 b = reinterpret_cast<const float4*>(z)[i];
    s += (double)a.x * b.x + (double)a.y * b.y + (double)a.z * b.z + (double)a.w * b.w;
  }
  double bs = block_reduce_d(s, sred);
  double tot;
  if (last_block_sum(bs, partial, counter, gridDim.x, &tot, sred)) {
    if (first) { sc->beta = 0.0; }
    else sc->beta = tot / sc->rho;
    sc->rho = tot;
    if (!isfinite(tot)) sc->flags |= 2;
  }
}

__global__ void k_mask_copy(const float* src, const float4* coef, float* dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = coef[i].x != 0.0f ? src[i] : 0.0f;
}

}  // namespace

void launch_apply(const ApplyArgs& a, cudaStream_t s) {
  if (a.NL == 0) return;
  if (a.partial) k_apply<true><<<a.NL, NT, 0, s>>>(a);
  else k_apply<false><<<a.NL, NT, 0, s>>>(a);
}

void launch_init(const float* b, const float4* coef, float* r, float* x, int64_t n, double* partial,
                 unsigned* counter, Scalars* sc, cudaStream_t s, int grid) {
  k_init<<<grid, 256, 0, s>>>(b, coef, r, x, n / 4, partial, counter, sc);
}
void launch_update(float* x, float* r, const float* p, const float* q, int64_t n, double* partial,
                   unsigned* counter, Scalars* sc, cudaStream_t s, int grid) {
  k_update<<<grid, 256, 0, s>>>(x, r, p, q, n / 4, partial, counter, sc);
}
void launch_project(float* r, const float4* coef, int64_t n, double* partial, unsigned* counter, Scalars* sc,
                    cudaStream_t s, int grid) {
  k_project<<<grid, 256, 0, s>>>(r, coef, n / 4, partial, counter, sc);
}
void launch_dot_rz(const float* r, const float* z, int64_t n, double* partial, unsigned* counter, Scalars* sc,
                   int first, cudaStream_t s, int grid) {
  k_dot_rz<<<grid, 256, 0, s>>>(r, z, n / 4, partial, counter, sc, first);
}
void launch_mask_copy(const float* src, const float4* coef, float* dst, int64_t n, cudaStream_t s) {
  k_mask_copy<<<592, 256, 0, s>>>(src, coef, dst, n);
}

}  // namespace octmg
