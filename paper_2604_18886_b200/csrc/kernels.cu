// PCG kernels (sm_100a): the composite operator fused with p = z + beta p and the fp64 p.q
// reduction, and the vector updates / dots.  One CTA per 8^3 tile for the operator; the
// stencil is gathered directly through L1/L2 (see direct.cu); coefficient records are
// float4 (c, c_x-, c_y-, c_z-) and the +face coefficient comes from the neighbour record or
// the ghost layer.
#include "octmg_internal.cuh"
#include "rowstencil.cuh"

namespace octmg {

namespace {

constexpr int NT = 256;  // threads per tile CTA; thread -> cells (2*x2, y, z), (2*x2+1, y, z)

__device__ __forceinline__ int loff(int x, int y, int z) { return cslot(x, y, z); }  // slot order
__device__ __forceinline__ float comp(const float4& v, int a) { return a == 0 ? v.y : (a == 1 ? v.z : v.w); }


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

// direction value p = z + beta p_old of cell i; z and p_old are zero on inactive cells (the
// cycle never writes them, octmg_apply masks its input first), so no activity test
__device__ __forceinline__ float pval(const ApplyArgs& a, float beta, size_t i) {
  float v = __ldg(a.z + i);
  if (a.pold) v = fmaf(beta, __ldg(a.pold + i), v);
  return v;
}

// Composite operator row: same-level leaf neighbours give their value, a
// same-level inner neighbour the mean of its active children (all leaves), a ghost
// g = p_i + (p_C - m_P)/2 (Eq. 12), walls 0.  Face order x-, x+, y-, y+, z-, z+.
__device__ __forceinline__ float composite_faces(const ApplyArgs& a, float beta, int t, int x, int y, int z,
                                                 const float4& q, float pi, float mP, float s0, const float* sp,
                                                 const float (*scm)[TB3]) {
  const int c[3] = {x, y, z};
  float s = s0;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1, sg = (f & 1) ? 1 : -1;
    int nc[3] = {c[0], c[1], c[2]};
    nc[ax] += sg;
    float v = 0.0f, cf = (f & 1) ? 0.0f : comp(q, ax);
    if (nc[ax] >= 0 && nc[ax] < 8) {
      const int no = loff(nc[0], nc[1], nc[2]);
      if (f & 1) cf = scm[ax][no];  // this tile's -face coefficients, staged (SoA)
      v = sp[no];                   // this tile's p, staged in shared memory
    } else {
      const int n = __ldg(a.nbr + 6 * t + f);
      nc[ax] &= 7;
      const int no = loff(nc[0], nc[1], nc[2]);
      if (n >= 0) {
        if (f & 1) cf = comp(ldcoef(a.coef, (size_t)n * TB3 + no), ax);
        if (n < a.NL) {
          v = pval(a, beta, (size_t)n * TB3 + no);
        } else {
          const int ct = __ldg(a.child + 8 * (n - a.NL) + (nc[0] >> 2) + 2 * (nc[1] >> 2) + 4 * (nc[2] >> 2));
          // the 8 children: activity and value loaded together (no load behind a branch)
          float sm = 0.0f;
          int k = 0;
#pragma unroll
          for (int d = 0; d < 8; ++d) {
            const size_t ci = (size_t)ct * TB3 + loff((2 * nc[0] + (d & 1)) & 7, (2 * nc[1] + ((d >> 1) & 1)) & 7,
                                                      (2 * nc[2] + (d >> 2)) & 7);
            const float cc = __ldg(a.coef + cidx(ci, 0));
            const float pv = pval(a, beta, ci);
            if (cc != 0.0f) { sm += pv; k++; }
          }
          v = k ? sm / (float)k : 0.0f;
        }
      } else if (n <= -2) {
        if (f & 1)
          cf = __ldg(a.glayer_val + (size_t)__ldg(a.glayer + 3 * t + ax) * 64 +
                     (ax == 0 ? y + 8 * z : (ax == 1 ? x + 8 * z : x + 8 * y)));
        const int C = -2 - n;
        const int4 tv = __ldg(a.tile + t);
        int g[3] = {tv.y * 8 + c[0], tv.z * 8 + c[1], tv.w * 8 + c[2]};
        g[ax] += sg;
        const size_t ci = (size_t)C * TB3 + loff((g[0] >> 1) & 7, (g[1] >> 1) & 7, (g[2] >> 1) & 7);
        const float cC = __ldg(a.coef + cidx(ci, 0));
        const float pC = pval(a, beta, ci);
        if (cC != 0.0f) v = pi + 0.5f * (pC - mP);
      }
    }
    s = fmaf(cf, v, s);
  }
  return s;
}

// q = A p with p = z + beta p_old formed on the fly (and stored), plus the fp64 partial of
// p.q with a deterministic last-block reduction that sets sigma and alpha = rho / sigma
// (Alg. 1 lines 9-10; fp64 dots P:L1233).  Thread layout as the restriction: the
// four lanes of a 2x2x2 block are xor 4 / xor 8 apart (ghost m_P by shuffles).
template <bool DOT>
__device__ __forceinline__ void apply_general(const ApplyArgs& a, int t, double* sred) {
  const int j = threadIdx.x;
  const int x2 = j & 3;
  const int y = ((j >> 2) & 1) | (((j >> 4) & 3) << 1);
  const int z = ((j >> 3) & 1) | ((j >> 6) << 1);
  const int x0 = 2 * x2;
  // beta = (r_k, z_k) / (r_{k-1}, z_{k-1}) (Alg. 1 line 12)
  const float beta = (a.use_beta && a.pold) ? a.sc->beta_f : 0.0f;  // Alg. 1 line 12
  const size_t base = (size_t)t * TB3;
  const int off0 = loff(x0, y, z), off1 = off0 ^ 256;  // the pair: same q, opposite colours
  const float4 q0 = ldcoef(a.coef, base + off0), q1 = ldcoef(a.coef, base + off1);
  float p0 = 0.0f, p1 = 0.0f;
  {
    p0 = __ldg(a.z + base + off0);
    p1 = __ldg(a.z + base + off1);
    if (a.pold) {
      p0 = fmaf(beta, __ldg(a.pold + base + off0), p0);
      p1 = fmaf(beta, __ldg(a.pold + base + off1), p1);
    }
    if (q0.x == 0.0f) p0 = 0.0f;
    if (q1.x == 0.0f) p1 = 0.0f;
  }
  if (a.pnew) {
    a.pnew[base + off0] = p0;
    a.pnew[base + off1] = p1;
  }
  __shared__ float sp[TB3];
  __shared__ float scm[3][TB3];
  sp[off0] = p0;
  sp[off1] = p1;
  scm[0][off0] = q0.y; scm[1][off0] = q0.z; scm[2][off0] = q0.w;
  scm[0][off1] = q1.y; scm[1][off1] = q1.z; scm[2][off1] = q1.w;
  float su = p0 + p1;
  int na = (q0.x != 0.0f) + (q1.x != 0.0f);
  su += __shfl_xor_sync(0xffffffffu, su, 4);
  na += __shfl_xor_sync(0xffffffffu, na, 4);
  su += __shfl_xor_sync(0xffffffffu, su, 8);
  na += __shfl_xor_sync(0xffffffffu, na, 8);
  const float mP = na ? su / (float)na : 0.0f;
  __syncthreads();
  const float r0 = q0.x != 0.0f ? composite_faces(a, beta, t, x0, y, z, q0, p0, mP, q0.x * p0, sp, scm) : 0.0f;
  const float r1 = q1.x != 0.0f ? composite_faces(a, beta, t, x0 + 1, y, z, q1, p1, mP, q1.x * p1, sp, scm) : 0.0f;
  a.q[base + off0] = r0;
  a.q[base + off1] = r1;
  if (DOT) {
    // per-tile fp64 partial; k_finish_sigma sums them in tile order (no per-CTA fence)
    double d = (double)p0 * (double)r0 + (double)p1 * (double)r1;
    double bs = block_reduce_d(d, sred);
    if (threadIdx.x == 0) a.partial[blockIdx.x] = bs;
  }
}

// q = A p as k_apply, on tiles whose six neighbours are all same-level leaves or walls (every
// tile of a uniform tree): no shared-memory staging and no branches on the stencil path —
// the neighbour entries are prefetched and the pair face sums are vectorised (row2_faces).
// Other tiles take the general composite path of k_apply.
template <bool DOT>
__global__ __launch_bounds__(NT, 6) void k_apply_v2(ApplyArgs a) {
  __shared__ double sred[NT / 32];
  const int t = a.tiles ? a.tiles[blockIdx.x] : (int)blockIdx.x;
  int nb[6];
  {
    const int2* np = reinterpret_cast<const int2*>(a.nbr + 6 * (size_t)t);
    const int2 n0 = __ldg(np), n1 = __ldg(np + 1), n2 = __ldg(np + 2);
    nb[0] = n0.x; nb[1] = n0.y; nb[2] = n1.x; nb[3] = n1.y; nb[4] = n2.x; nb[5] = n2.y;
  }
  bool regular = true;
#pragma unroll
  for (int f = 0; f < 6; ++f) regular &= nb[f] >= -1 && nb[f] < a.NL;
  if (!regular) {
    apply_general<DOT>(a, t, sred);
    return;
  }
  const int j = threadIdx.x;
  const int x2 = j & 3;
  const int y = ((j >> 2) & 1) | (((j >> 4) & 3) << 1);
  const int z = ((j >> 3) & 1) | ((j >> 6) << 1);
  const int x0 = 2 * x2;
  const float beta = (a.use_beta && a.pold) ? a.sc->beta_f : 0.0f;  // Alg. 1 line 12
  const size_t base = (size_t)t * TB3;
  const int off0 = loff(x0, y, z);
  const float* cb = a.coef + ((size_t)t << 11);
  const float2 c0 = ldpair(cb, off0), cxm = ldpair(cb + 512, off0), cym = ldpair(cb + 1024, off0),
               czm = ldpair(cb + 1536, off0);
  // p = z + beta p_old of any leaf cell (zero on inactive cells, see pval)
  const RowTiles rt = row_tiles(t, nb, y, z);
  DirVals vals;
  vals.beta = beta;
  vals.z = a.z;
  vals.po = a.pold;
#pragma unroll
  for (int f = 0; f < 6; ++f) vals.tf[f] = rt.tf[f];
  float2 pp = ldpair(a.z + base, off0);
  if (a.pold) {
    const float2 w = ldpair(a.pold + base, off0);
    pp.x = fmaf(beta, w.x, pp.x);
    pp.y = fmaf(beta, w.y, pp.y);
  }
  const float p0 = c0.x != 0.0f ? pp.x : 0.0f, p1 = c0.y != 0.0f ? pp.y : 0.0f;
  // same summation order as the general path: c*p, then the faces x-, x+, y-, y+, z-, z+
  const float2 f = row2_faces(vals, rt, x2, y, z, pp, cxm, cym, czm, make_float2(c0.x * p0, c0.y * p1),
                              a.coef + ((size_t)rt.tf[1] << 11) + 512, a.coef + ((size_t)rt.tf[3] << 11) + 1024,
                              a.coef + ((size_t)rt.tf[5] << 11) + 1536);
  const float r0 = c0.x != 0.0f ? f.x : 0.0f;
  const float r1 = c0.y != 0.0f ? f.y : 0.0f;
  if (a.pnew) {
    a.pnew[base + off0] = p0;
    a.pnew[base + (off0 ^ 256)] = p1;
  }
  a.q[base + off0] = r0;
  a.q[base + (off0 ^ 256)] = r1;
  if (DOT) {
    double d = (double)p0 * (double)r0 + (double)p1 * (double)r1;
    double bs = block_reduce_d(d, sred);
    if (threadIdx.x == 0) a.partial[blockIdx.x] = bs;
  }
}

// q = A p for a precomputed p (split PCG form: a.z = p, no p_old), tiles without a ghost face
// or inner neighbour: thread j < 128 owns red cells j, j + 128 of the tile, thread j >= 128
// the black ones — the colour-pass layout: every neighbour of a cell is in the other colour
// half at a fixed slot offset (see face_sum_regular in direct.cu), one load per neighbour.
// Other tiles take the general composite path (same 256-thread CTA).
template <bool DOT>
__global__ __launch_bounds__(NT, 6) void k_apply_v4(ApplyArgs a) {
  __shared__ double sred[NT / 32];
  const int t = a.tiles ? a.tiles[blockIdx.x] : (int)blockIdx.x;
  int nb[6];
#pragma unroll
  for (int f = 0; f < 6; ++f) nb[f] = __ldg(a.nbr + 6 * (size_t)t + f);
  bool regular = true;
#pragma unroll
  for (int f = 0; f < 6; ++f) regular &= nb[f] >= -1 && nb[f] < a.NL;
  if (!regular) {
    apply_general<DOT>(a, t, sred);
    return;
  }
  const int j = threadIdx.x;
  const int colour = j >> 7, jj = j & 127;
  const int y = (jj >> 2) & 7, z0 = jj >> 5;
  const float* pt = a.z + ((size_t)t << 9);
  const float* ct = a.coef + ((size_t)t << 11);
  const float* pn[6];
  const float* cn[3];
#pragma unroll
  for (int f = 0; f < 6; ++f) pn[f] = nb[f] >= 0 ? a.z + ((size_t)nb[f] << 9) : pt;
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const int n = nb[2 * ax + 1];
    cn[ax] = (n >= 0 ? a.coef + ((size_t)n << 11) : ct) + ((1 + ax) << 9);
  }
  double d = 0.0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int z = z0 + 4 * k;
    const int x = 2 * (jj & 3) + ((colour + y + z) & 1);
    const int sl = (colour << 8) + jj + 128 * k;
    const float c0 = __ldg(ct + sl), cxm = __ldg(ct + 512 + sl), cym = __ldg(ct + 1024 + sl),
                czm = __ldg(ct + 1536 + sl);
    const float pc = __ldg(pt + sl);
    const int base = sl ^ 256;
    const int p = x & 1;
    const bool in[6] = {x > 0, x < 7, y > 0, y < 7, z > 0, z < 7};
    const int dlt[6] = {in[0] ? p - 1 : 3, in[1] ? p : -3, in[2] ? -4 : 28, in[3] ? 4 : -28, in[4] ? -32 : 224,
                        in[5] ? 32 : -224};
    const float cm3[3] = {cxm, cym, czm};
    const float pv = c0 != 0.0f ? pc : 0.0f;
    float sm = c0 * pv;  // the general path's order: c*p, then x-, x+, y-, y+, z-, z+
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int ax = f >> 1;
      const int no = base + dlt[f];
      float v = __ldg((in[f] ? pt : pn[f]) + no);
      const float cf = (f & 1) ? __ldg((in[f] ? ct + ((1 + ax) << 9) : cn[ax]) + no) : cm3[ax];
      if (!in[f] && nb[f] < 0) v = 0.0f;
      sm = fmaf(cf, v, sm);
    }
    const float r = c0 != 0.0f ? sm : 0.0f;
    a.q[((size_t)t << 9) + sl] = r;
    d += (double)pv * (double)r;
  }
  if (DOT) {
    double bs = block_reduce_d(d, sred);
    if (threadIdx.x == 0) a.partial[blockIdx.x] = bs;
  }
}

// k_apply_v4 with vector loads: thread j owns the two colour cells of slots 2jj, 2jj + 1 of
// colour j >> 7 (jj = j & 127: one half of a colour row, elements m = 2h, 2h + 1 of row
// (y, z), x_m = 2m + p, p = (colour + y + z) & 1).  The other colour's row at the same slots
// holds both cells' x-neighbours but one (element m + p - 1 / m + p: one extra scalar, in the
// tile or the x-neighbour tile), and its rows 4 / 32 slots away are the y / z neighbours
// (wrapped: -28 / +28, -224 / +224 into the neighbour tile), so a cell pair costs 15 float2 /
// scalar loads instead of 28.  The y / z side tests are uniform per thread.  Same per-cell
// fmaf order as k_apply_v4 (c p, then x-, x+, y-, y+, z-, z+), so q is bit-identical.
template <bool DOT, int MINB>
__global__ __launch_bounds__(NT, MINB) void k_apply_v5(ApplyArgs a) {
  __shared__ double sred[NT / 32];
  const int t = a.tiles ? a.tiles[blockIdx.x] : (int)blockIdx.x;
  int nb[6];
  {
    const int2* np = reinterpret_cast<const int2*>(a.nbr + 6 * (size_t)t);
    const int2 n0 = __ldg(np), n1 = __ldg(np + 1), n2 = __ldg(np + 2);
    nb[0] = n0.x; nb[1] = n0.y; nb[2] = n1.x; nb[3] = n1.y; nb[4] = n2.x; nb[5] = n2.y;
  }
  bool regular = true;
#pragma unroll
  for (int f = 0; f < 6; ++f) regular &= nb[f] >= -1 && nb[f] < a.NL;
  if (!regular) {
    apply_general<DOT>(a, t, sred);
    return;
  }
  const int j = threadIdx.x;
  const int colour = j >> 7, jj = j & 127;
  const int row = jj >> 1, h = jj & 1;
  const int y = row & 7, z = row >> 3;
  const int p = (colour + y + z) & 1;
  const int own = (colour << 8) + 2 * jj;  // slots of elements 2h, 2h + 1
  const int oth = own ^ 256;               // the other colour's row, same elements
  const float* pt = a.z + ((size_t)t << 9);
  const float* ct = a.coef + ((size_t)t << 11);
  auto tz = [&](int n) { return n >= 0 ? a.z + ((size_t)n << 9) : pt; };
  auto tc = [&](int n) { return n >= 0 ? a.coef + ((size_t)n << 11) : ct; };
  const float2 pc = __ldg(reinterpret_cast<const float2*>(pt + own));
  const float2 c0 = __ldg(reinterpret_cast<const float2*>(ct + own));
  const float2 cxm = __ldg(reinterpret_cast<const float2*>(ct + 512 + own));
  const float2 cym = __ldg(reinterpret_cast<const float2*>(ct + 1024 + own));
  const float2 czm = __ldg(reinterpret_cast<const float2*>(ct + 1536 + own));
  // x: the other row's elements 2h, 2h + 1 and the one outside them (p = 0: element 2h - 1,
  // p = 1: element 2h + 2), in the tile or the x-neighbour tile (element 3 / 0 of its row)
  const float2 ox = __ldg(reinterpret_cast<const float2*>(pt + oth));
  const float2 cxo = __ldg(reinterpret_cast<const float2*>(ct + 512 + oth));
  const bool xin = p ? h == 0 : h == 1;
  const int nx = p ? nb[1] : nb[0];  // the tile across the face the extra element lies beyond
  const int xo = p ? (xin ? oth + 2 : oth - 2) : (xin ? oth - 1 : oth + 3);
  float xs = __ldg((xin ? pt : tz(nx)) + xo);
  const float xsc = __ldg((xin ? ct : tc(nx)) + 512 + xo);  // its c_x- (used when p = 1)
  if (!xin && nx < 0) xs = 0.0f;
  // y / z: the other row 4 / 32 slots away (wrapped into the neighbour tile at the sides)
  const bool yl = y > 0, yh = y < 7, zl = z > 0, zh = z < 7;
  float2 ym = __ldg(reinterpret_cast<const float2*>((yl ? pt : tz(nb[2])) + oth + (yl ? -4 : 28)));
  float2 yp = __ldg(reinterpret_cast<const float2*>((yh ? pt : tz(nb[3])) + oth + (yh ? 4 : -28)));
  float2 zm = __ldg(reinterpret_cast<const float2*>((zl ? pt : tz(nb[4])) + oth + (zl ? -32 : 224)));
  float2 zp = __ldg(reinterpret_cast<const float2*>((zh ? pt : tz(nb[5])) + oth + (zh ? 32 : -224)));
  const float2 cyp = __ldg(reinterpret_cast<const float2*>((yh ? ct : tc(nb[3])) + 1024 + oth + (yh ? 4 : -28)));
  const float2 czp = __ldg(reinterpret_cast<const float2*>((zh ? ct : tc(nb[5])) + 1536 + oth + (zh ? 32 : -224)));
  if (!yl && nb[2] < 0) ym = make_float2(0.0f, 0.0f);
  if (!yh && nb[3] < 0) yp = make_float2(0.0f, 0.0f);
  if (!zl && nb[4] < 0) zm = make_float2(0.0f, 0.0f);
  if (!zh && nb[5] < 0) zp = make_float2(0.0f, 0.0f);
  // per element e: x- / x+ values and the x+ coupling
  const float xm0 = p ? ox.x : xs, xm1 = p ? ox.y : ox.x;
  const float xp0 = p ? ox.y : ox.x, xp1 = p ? xs : ox.y;
  const float cxp0 = p ? cxo.y : cxo.x, cxp1 = p ? xsc : cxo.y;
  const float pv0 = c0.x != 0.0f ? pc.x : 0.0f, pv1 = c0.y != 0.0f ? pc.y : 0.0f;
  float s0 = c0.x * pv0, s1 = c0.y * pv1;
  s0 = fmaf(cxm.x, xm0, s0); s1 = fmaf(cxm.y, xm1, s1);
  s0 = fmaf(cxp0, xp0, s0);  s1 = fmaf(cxp1, xp1, s1);
  s0 = fmaf(cym.x, ym.x, s0); s1 = fmaf(cym.y, ym.y, s1);
  s0 = fmaf(cyp.x, yp.x, s0); s1 = fmaf(cyp.y, yp.y, s1);
  s0 = fmaf(czm.x, zm.x, s0); s1 = fmaf(czm.y, zm.y, s1);
  s0 = fmaf(czp.x, zp.x, s0); s1 = fmaf(czp.y, zp.y, s1);
  const float r0 = c0.x != 0.0f ? s0 : 0.0f, r1 = c0.y != 0.0f ? s1 : 0.0f;
  *reinterpret_cast<float2*>(a.q + ((size_t)t << 9) + own) = make_float2(r0, r1);
  if (DOT) {
    const double d = (double)pv0 * (double)r0 + (double)pv1 * (double)r1;
    double bs = block_reduce_d(d, sred);
    if (threadIdx.x == 0) a.partial[blockIdx.x] = bs;
  }
}

template <bool DOT>
__global__ __launch_bounds__(NT, 5) void k_apply(ApplyArgs a) {
  __shared__ double sred[NT / 32];
  apply_general<DOT>(a, a.tiles ? a.tiles[blockIdx.x] : (int)blockIdx.x, sred);
}

// sigma = p.q from the per-tile partials (fixed order => deterministic)
__global__ __launch_bounds__(1024) void k_finish_sigma(const double* partial, int n, Scalars* sc) {
  __shared__ double sred[32];
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
    sc->sum_pq = tot;
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
  FOR_RANGES(R, i) {
    // b is in the caller's natural cell order: gather the 4 slots' cells
    const int64_t c0 = 4 * i, tb = c0 & ~(int64_t)511;
    const int s0 = (int)(c0 & 511);
    float m[4];
    for (int k = 0; k < 4; ++k) m[k] = __ldg(b + tb + slot_nat(s0 + k));
    const unsigned am = act4(act, i);
    for (int k = 0; k < 4; ++k) {
      if (!((am >> k) & 1u)) m[k] = 0.0f;
      s2 += (double)m[k] * m[k];
      s1 += (double)m[k];
    }
    reinterpret_cast<float4*>(r)[i] = make_float4(m[0], m[1], m[2], m[3]);
    reinterpret_cast<float4*>(x)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) sc->flags = 0;
  reduce2(s2, s1, partial, counter, sc, SF_RR, SF_R, sred);
}

// x += alpha p, r -= alpha q with alpha = (r,z)/(p,Ap) (Alg. 1 lines 9-11); sums ||r||^2,
// sum r.  The last block flags a breakdown and records rho = (r, z) for the next beta.
// alpha_fixed != 0: that step length instead (standalone multigrid: x += z, r -= A z)
__global__ __launch_bounds__(256) void k_update(float* __restrict__ x, float* __restrict__ r,
                                                const float* __restrict__ p, const float* __restrict__ q, Ranges R,
                                                double* partial, unsigned* counter, Scalars* sc, float alpha_fixed) {
  __shared__ double sred[8];
  const double pq = sc->sum_pq, rz = sc->sum_rz;
  const bool ok = alpha_fixed != 0.0f || (pq > 0.0 && isfinite(pq) && isfinite(rz));
  const float alpha = alpha_fixed != 0.0f ? alpha_fixed : (ok ? (float)(rz / pq) : 0.0f);
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
  double s2 = 0.0;
  FOR_RANGES(R, i) {
    float4 v = reinterpret_cast<float4*>(r)[i];
    float e[4] = {v.x, v.y, v.z, v.w};
    const unsigned am = act4(act, i);
    for (int k = 0; k < 4; ++k) {
      if ((am >> k) & 1u) e[k] -= m;
      s2 += (double)e[k] * e[k];
    }
    reinterpret_cast<float4*>(r)[i] = make_float4(e[0], e[1], e[2], e[3]);
  }
  double b2 = block_reduce_d(s2, sred);
  double tot;
  if (last_block_sum(b2, partial, counter, gridDim.x, &tot, sred)) sc->sum_rr = tot;
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

// dst (caller's natural order) = src (slot order) on the cells of the ranges
__global__ void k_copy_to_nat(const float* src, float* dst, Ranges R) {
  FOR_RANGES(R, i) {
    const float4 v = reinterpret_cast<const float4*>(src)[i];
    const int64_t c0 = 4 * i, tb = c0 & ~(int64_t)511;
    const int s0 = (int)(c0 & 511);
    dst[tb + slot_nat(s0)] = v.x;
    dst[tb + slot_nat(s0 + 1)] = v.y;
    dst[tb + slot_nat(s0 + 2)] = v.z;
    dst[tb + slot_nat(s0 + 3)] = v.w;
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

void launch_apply(const ApplyArgs& a, cudaStream_t s) {
  if (a.ntiles == 0) {
    if (a.partial) cudaMemsetAsync(&a.sc->sum_pq, 0, sizeof(double), s);
    return;
  }
  if (a.partial) {
    if (a.v2 == 5) k_apply_v5<true, 8><<<a.ntiles, NT, 0, s>>>(a);
    else if (a.v2 == 6) k_apply_v5<true, 6><<<a.ntiles, NT, 0, s>>>(a);
    else if (a.v2 == 4) k_apply_v4<true><<<a.ntiles, NT, 0, s>>>(a);
    else if (a.v2) k_apply_v2<true><<<a.ntiles, NT, 0, s>>>(a);
    else k_apply<true><<<a.ntiles, NT, 0, s>>>(a);
    k_finish_sigma<<<1, 1024, 0, s>>>(a.partial, a.ntiles, a.sc);
  } else {
    if (a.v2 == 5) k_apply_v5<false, 8><<<a.ntiles, NT, 0, s>>>(a);
    else if (a.v2 == 6) k_apply_v5<false, 6><<<a.ntiles, NT, 0, s>>>(a);
    else if (a.v2 == 4) k_apply_v4<false><<<a.ntiles, NT, 0, s>>>(a);
    else if (a.v2) k_apply_v2<false><<<a.ntiles, NT, 0, s>>>(a);
    else k_apply<false><<<a.ntiles, NT, 0, s>>>(a);
  }
}

void launch_init(const float* b, const uint32_t* act, float* r, float* x, const Ranges& R, double* partial,
                 unsigned* counter, Scalars* sc, cudaStream_t s, int grid) {
  k_init<<<grid, 256, 0, s>>>(b, act, r, x, R, partial, counter, sc);
}
void launch_update(float* x, float* r, const float* p, const float* q, const Ranges& R, double* partial,
                   unsigned* counter, Scalars* sc, cudaStream_t s, int grid, float alpha_fixed) {
  k_update<<<grid, 256, 0, s>>>(x, r, p, q, R, partial, counter, sc, alpha_fixed);
}
void launch_project(float* r, const uint32_t* act, const Ranges& R, double* partial, unsigned* counter, Scalars* sc,
                    cudaStream_t s, int grid) {
  k_project<<<grid, 256, 0, s>>>(r, act, R, partial, counter, sc);
}
void launch_dot_rz(const float* r, const float* z, const Ranges& R, double* partial, unsigned* counter, Scalars* sc,
                   cudaStream_t s, int grid) {
  k_dot_rz<<<grid, 256, 0, s>>>(r, z, R, partial, counter, sc);
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
