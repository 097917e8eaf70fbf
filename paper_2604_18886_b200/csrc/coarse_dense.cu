// The coarsest levels of the cycle as dense grids in shared memory (sm_100a).
//
// Below the coarsest leaf level every level of the tile octree is complete: level l is the
// whole domain, an (8 ext_x 2^l) x (8 ext_y 2^l) x (8 ext_z 2^l) box of inner cells (the
// leaves tile the domain, so each level-l tile has descendants and exists).  Their part of
// Alg. 4 — pre-smoothing, residual + restriction + Avg, FAS rhs, the mu
// recursive calls, the coarsest smoothing nu_b/2 x (R,B) + nu_b/2 x (B,R),
// prolongation, post-smoothing — runs here in ONE CTA with every value in shared memory,
// stored as a dense colour-split grid per level:
//
//   idx(x, y, z) = ((x + y + z) & 1) * n/2 + (z * ny + y) * nx/2 + (x >> 1),
//
// so a colour pass reads the other colour half at fixed offsets (x: -1 + p / +p, y: -+ nx/2,
// z: -+ nx ny / 2, p = x & 1) and consecutive threads touch consecutive words (no bank
// conflicts).  The coefficient records (c, c_x-, c_y-, c_z-) of these levels are converted
// to the same dense layout once at setup (build_coarse_dense) and copied in per visit with
// 128-bit loads; the +face coupling of a cell is its neighbour's -face entry.  The level-K
// rhs b^K and iterate u^K = u* arrive in the tile layout (written by the level-(K+1)
// restriction) and u^K (and b^K, which the first of the mu calls turns into the FAS rhs)
// leave the same way.  Per-cell arithmetic as the tile kernels (face sums in the order x-,
// x+, y-, y+, z-, z+ from 0, or from c u; block sums pair / y / z), so the replaced
// k_subcycle and this kernel agree to rounding.
//
// A phase (one colour pass, a restriction half, ...) is a few shared-memory loads per cell
// and one CTA barrier: ~0.1-0.3 us against the ~2 us of the global-memory sub-cycle, whose
// phases are dependent L1/L2 round trips plus ~100 instructions of tile indexing per cell.
#include <algorithm>
#include <cstdlib>
#include <vector>

#include <cooperative_groups.h>

#include "octmg_internal.cuh"

namespace cg = cooperative_groups;

namespace octmg {

namespace {



struct CDLevel {
  int nx, ny, nz;   // cells per axis
  int n;            // nx * ny * nz
  int shx, shy;     // log2(nx / 2), log2(ny) when powers of two, else -1 (division)
  int off;          // first cell of the level in the concatenated dense arrays
  int ntx, nty;     // tiles per axis (x, y)
  const int* tmap;  // [ntz][nty][ntx] global tile index of each level tile
};

struct CDArgs {
  CDLevel lv[CD_MAXL + 1];
  int K;                 // top level (the cycle enters here)
  int fas_first;         // form the FAS rhs of level K first
  int mu, nu_pre, nu_post, nu_coarsest;
  int std_form;          // Alg. 2: zero coarse guess, u* = 0, no FAS rhs, beta at prolongation
  float alpha, beta, pro_scale;
  const float* dcoef;    // dense coefficients: NP planes per level (c, c_x-, c_y-, c_z-, 1/c or 0), plane k of level l at NP off_l + k n_l
  // level-K fields in the tile layout (inner tiles): u (= u* on entry), b
  float* u_inner;
  float* b_inner;
  const int4* tile;      // tile table; level K's inner tiles are tK0 .. tK0 + n_K/512 - 1
  int tK0;
  int NL;
  int total;             // cells of levels 0..K
};

constexpr int NP = 5;  // coefficient planes per level: c, c_x-, c_y-, c_z-, 1/c (0 where inactive)

// shared memory: coef[NP * total] | u[total] | b[total] | ustar[total] | scratch[n_K]
struct CDMem {
  float* coef;
  float* u;
  float* b;
  float* us;
  float* scr;
};

__device__ __forceinline__ int didx(const CDLevel& L, int x, int y, int z) {
  return (((x + y + z) & 1) * (L.n >> 1)) + (z * L.ny + y) * (L.nx >> 1) + (x >> 1);
}

// coordinates of colour-c cell k of level L
__device__ __forceinline__ void dcell(const CDLevel& L, int c, int k, int& x, int& y, int& z) {
  const int hx = L.nx >> 1;
  int row;
  if (L.shx >= 0 && L.shy >= 0) {
    row = k >> L.shx;
    y = row & (L.ny - 1);
    z = row >> L.shy;
  } else {
    row = k / hx;
    y = row % L.ny;
    z = row / L.ny;
  }
  x = 2 * (k - row * hx) + ((c + y + z) & 1);
}

__device__ __forceinline__ float4 lds4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ float g4(const float4& v, int m) { return m == 0 ? v.x : m == 1 ? v.y : m == 2 ? v.z : v.w; }

// One colour row segment of 4 cells (x = 2m + p, m = 4 seg .. 4 seg + 3) of a dense colour-split
// grid: the face sums of the 4 cells from 128-bit shared-memory loads of the other colour's
// rows (same / y-+1 / z-+1) and coupling planes plus the one x-neighbour outside the segment
// — the row form of the tile kernels (rowtile.cuh) on shared memory, sum order x-, x+,
// y-, y+, z-, z+ from 0 or c u (the tile kernels'; walls 0), ~16 loads per 4 cells instead of ~14
// per cell and the index arithmetic once per segment.  vzm/vzp, czp: the z-neighbour rows
// (given by the caller: in the level, or across a slab boundary through distributed smem).
// (segment, row, y, z) of row-segment work item w of a dense level: shifts when the dims are
// powers of two (every unit-cube level), divisions otherwise
__device__ __forceinline__ void seg_rc(const CDLevel& L, int w, int nseg, int& seg, int& y, int& z) {
  int row;
  if (L.shx >= 2 && L.shy >= 0) {
    seg = w & (nseg - 1);
    row = w >> (L.shx - 2);
    y = row & (L.ny - 1);
    z = row >> L.shy;
  } else {
    seg = w % nseg;
    row = w / nseg;
    y = row % L.ny;
    z = row / L.ny;
  }
}

struct RowNb {
  float4 ox, ym, yp, zm, zp, cxo, cyp, czp;
  float xs, xsc;
};
__device__ __forceinline__ float4 row_face4(const RowNb& r, int p, const float4& qx, const float4& qy,
                                            const float4& qz, const float4& s0 = make_float4(0.0f, 0.0f, 0.0f, 0.0f)) {
  float o[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const float vxm = p ? g4(r.ox, m) : (m == 0 ? r.xs : g4(r.ox, m - 1));
    const float vxp = p ? (m == 3 ? r.xs : g4(r.ox, m + 1)) : g4(r.ox, m);
    const float cxp = p ? (m == 3 ? r.xsc : g4(r.cxo, m + 1)) : g4(r.cxo, m);
    float sm = g4(s0, m);
    sm = fmaf(g4(qx, m), vxm, sm);
    sm = fmaf(cxp, vxp, sm);
    sm = fmaf(g4(qy, m), g4(r.ym, m), sm);
    sm = fmaf(g4(r.cyp, m), g4(r.yp, m), sm);
    sm = fmaf(g4(qz, m), g4(r.zm, m), sm);
    sm = fmaf(g4(r.czp, m), g4(r.zp, m), sm);
    o[m] = sm;
  }
  return make_float4(o[0], o[1], o[2], o[3]);
}

// the in-plane part of a segment's neighbours (x, y) from the other colour's row at `oth`
__device__ __forceinline__ void row_nb_xy(RowNb& r, const float* u, const float* cx, const float* cy, int oth,
                                          int p, int seg, int nseg, int hx, int y, int ny) {
  const float4 Z4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  r.ox = lds4(u + oth);
  r.cxo = lds4(cx + oth);
  const bool xin = p ? seg < nseg - 1 : seg > 0;  // the x-neighbour outside the segment exists
  const int xo = p ? oth + 4 : oth - 1;
  r.xs = xin ? u[xo] : 0.0f;
  r.xsc = (p && xin) ? cx[xo] : 0.0f;
  r.ym = y > 0 ? lds4(u + oth - hx) : Z4;
  r.yp = y < ny - 1 ? lds4(u + oth + hx) : Z4;
  r.cyp = y < ny - 1 ? lds4(cy + oth + hx) : Z4;
}

// RBGS colour pass at level l, in place (reads only the other colour), row segments of 4
template <int NT>
__device__ __forceinline__ void cd_pass(const CDArgs& A, const CDMem& M, int l, int colour) {
  const CDLevel& L = A.lv[l];
  const int nh = L.n >> 1, hx = L.nx >> 1, nseg = hx >> 2, hxy = hx * L.ny;
  const float* u = M.u + L.off;
  const float* cc = M.coef + NP * L.off;
  const float *cx = cc + L.n, *cy = cx + L.n, *cz = cy + L.n, *inv = cz + L.n;
  const float* b = M.b + L.off;
  const int nw = (L.n >> 3);  // rows x segments of one colour (nh / 4)
  const float4 Z4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  for (int w = threadIdx.x; w < nw; w += NT) {
    int seg, y, z;
    seg_rc(L, w, nseg, seg, y, z);
    const int row = z * L.ny + y;
    const int p = (colour + y + z) & 1;
    const int own = colour * nh + row * hx + 4 * seg, oth = own + (colour ? -nh : nh);
    RowNb r;
    row_nb_xy(r, u, cx, cy, oth, p, seg, nseg, hx, y, L.ny);
    r.zm = z > 0 ? lds4(u + oth - hxy) : Z4;
    r.zp = z < L.nz - 1 ? lds4(u + oth + hxy) : Z4;
    r.czp = z < L.nz - 1 ? lds4(cz + oth + hxy) : Z4;
    const float4 f = row_face4(r, p, lds4(cx + own), lds4(cy + own), lds4(cz + own));
    const float4 bb = lds4(b + own), iv = lds4(inv + own);
    // u = (b - sum) / c with the precomputed 1/c (0 on inactive cells: u = 0 there)
    *reinterpret_cast<float4*>(M.u + L.off + own) =
        make_float4((bb.x - f.x) * iv.x, (bb.y - f.y) * iv.y, (bb.z - f.z) * iv.z, (bb.w - f.w) * iv.w);
  }
  __syncthreads();
}

// every row segment of both colours of a dense level: op(own, c, b, A u) with (A u) = c u +
// the face sums (row_face4's order from c u) — the residual and FAS-rhs phases in row form
template <int NT, class Op>
__device__ __forceinline__ void cd_rows_au(const CDLevel& L, const CDMem& M, const Op& op) {
  const int nh = L.n >> 1, hx = L.nx >> 1, nseg = hx >> 2, hxy = hx * L.ny, nw = L.n >> 3;
  const float* u = M.u + L.off;
  const float* cc = M.coef + NP * L.off;
  const float *cx = cc + L.n, *cy = cx + L.n, *cz = cy + L.n;
  const float4 Z4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  for (int w = threadIdx.x; w < 2 * nw; w += NT) {
    const int colour = w >= nw, ww = w - colour * nw;
    int seg, y, z;
    seg_rc(L, ww, nseg, seg, y, z);
    const int row = z * L.ny + y;
    const int p = (colour + y + z) & 1;
    const int own = colour * nh + row * hx + 4 * seg, oth = own + (colour ? -nh : nh);
    RowNb r;
    row_nb_xy(r, u, cx, cy, oth, p, seg, nseg, hx, y, L.ny);
    r.zm = z > 0 ? lds4(u + oth - hxy) : Z4;
    r.zp = z < L.nz - 1 ? lds4(u + oth + hxy) : Z4;
    r.czp = z < L.nz - 1 ? lds4(cz + oth + hxy) : Z4;
    const float4 c4 = lds4(cc + own), u4 = lds4(u + own);
    const float4 f = row_face4(r, p, lds4(cx + own), lds4(cy + own), lds4(cz + own),
                               make_float4(c4.x * u4.x, c4.y * u4.y, c4.z * u4.z, c4.w * u4.w));
    op(own, c4, f);
  }
}

template <int NT>
__device__ __forceinline__ void cd_passes(const CDArgs& A, const CDMem& M, int l, int iters, bool red_first) {
  for (int k = 0; k < iters; ++k) {
    cd_pass<NT>(A, M, l, red_first ? 0 : 1);
    cd_pass<NT>(A, M, l, red_first ? 1 : 0);
  }
}

// residual r = b - A u (active cells) into scratch, then per parent: u* = mean of the active
// children, u^{l-1} = u*, b^{l-1} = beta (R r) = beta sum(r) / alpha (Alg. 4 lines 8-10)
template <int NT>
__device__ __forceinline__ void cd_restrict(const CDArgs& A, const CDMem& M, int l) {
  const CDLevel& L = A.lv[l];
  const CDLevel& P = A.lv[l - 1];
  const float* bl = M.b + L.off;
  float* scr = M.scr;
  cd_rows_au<NT>(L, M, [&](int own, const float4& c4, const float4& f) {
    const float4 bb = lds4(bl + own);
    *reinterpret_cast<float4*>(scr + own) =
        make_float4(c4.x != 0.0f ? bb.x - f.x : 0.0f, c4.y != 0.0f ? bb.y - f.y : 0.0f,
                    c4.z != 0.0f ? bb.z - f.z : 0.0f, c4.w != 0.0f ? bb.w - f.w : 0.0f);
  });
  __syncthreads();
  for (int i = threadIdx.x; i < P.n; i += NT) {
    const int c = i >= (P.n >> 1);
    int X, Y, Z;
    dcell(P, c, i - c * (P.n >> 1), X, Y, Z);
    float rs[2][2], us[2][2];
    int na = 0;
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy) {
        float r2 = 0.0f, u2 = 0.0f;
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const int ci = didx(L, 2 * X + dx, 2 * Y + dy, 2 * Z + dz);
          const bool act = M.coef[NP * L.off + ci] != 0.0f;
          const float uv = act ? M.u[L.off + ci] : 0.0f;
          r2 = dx ? r2 + M.scr[ci] : M.scr[ci];
          u2 = dx ? u2 + uv : uv;
          na += act;
        }
        rs[dz][dy] = r2;
        us[dz][dy] = u2;
      }
    const float rsum = (rs[0][0] + rs[0][1]) + (rs[1][0] + rs[1][1]);
    const float usum = (us[0][0] + us[0][1]) + (us[1][0] + us[1][1]);
    const float mP = na ? usum / (float)na : 0.0f;
    M.u[P.off + i] = A.std_form ? 0.0f : mP;
    M.us[P.off + i] = A.std_form ? 0.0f : mP;
    M.b[P.off + i] = A.beta * (rsum / A.alpha);
  }
  __syncthreads();
}

// FAS rhs of level l: b += A^l u* (u holds u* here; Alg. 4 line 10)
template <int NT>
__device__ __forceinline__ void cd_fasrhs(const CDArgs& A, const CDMem& M, int l) {
  const CDLevel& L = A.lv[l];
  float* bl = M.b + L.off;
  // each thread reads and writes only its own b (the stencil reads u)
  cd_rows_au<NT>(L, M, [&](int own, const float4& c4, const float4& f) {
    const float4 bb = lds4(bl + own);
    *reinterpret_cast<float4*>(bl + own) =
        make_float4(c4.x != 0.0f ? bb.x + f.x : 0.0f, c4.y != 0.0f ? bb.y + f.y : 0.0f,
                    c4.z != 0.0f ? bb.z + f.z : 0.0f, c4.w != 0.0f ? bb.w + f.w : 0.0f);
  });
  __syncthreads();
}

// u^l += pro_scale (u^{l-1} - u*) on the active cells (Alg. 4 line 15)
template <int NT>
__device__ __forceinline__ void cd_prolong(const CDArgs& A, const CDMem& M, int l) {
  const CDLevel& L = A.lv[l];
  const CDLevel& P = A.lv[l - 1];
  // row segments of 4 cells (x = 2m + p, m = 4 seg + k): their parents X = m (both colours)
  const int nh = L.n >> 1, hx = L.nx >> 1, nseg = hx >> 2, nw = L.n >> 3, phx = P.nx >> 1, pnh = P.n >> 1;
  const float* pu = M.u + P.off;
  const float* ps = M.us + P.off;
  for (int w = threadIdx.x; w < 2 * nw; w += NT) {
    const int colour = w >= nw, ww = w - colour * nw;
    int seg, y, z;
    seg_rc(L, ww, nseg, seg, y, z);
    const int own = colour * nh + (z * L.ny + y) * hx + 4 * seg;
    const int Y = y >> 1, Z = z >> 1, pb = (Z * P.ny + Y) * phx;
    float4 u4 = lds4(M.u + L.off + own);
    const float4 c4 = lds4(M.coef + NP * L.off + own);
    float d[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int X = 4 * seg + m;
      const int pi = ((X + Y + Z) & 1) * pnh + pb + (X >> 1);
      d[m] = A.pro_scale * (pu[pi] - ps[pi]);
    }
    if (c4.x != 0.0f) u4.x += d[0];
    if (c4.y != 0.0f) u4.y += d[1];
    if (c4.z != 0.0f) u4.z += d[2];
    if (c4.w != 0.0f) u4.w += d[3];
    *reinterpret_cast<float4*>(M.u + L.off + own) = u4;
  }
  __syncthreads();
}

// Alg. 4 from level `top` down, iteratively (explicit per-level count of the mu coarse calls);
// fas_first: the first of the mu calls from level top + 1 (forms the FAS rhs of level top)
template <int NT>
__device__ void cd_cycle(const CDArgs& A, const CDMem& M, int top, bool fas_first) {
  int done[CD_MAXL + 1];
  int l = top;
  bool ff = fas_first;
  bool entering = true;
  while (true) {
    if (entering) {
      if (ff && !A.std_form) cd_fasrhs<NT>(A, M, l);
      if (l == 0) {
        const int h1 = A.nu_coarsest / 2;
        cd_passes<NT>(A, M, 0, h1, true);
        cd_passes<NT>(A, M, 0, A.nu_coarsest - h1, false);
      } else {
        cd_passes<NT>(A, M, l, A.nu_pre, true);
        cd_restrict<NT>(A, M, l);
        done[l] = 0;
        l -= 1;
        ff = true;
        continue;
      }
      entering = false;
    }
    if (l == top) break;
    const int p = l + 1;
    if (++done[p] < A.mu) {  // the next coarse call starts from the previous one's u^l
      l = p - 1;
      ff = false;
      entering = true;
      continue;
    }
    cd_prolong<NT>(A, M, p);
    cd_passes<NT>(A, M, p, A.nu_post, false);
    l = p;
  }
}

template <int NT>
__global__ __launch_bounds__(NT, 1) void k_coarse_dense(const __grid_constant__ CDArgs A) {
  extern __shared__ __align__(16) float smem[];
  CDMem M;
  M.coef = smem;
  M.u = M.coef + NP * A.total;
  M.b = M.u + A.total;
  M.us = M.b + A.total;
  M.scr = M.us + A.total;
  // copy in: the dense coefficients of levels 0..K (128-bit, 8 loads in flight per thread),
  // u^K and b^K from the level-K tiles (global inner tiles tK0.., coalesced slot runs)
  {
    const float4* src = reinterpret_cast<const float4*>(A.dcoef);
    float4* dst = reinterpret_cast<float4*>(M.coef);
    const int nv = NP * A.total / 4;
    for (int i0 = threadIdx.x; i0 < nv; i0 += 8 * NT) {
      float4 v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i0 + k * NT < nv) v[k] = __ldg(src + i0 + k * NT);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (i0 + k * NT < nv) dst[i0 + k * NT] = v[k];
    }
    // u^K, b^K: a tile's colour row (4 slots, one 128-bit run) is 4 consecutive dense cells
    const CDLevel& L = A.lv[A.K];
    const int nrow = (L.n >> 9) * 128;  // tiles x 2 colours x 64 rows
    for (int w = threadIdx.x; w < nrow; w += NT) {
      const int t = A.tK0 + (w >> 7), rc = w & 127;
      const int4 tv = __ldg(A.tile + t);
      const int sl = 4 * rc;  // colour (rc >> 6) half, row (y, z) = (rc & 7, (rc >> 3) & 7)
      const int di = ((rc >> 6) * (L.n >> 1)) + ((tv.w * 8 + ((rc >> 3) & 7)) * L.ny + tv.z * 8 + (rc & 7)) * (L.nx >> 1) +
                     4 * tv.y;
      const size_t gi = (size_t)(t - A.NL) * TB3 + sl;
      *reinterpret_cast<float4*>(M.u + L.off + di) = __ldg(reinterpret_cast<const float4*>(A.u_inner + gi));
      *reinterpret_cast<float4*>(M.b + L.off + di) = __ldg(reinterpret_cast<const float4*>(A.b_inner + gi));
    }
  }
  __syncthreads();
  cd_cycle<NT>(A, M, A.K, A.fas_first != 0);
  // copy out u^K and b^K (the FAS rhs persists across the mu calls from level K+1), tile rows
  const CDLevel& L = A.lv[A.K];
  const int nrow = (L.n >> 9) * 128;
  for (int w = threadIdx.x; w < nrow; w += NT) {
    const int t = A.tK0 + (w >> 7), rc = w & 127;
    const int4 tv = __ldg(A.tile + t);
    const int di = ((rc >> 6) * (L.n >> 1)) + ((tv.w * 8 + ((rc >> 3) & 7)) * L.ny + tv.z * 8 + (rc & 7)) * (L.nx >> 1) +
                   4 * tv.y;
    const size_t gi = (size_t)(t - A.NL) * TB3 + 4 * rc;
    *reinterpret_cast<float4*>(A.u_inner + gi) = lds4(M.u + L.off + di);
    if (A.fas_first) *reinterpret_cast<float4*>(A.b_inner + gi) = lds4(M.b + L.off + di);
  }
}

// setup: tile-layout coefficient records -> the dense colour-split planes of level l
__global__ void k_dense_coef(const float* coef, CDLevel L, int NL, float* dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.n) return;
  const int c = i >= (L.n >> 1);
  int x, y, z;
  dcell(L, c, i - c * (L.n >> 1), x, y, z);
  const int t = L.tmap[((z >> 3) * L.nty + (y >> 3)) * L.ntx + (x >> 3)];
  const float* p = coef + ((size_t)t << 11) + cslot(x & 7, y & 7, z & 7);
  for (int k = 0; k < 4; ++k) dst[(size_t)k * L.n + i] = p[k * 512];
  dst[(size_t)4 * L.n + i] = p[0] != 0.0f ? 1.0f / p[0] : 0.0f;
}

int shift_of(int v) {  // log2(v) for a power of two, else -1
  for (int k = 0; k < 31; ++k)
    if (v == (1 << k)) return k;
  return -1;
}


// ------------------------------------------------------------------------------------
// Levels 0..2 in one thread-block cluster (ext = (1,1,1)): level 2 (32^3 cells) is cut into
// CC z-slabs of 32 x 32 x SLZ cells, one per CTA of the cluster, each a dense colour-split
// grid in its CTA's shared memory (the colour of a cell is (x + y + z_local) & 1 since the
// slab origin is even); the z-neighbours across a slab boundary are read from the adjacent
// CTA's shared memory (distributed shared memory), and every level-2 phase ends with a
// cluster barrier (release/acquire at cluster scope).  Levels 0-1 live in CTA 0 as in
// k_coarse_dense and run there between two cluster barriers; the level-2 restriction writes
// the level-1 parents (slab c -> level-1 plane c) and the prolongation reads them through
// distributed shared memory.  One launch per level-2 visit replaces ~11 per-level launches
// and the level-1 dense launches of the W-cycle.
// ------------------------------------------------------------------------------------
constexpr int CC = 16;        // CTAs per cluster (non-portable cluster size)
constexpr int SLZ = 2;        // level-2 planes per CTA (32 / CC)

struct CCArgs {
  CDArgs A;                   // levels 0..1 (CTA 0), K = 1
  int nx, ny;                 // level-2 plane (32 x 32)
  const float* dcoef2;        // [CC][NP][nS] slab coefficient planes
  const int* tmap2;           // level-2 tile map [tz][ty][tx] (4 x 4 x 4)
  int fas_first;              // form the FAS rhs of level 2 first
  int tK0;                    // (unused: level-2 tiles via tmap2)
};

struct Slab {
  int nx, ny, n, hx, hxy;     // n = nx * ny * SLZ, hx = nx / 2, hxy = hx * ny
  int shseg, shy;             // log2(hx / 4), log2(ny) (powers of two: the unit cube's level 2)
  int c;                      // cluster rank = slab index
  float* coef;                // NP planes of n
  float* u;
  float* b;
  float* scr;
  const float* u_lo;          // u of the slab below (rank c - 1; null at the bottom wall)
  const float* cz_hi;         // c_z- plane of the slab above (rank c + 1; null at the top wall)
  const float* u_hi;
};

__device__ __forceinline__ void slab_cell(const Slab& S, int c, int k, int& x, int& y, int& z) {
  // k-th cell of colour c: row = k / hx (power-of-two dims)
  const int row = k / S.hx;
  y = row % S.ny;
  z = row / S.ny;
  x = 2 * (k - row * S.hx) + ((c + y + z) & 1);
}
__device__ __forceinline__ int slab_idx(const Slab& S, int x, int y, int z) {
  return (((x + y + z) & 1) * (S.n >> 1)) + (z * S.ny + y) * S.hx + (x >> 1);
}

// every row segment of both colours of the slab: op(own, c, A u) (cd_rows_au's form, the
// z-neighbour rows across the slab boundary from the adjacent CTAs' shared memory)
template <int NT, class Op>
__device__ __forceinline__ void slab_rows_au(const Slab& S, const Op& op) {
  const int nh = S.n >> 1, hx = S.hx, nseg = hx >> 2, hxy = S.hxy, nw = S.n >> 3;
  const float* u = S.u;
  const float *cx = S.coef + S.n, *cy = cx + S.n, *cz = cy + S.n;
  const float4 Z4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  for (int w = threadIdx.x; w < 2 * nw; w += NT) {
    const int colour = w >= nw, ww = w - colour * nw;
    const int seg = ww & (nseg - 1), row = ww >> S.shseg;  // (slab dims are powers of two)
    const int y = row & (S.ny - 1), z = row >> S.shy;
    const int p = (colour + y + z) & 1;
    const int own = colour * nh + row * hx + 4 * seg, oth = own + (colour ? -nh : nh);
    RowNb r;
    row_nb_xy(r, u, cx, cy, oth, p, seg, nseg, hx, y, S.ny);
    if (z > 0) r.zm = lds4(u + oth - hxy);
    else r.zm = S.u_lo ? lds4(S.u_lo + oth + hxy) : Z4;
    if (z < SLZ - 1) {
      r.zp = lds4(u + oth + hxy);
      r.czp = lds4(cz + oth + hxy);
    } else if (S.u_hi) {
      r.zp = lds4(S.u_hi + oth - hxy);
      r.czp = lds4(S.cz_hi + oth - hxy);
    } else {
      r.zp = Z4;
      r.czp = Z4;
    }
    const float4 c4 = lds4(S.coef + own), u4 = lds4(u + own);
    const float4 f = row_face4(r, p, lds4(cx + own), lds4(cy + own), lds4(cz + own),
                               make_float4(c4.x * u4.x, c4.y * u4.y, c4.z * u4.z, c4.w * u4.w));
    op(own, c4, f);
  }
}

// the slab colour pass in row segments of 4 (cd_pass's form; the z-neighbour rows across the
// slab boundary from the adjacent CTAs' shared memory, 128-bit distributed-smem loads)
template <int NT>
__device__ __forceinline__ void slab_pass(const Slab& S, int colour, cg::cluster_group& cl) {
  const int nh = S.n >> 1, hx = S.hx, nseg = hx >> 2, hxy = S.hxy;
  const float* u = S.u;
  const float *cx = S.coef + S.n, *cy = cx + S.n, *cz = cy + S.n, *inv = cz + S.n;
  const int nw = S.n >> 3;
  const float4 Z4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  for (int w = threadIdx.x; w < nw; w += NT) {
    const int seg = w & (nseg - 1), row = w >> S.shseg;
    const int y = row & (S.ny - 1), z = row >> S.shy;
    const int p = (colour + y + z) & 1;
    const int own = colour * nh + row * hx + 4 * seg, oth = own + (colour ? -nh : nh);
    RowNb r;
    row_nb_xy(r, u, cx, cy, oth, p, seg, nseg, hx, y, S.ny);
    if (z > 0) r.zm = lds4(u + oth - hxy);
    else r.zm = S.u_lo ? lds4(S.u_lo + oth + hxy) : Z4;
    if (z < SLZ - 1) {
      r.zp = lds4(u + oth + hxy);
      r.czp = lds4(cz + oth + hxy);
    } else if (S.u_hi) {
      r.zp = lds4(S.u_hi + oth - hxy);
      r.czp = lds4(S.cz_hi + oth - hxy);
    } else {
      r.zp = Z4;
      r.czp = Z4;
    }
    const float4 f = row_face4(r, p, lds4(cx + own), lds4(cy + own), lds4(cz + own));
    const float4 bb = lds4(S.b + own), iv = lds4(inv + own);
    *reinterpret_cast<float4*>(S.u + own) =
        make_float4((bb.x - f.x) * iv.x, (bb.y - f.y) * iv.y, (bb.z - f.z) * iv.z, (bb.w - f.w) * iv.w);
  }
  cl.sync();
}

template <int NT>
__global__ __launch_bounds__(NT, 1) void k_coarse_cluster(const __grid_constant__ CCArgs C) {
  extern __shared__ __align__(16) float smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const CDArgs& A = C.A;
  // shared memory: levels 0-1 (used by CTA 0) | level-2 slab
  CDMem M;
  M.coef = smem;
  M.u = M.coef + NP * A.total;
  M.b = M.u + A.total;
  M.us = M.b + A.total;
  M.scr = M.us + A.total;
  Slab S;
  S.nx = C.nx;
  S.ny = C.ny;
  S.n = C.nx * C.ny * SLZ;
  S.hx = C.nx >> 1;
  S.hxy = S.hx * C.ny;
  S.shseg = 31 - __clz(S.hx >> 2);
  S.shy = 31 - __clz(C.ny);
  S.c = rank;
  S.coef = M.scr + A.lv[1].n;
  S.u = S.coef + NP * S.n;
  S.b = S.u + S.n;
  S.scr = M.scr;  // the level-1 residual scratch is idle while level 2 runs
  S.u_lo = rank > 0 ? cl.map_shared_rank(S.u, rank - 1) : nullptr;
  S.u_hi = rank < CC - 1 ? cl.map_shared_rank(S.u, rank + 1) : nullptr;
  S.cz_hi = rank < CC - 1 ? cl.map_shared_rank(S.coef + 3 * S.n, rank + 1) : nullptr;
  // level-1 fields of CTA 0 (written by the restriction, read by the prolongation)
  const CDLevel& L1 = A.lv[1];
  float* u1 = cl.map_shared_rank(M.u + L1.off, 0);
  float* us1 = cl.map_shared_rank(M.us + L1.off, 0);
  float* b1 = cl.map_shared_rank(M.b + L1.off, 0);
  // copy in: the slab's coefficients, its u^2 and b^2 (tile layout); CTA 0 also levels 0-1
  {
    const float4* src = reinterpret_cast<const float4*>(C.dcoef2 + (size_t)rank * NP * S.n);
    float4* dst = reinterpret_cast<float4*>(S.coef);
    for (int i = threadIdx.x; i < NP * S.n / 4; i += NT) dst[i] = __ldg(src + i);
    if (rank == 0) {
      const float4* s0 = reinterpret_cast<const float4*>(A.dcoef);
      float4* d0 = reinterpret_cast<float4*>(M.coef);
      for (int i = threadIdx.x; i < NP * A.total / 4; i += NT) d0[i] = __ldg(s0 + i);
    }
    // u^2, b^2: a row segment of 4 same-colour cells (x = 2(4 seg + k) + p) is one 128-bit run of
    // 4 slots of tile x >> 3 = seg (the tile's colour = the slab's: the slab origin is even)
    const int nseg = S.hx >> 2, nw = S.n >> 3, nh = S.n >> 1;
    for (int w = threadIdx.x; w < 2 * nw; w += NT) {
      const int colour = w >= nw, ww = w - colour * nw;
      const int seg = ww & (nseg - 1), row = ww >> S.shseg;
      const int y = row & (S.ny - 1), z = row >> S.shy;
      const int zg = SLZ * rank + z;
      const int t = __ldg(C.tmap2 + ((zg >> 3) * (C.ny >> 3) + (y >> 3)) * (C.nx >> 3) + seg);
      const size_t gi = (size_t)(t - A.NL) * TB3 + (colour << 8) + 4 * (y & 7) + 32 * (zg & 7);
      const int own = colour * nh + row * S.hx + 4 * seg;
      *reinterpret_cast<float4*>(S.u + own) = __ldg(reinterpret_cast<const float4*>(A.u_inner + gi));
      *reinterpret_cast<float4*>(S.b + own) = __ldg(reinterpret_cast<const float4*>(A.b_inner + gi));
    }
  }
  cl.sync();
  if (C.fas_first && !A.std_form) {  // b^2 += A^2 u* (u^2 = u* on entry; the stencil reads u only)
    slab_rows_au<NT>(S, [&](int own, const float4& c4, const float4& f) {
      const float4 bb = lds4(S.b + own);
      *reinterpret_cast<float4*>(S.b + own) =
          make_float4(c4.x != 0.0f ? bb.x + f.x : 0.0f, c4.y != 0.0f ? bb.y + f.y : 0.0f,
                      c4.z != 0.0f ? bb.z + f.z : 0.0f, c4.w != 0.0f ? bb.w + f.w : 0.0f);
    });
    cl.sync();  // the neighbours' reads of u done before the passes write it
  }
  // pre-smoothing (R, B) x nu_pre
  for (int k = 0; k < A.nu_pre; ++k) {
    slab_pass<NT>(S, 0, cl);
    slab_pass<NT>(S, 1, cl);
  }
  // residual, then the level-1 parents of this slab (plane `rank`) into CTA 0
  slab_rows_au<NT>(S, [&](int own, const float4& c4, const float4& f) {
    const float4 bb = lds4(S.b + own);
    *reinterpret_cast<float4*>(S.scr + own) =
        make_float4(c4.x != 0.0f ? bb.x - f.x : 0.0f, c4.y != 0.0f ? bb.y - f.y : 0.0f,
                    c4.z != 0.0f ? bb.z - f.z : 0.0f, c4.w != 0.0f ? bb.w - f.w : 0.0f);
  });
  __syncthreads();
  for (int q = threadIdx.x; q < (S.nx >> 1) * (S.ny >> 1); q += NT) {
    const int X = q % (S.nx >> 1), Y = q / (S.nx >> 1);
    float rs[2][2], us[2][2];
    int na = 0;
#pragma unroll
    for (int dz = 0; dz < 2; ++dz)
#pragma unroll
      for (int dy = 0; dy < 2; ++dy) {
        float r2 = 0.0f, u2 = 0.0f;
#pragma unroll
        for (int dx = 0; dx < 2; ++dx) {
          const int ci = slab_idx(S, 2 * X + dx, 2 * Y + dy, dz);
          const bool act = S.coef[ci] != 0.0f;
          const float uv = act ? S.u[ci] : 0.0f;
          r2 = dx ? r2 + S.scr[ci] : S.scr[ci];
          u2 = dx ? u2 + uv : uv;
          na += act;
        }
        rs[dz][dy] = r2;
        us[dz][dy] = u2;
      }
    const float rsum = (rs[0][0] + rs[0][1]) + (rs[1][0] + rs[1][1]);
    const float usum = (us[0][0] + us[0][1]) + (us[1][0] + us[1][1]);
    const float mP = na ? usum / (float)na : 0.0f;
    const int pi = didx(L1, X, Y, rank);
    u1[pi] = A.std_form ? 0.0f : mP;
    us1[pi] = A.std_form ? 0.0f : mP;
    b1[pi] = A.beta * (rsum / A.alpha);
  }
  cl.sync();
  // the mu coarse calls at levels 1..0 in CTA 0 (shared memory, CTA barriers)
  if (rank == 0)
    for (int k = 0; k < A.mu; ++k) cd_cycle<NT>(A, M, 1, k == 0);
  cl.sync();
  // prolongation u^2 += pro_scale (u^1 - u*) from CTA 0, then post-smoothing (B, R) x nu_post
  {
    // row segments of 4 cells: their parents X = 4 seg + k in plane `rank` of level 1 (CTA 0)
    const int nseg = S.hx >> 2, nw = S.n >> 3, nh = S.n >> 1, phx = L1.nx >> 1, pnh = L1.n >> 1;
    for (int w = threadIdx.x; w < 2 * nw; w += NT) {
      const int colour = w >= nw, ww = w - colour * nw;
      const int seg = ww & (nseg - 1), row = ww >> S.shseg;
      const int y = row & (S.ny - 1), z = row >> S.shy;
      const int own = colour * nh + row * S.hx + 4 * seg;
      const int Y = y >> 1, Z = rank, pb = (Z * L1.ny + Y) * phx;
      float4 u4 = lds4(S.u + own);
      const float4 c4 = lds4(S.coef + own);
      float d[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int X = 4 * seg + m;
        const int pi = ((X + Y + Z) & 1) * pnh + pb + (X >> 1);
        d[m] = A.pro_scale * (u1[pi] - us1[pi]);
      }
      (void)z;
      if (c4.x != 0.0f) u4.x += d[0];
      if (c4.y != 0.0f) u4.y += d[1];
      if (c4.z != 0.0f) u4.z += d[2];
      if (c4.w != 0.0f) u4.w += d[3];
      *reinterpret_cast<float4*>(S.u + own) = u4;
    }
  }
  cl.sync();
  for (int k = 0; k < A.nu_post; ++k) {
    slab_pass<NT>(S, 1, cl);
    slab_pass<NT>(S, 0, cl);
  }
  // copy out u^2 (and the FAS rhs b^2 of the first mu call), row segments as the copy-in
  {
    const int nseg = S.hx >> 2, nw = S.n >> 3, nh = S.n >> 1;
    for (int w = threadIdx.x; w < 2 * nw; w += NT) {
      const int colour = w >= nw, ww = w - colour * nw;
      const int seg = ww & (nseg - 1), row = ww >> S.shseg;
      const int y = row & (S.ny - 1), z = row >> S.shy;
      const int zg = SLZ * rank + z;
      const int t = __ldg(C.tmap2 + ((zg >> 3) * (C.ny >> 3) + (y >> 3)) * (C.nx >> 3) + seg);
      const size_t gi = (size_t)(t - A.NL) * TB3 + (colour << 8) + 4 * (y & 7) + 32 * (zg & 7);
      const int own = colour * nh + row * S.hx + 4 * seg;
      *reinterpret_cast<float4*>(A.u_inner + gi) = lds4(S.u + own);
      if (C.fas_first) *reinterpret_cast<float4*>(A.b_inner + gi) = lds4(S.b + own);
    }
  }
}

// setup: level-2 coefficient records -> the slab planes [CC][NP][nS]
__global__ void k_slab_coef(const float* coef, const int* tmap2, int nx, int ny, float* dst) {
  const int nS = nx * ny * SLZ;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= nS * CC) return;
  const int rank = g / nS, i = g % nS;
  Slab S;
  S.nx = nx; S.ny = ny; S.n = nS; S.hx = nx >> 1; S.hxy = S.hx * ny;
  const int c = i >= (nS >> 1);
  int x, y, z;
  slab_cell(S, c, i - c * (nS >> 1), x, y, z);
  const int zg = SLZ * rank + z;
  const int t = tmap2[((zg >> 3) * (ny >> 3) + (y >> 3)) * (nx >> 3) + (x >> 3)];
  const float* p = coef + ((size_t)t << 11) + cslot(x & 7, y & 7, zg & 7);
  float* d = dst + (size_t)rank * NP * nS;
  for (int k = 0; k < 4; ++k) d[(size_t)k * nS + i] = p[k * 512];
  d[(size_t)4 * nS + i] = p[0] != 0.0f ? 1.0f / p[0] : 0.0f;
}
}  // namespace

size_t coarse_dense_smem(int total_cells, int nK) { return sizeof(float) * ((size_t)(NP + 3) * total_cells + nK); }

// Levels 0..K as dense grids if every tile of those levels is an inner tile (K below the
// coarsest leaf level) and their fields fit the shared memory of one CTA.  Returns K, or -1.
octmg_status build_coarse_dense(Hier& h, int Kmax, cudaStream_t s) {
  const Tree& T = *h.tree;
  h.cd_K = -1;
  if (getenv("OCTMG_COARSE_DENSE") && std::string(getenv("OCTMG_COARSE_DENSE")) == "0") return OCTMG_OK;
  int lmin = T.L;
  for (int l = 0; l <= T.L; ++l)
    if (T.lc[l] > 0) { lmin = l; break; }
  int dev = 0, smem_optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  int K = -1, total = 0;
  for (int l = 0; l <= std::min({Kmax, lmin - 1, CD_MAXL}); ++l) {
    const int n = T.ic[l] * TB3;
    const int expect = T.ext[0] * T.ext[1] * T.ext[2] * (1 << (3 * l)) * TB3;
    if (n != expect) break;  // not a complete level
    if (coarse_dense_smem(total + n, n) > (size_t)smem_optin) break;
    total += n;
    K = l;
  }
  if (K < 0) return OCTMG_OK;
  // tile maps (host) from the tile table
  std::vector<int4> tile(T.T);
  OCTMG_CUDA(cudaMemcpy(tile.data(), T.tile, sizeof(int4) * T.T, cudaMemcpyDeviceToHost));
  std::vector<int> maps;
  std::vector<int> moff(K + 1);
  for (int l = 0; l <= K; ++l) {
    const int ntx = T.ext[0] << l, nty = T.ext[1] << l, ntz = T.ext[2] << l;
    moff[l] = (int)maps.size();
    maps.resize(maps.size() + (size_t)ntx * nty * ntz, -1);
    for (int t = T.ib[l]; t < T.ib[l] + T.ic[l]; ++t) {  // ib: global tile index of the level's first inner tile
      const int4 v = tile[t];
      if (v.x != l || v.y < 0 || v.y >= ntx || v.z < 0 || v.z >= nty || v.w < 0 || v.w >= ntz) return OCTMG_OK;
      maps[moff[l] + ((size_t)v.w * nty + v.z) * ntx + v.y] = t;
    }
  }
  for (int v : maps)
    if (v < 0) return OCTMG_OK;  // (cannot happen for a complete level)
  int* dmap = (int*)dev_malloc(sizeof(int) * maps.size());
  float* dcoef = (float*)dev_malloc(sizeof(float) * NP * (size_t)total);
  if (!dmap || !dcoef) {
    set_error("device allocation failed (dense coarse levels)");
    return OCTMG_E_OOM;
  }
  h.allocs.push_back(dmap);
  h.allocs.push_back(dcoef);
  OCTMG_CUDA(cudaMemcpy(dmap, maps.data(), sizeof(int) * maps.size(), cudaMemcpyHostToDevice));
  int off = 0;
  for (int l = 0; l <= K; ++l) {
    CDLevel L;
    L.nx = T.ext[0] * 8 << l;
    L.ny = T.ext[1] * 8 << l;
    L.nz = T.ext[2] * 8 << l;
    L.n = L.nx * L.ny * L.nz;
    L.off = off;
    L.ntx = T.ext[0] << l;
    L.nty = T.ext[1] << l;
    L.tmap = dmap + moff[l];
    L.shx = shift_of(L.nx >> 1);
    L.shy = shift_of(L.ny);
    k_dense_coef<<<(L.n + 255) / 256, 256, 0, s>>>(h.ccoef, L, T.NL, dcoef + NP * (size_t)off);
    h.cd_lv[l][0] = L.nx; h.cd_lv[l][1] = L.ny; h.cd_lv[l][2] = L.nz; h.cd_lv[l][3] = off;
    off += L.n;
  }
  OCTMG_CUDA(cudaGetLastError());
  const size_t smem = coarse_dense_smem(total, T.ic[K] * TB3);
  OCTMG_CUDA(cudaFuncSetAttribute(k_coarse_dense<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  OCTMG_CUDA(cudaFuncSetAttribute(k_coarse_dense<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  OCTMG_CUDA(cudaFuncSetAttribute(k_coarse_dense<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const char* ct = getenv("OCTMG_CD_THREADS");  // threads of the dense coarse CTA (256 / 512 / 1024)
  h.cd_threads = ct ? atoi(ct) : 512;
  h.cd_K = K;
  h.cd_total = total;
  h.cd_map = dmap;
  h.cd_moff = moff;
  h.cd_coef = dcoef;
  return OCTMG_OK;
}

void launch_coarse_dense(const Hier& h, int K, int fas_first, float* u_inner, float* b_inner, cudaStream_t s) {
  const Tree& T = *h.tree;
  CDArgs A;
  for (int l = 0; l <= CD_MAXL; ++l) {
    CDLevel& L = A.lv[l];
    if (l <= K) {
      L.nx = h.cd_lv[l][0]; L.ny = h.cd_lv[l][1]; L.nz = h.cd_lv[l][2];
      L.n = L.nx * L.ny * L.nz;
      L.off = h.cd_lv[l][3];
      L.ntx = T.ext[0] << l;
      L.nty = T.ext[1] << l;
      L.tmap = h.cd_map + h.cd_moff[l];
      L.shx = shift_of(L.nx >> 1);
      L.shy = shift_of(L.ny);
    } else {
      L = CDLevel{0, 0, 0, 0, -1, -1, 0, 0, 0, nullptr};
    }
  }
  A.K = K;
  A.fas_first = fas_first;
  A.mu = h.prm.mu;
  A.nu_pre = h.prm.nu_pre;
  A.nu_post = h.prm.nu_post;
  A.nu_coarsest = h.prm.nu_coarsest;
  A.std_form = h.prm.form == 1;
  A.alpha = h.prm.alpha;
  A.beta = A.std_form ? 1.0f : h.prm.beta_overshoot;
  A.pro_scale = A.std_form ? h.prm.beta_overshoot : 1.0f;
  A.dcoef = h.cd_coef;
  A.u_inner = u_inner;
  A.b_inner = b_inner;
  A.tile = T.tile;
  A.tK0 = T.ib[K];
  A.NL = T.NL;
  int total = 0;
  for (int l = 0; l <= K; ++l) total += A.lv[l].n;
  A.total = total;
  const size_t sm = coarse_dense_smem(total, A.lv[K].n);
  switch (h.cd_threads) {
    case 256: k_coarse_dense<256><<<1, 256, sm, s>>>(A); break;
    case 512: k_coarse_dense<512><<<1, 512, sm, s>>>(A); break;
    default: k_coarse_dense<1024><<<1, 1024, sm, s>>>(A); break;
  }
}

}  // namespace octmg

namespace octmg {

// Levels 0..2 in one cluster of CC CTAs (k_coarse_cluster): needs the dense levels 0-1
// (cd_K == 1), a complete inner level 2 of a unit-cube domain, and a device that can host a
// cluster of CC CTAs with this much shared memory each.  Sets h.cc_K = 2 on success.
octmg_status build_coarse_cluster(Hier& h, cudaStream_t s) {
  const Tree& T = *h.tree;
  h.cc_K = -1;
  const char* e = getenv("OCTMG_COARSE_CLUSTER");
  if (e && atoi(e) == 0) return OCTMG_OK;
  if (h.cd_K != 1 || T.L < 3 || T.ext[0] != 1 || T.ext[1] != 1 || T.ext[2] != 1) return OCTMG_OK;
  if (T.lc[2] != 0 || T.ic[2] != 64) return OCTMG_OK;
  const int nx = 32, ny = 32, nS = nx * ny * SLZ;
  // level-2 tile map
  std::vector<int4> tile(T.T);
  OCTMG_CUDA(cudaMemcpy(tile.data(), T.tile, sizeof(int4) * T.T, cudaMemcpyDeviceToHost));
  std::vector<int> map(64, -1);
  for (int t = T.ib[2]; t < T.ib[2] + T.ic[2]; ++t) {
    const int4 v = tile[t];
    if (v.x != 2 || v.y < 0 || v.y > 3 || v.z < 0 || v.z > 3 || v.w < 0 || v.w > 3) return OCTMG_OK;
    map[(v.w * 4 + v.z) * 4 + v.y] = t;
  }
  for (int v : map)
    if (v < 0) return OCTMG_OK;
  const size_t smem = coarse_dense_smem(h.cd_total, T.ic[1] * TB3) + sizeof(float) * (size_t)(NP + 2) * nS;
  const int NTc = 512;
  if (cudaFuncSetAttribute(k_coarse_cluster<NTc>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
      cudaFuncSetAttribute(k_coarse_cluster<NTc>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
    cudaGetLastError();
    return OCTMG_OK;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CC);
  cfg.blockDim = dim3(NTc);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  if (cudaOccupancyMaxActiveClusters(&nclusters, k_coarse_cluster<NTc>, &cfg) != cudaSuccess || nclusters < 1) {
    cudaGetLastError();
    return OCTMG_OK;
  }
  int* dmap = (int*)dev_malloc(sizeof(int) * 64);
  float* dc2 = (float*)dev_malloc(sizeof(float) * (size_t)CC * NP * nS);
  if (!dmap || !dc2) {
    set_error("device allocation failed (cluster coarse levels)");
    return OCTMG_E_OOM;
  }
  h.allocs.push_back(dmap);
  h.allocs.push_back(dc2);
  OCTMG_CUDA(cudaMemcpy(dmap, map.data(), sizeof(int) * 64, cudaMemcpyHostToDevice));
  k_slab_coef<<<(nS * CC + 255) / 256, 256, 0, s>>>(h.ccoef, dmap, nx, ny, dc2);
  OCTMG_CUDA(cudaGetLastError());
  h.cc_map = dmap;
  h.cc_coef = dc2;
  h.cc_smem = smem;
  h.cc_K = 2;
  return OCTMG_OK;
}

void launch_coarse_cluster(const Hier& h, int fas_first, float* u_inner, float* b_inner, cudaStream_t s) {
  const Tree& T = *h.tree;
  CCArgs C;
  CDArgs& A = C.A;
  for (int l = 0; l <= CD_MAXL; ++l) {
    CDLevel& L = A.lv[l];
    if (l <= 1) {
      L.nx = h.cd_lv[l][0]; L.ny = h.cd_lv[l][1]; L.nz = h.cd_lv[l][2];
      L.n = L.nx * L.ny * L.nz;
      L.off = h.cd_lv[l][3];
      L.ntx = T.ext[0] << l;
      L.nty = T.ext[1] << l;
      L.tmap = h.cd_map + h.cd_moff[l];
      L.shx = shift_of(L.nx >> 1);
      L.shy = shift_of(L.ny);
    } else {
      L = CDLevel{0, 0, 0, 0, -1, -1, 0, 0, 0, nullptr};
    }
  }
  A.K = 1;
  A.fas_first = 0;
  A.mu = h.prm.mu;
  A.nu_pre = h.prm.nu_pre;
  A.nu_post = h.prm.nu_post;
  A.nu_coarsest = h.prm.nu_coarsest;
  A.std_form = h.prm.form == 1;
  A.alpha = h.prm.alpha;
  A.beta = A.std_form ? 1.0f : h.prm.beta_overshoot;
  A.pro_scale = A.std_form ? h.prm.beta_overshoot : 1.0f;
  A.dcoef = h.cd_coef;
  A.u_inner = u_inner;
  A.b_inner = b_inner;
  A.tile = T.tile;
  A.tK0 = T.ib[1];
  A.NL = T.NL;
  A.total = A.lv[0].n + A.lv[1].n;
  C.nx = 32;
  C.ny = 32;
  C.dcoef2 = h.cc_coef;
  C.tmap2 = h.cc_map;
  C.fas_first = fas_first;
  C.tK0 = T.ib[2];
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CC);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = h.cc_smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k_coarse_cluster<512>, C);
}

}  // namespace octmg
