// Sync-light tile kernels (sm_100a): RBGS colour pass, residual + restriction + Avg,
// prolongation.  One CTA of 256 threads per 8^3 tile; each thread gathers the 7-point
// stencil of its cell(s) directly through L1/L2 (in-tile neighbours are L1 hits of the
// CTA's own loads; face neighbours come from the adjacent tiles via the cached neighbour
// table).  No shared-memory staging: every load of a cell is independent and
// in flight at once.  Ghost values are reconstructed per access (Eq. 12, P:L661-665,
// P:L880-882) from the pass-start snapshot.
#include <cstdlib>
#include <string>

#include "stencil.cuh"
#include "rowstencil.cuh"
#include "rowtile.cuh"

namespace octmg {

namespace {

constexpr int NT = 256;

// Regular-tile stencil context: the tile's and its six neighbours' value pointers and the
// +face coupling planes, set up once per thread and shared by its colour cells.  In the
// colour-split slot order all six neighbours of a cell sit in the other colour's half at
// fixed offsets from the cell's own index q (x: q-1+p / q+p with p = x&1; y: q-+4; z: q-+32;
// wrapped into the neighbour tile: +3 / -3, +28 / -28, +224 / -224).
struct RegCtx {
  const float* un[6];   // u of the face-neighbour tile (own tile at walls)
  const float* cn[3];   // c_x- / c_y- / c_z- planes of the +x / +y / +z neighbour tile
  const float* cown[3]; // the same planes of this tile
  bool wall[6];
};

__device__ __forceinline__ void reg_ctx(const SmoothArgs& a, int t, const int (&nb)[6], const float* ut, RegCtx& c) {
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int n = nb[f];
    c.wall[f] = n < 0;
    c.un[f] = n >= 0 ? tptr(a.u, n, a.NL) : ut;
  }
#pragma unroll
  for (int ax = 0; ax < 3; ++ax) {
    const int n = nb[2 * ax + 1];
    c.cown[ax] = a.coef + ((size_t)t << 11) + ((1 + ax) << 9);
    c.cn[ax] = n >= 0 ? a.coef + ((size_t)n << 11) + ((1 + ax) << 9) : c.cown[ax];
  }
}

// Face sum of a cell (slot sl, coordinates x, y, z) of a tile with no ghost face.  Every
// load is issued unconditionally (walls read the tile itself and are zeroed), so all loads
// of a cell are in flight at once and none waits on the cell's activity test.
__device__ __forceinline__ float face_sum_regular(const RegCtx& c, const float* ut, int sl, int x, int y, int z,
                                                  const float4& q) {
  const int base = sl ^ 256;
  const int p = x & 1;
  const bool in[6] = {x > 0, x < 7, y > 0, y < 7, z > 0, z < 7};
  const int dlt[6] = {in[0] ? p - 1 : 3, in[1] ? p : -3, in[2] ? -4 : 28, in[3] ? 4 : -28, in[4] ? -32 : 224,
                      in[5] ? 32 : -224};
  float s = 0.0f;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int ax = f >> 1;
    const int no = base + dlt[f];
    float v = __ldg((in[f] ? ut : c.un[f]) + no);
    const float cf = (f & 1) ? __ldg((in[f] ? c.cown[ax] : c.cn[ax]) + no) : comp(q, ax);
    if (!in[f] && c.wall[f]) v = 0.0f;
    s = fmaf(cf, v, s);
  }
  return s;
}

// The colour pass with the neighbour entries prefetched and, on tiles without a ghost face
// (every tile of a uniform level), the branch-free face sum above.  Thread j's colour cells
// are the contiguous slots colour*256 + j + k*256/CPT.
template <int MODE, int CPT>
__global__ __launch_bounds__(NT / CPT, 7 * CPT) void k_pass_v2(SmoothArgs a) {
  const int t = level_tile(a, blockIdx.x);
  int nb[6];
  {
    const int2* np = reinterpret_cast<const int2*>(a.nbr + 6 * (size_t)t);
    const int2 n0 = __ldg(np), n1 = __ldg(np + 1), n2 = __ldg(np + 2);
    nb[0] = n0.x; nb[1] = n0.y; nb[2] = n1.x; nb[3] = n1.y; nb[4] = n2.x; nb[5] = n2.y;
  }
  const int colour = a.stage[0] & 1;
  const int j = threadIdx.x;
  const int y = (j >> 2) & 7, z0 = j >> 5;
  float* ut = tptr(a.u, t, a.NL);
  const float* bt = tptr(a.b, t, a.NL);
  const float* ct = a.coef + ((size_t)t << 11);
  bool ghost = false;
#pragma unroll
  for (int f = 0; f < 6; ++f) ghost |= nb[f] <= -2;
  ghost = ghost && MODE != SM_ZERO1;
  RegCtx rc;
  if (MODE != SM_ZERO1 && !ghost) reg_ctx(a, t, nb, ut, rc);
  float unew[CPT];
  bool act[CPT];
  int offs[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int z = z0 + k * (8 / CPT);
    const int x = 2 * (j & 3) + ((colour + y + z) & 1);
    const int off = (colour << 8) + j + k * (256 / CPT);  // = loff(x, y, z): this colour's q
    offs[k] = off;
    const float4 q = make_float4(__ldg(ct + off), __ldg(ct + 512 + off), __ldg(ct + 1024 + off),
                                 __ldg(ct + 1536 + off));
    const float b = __ldg(bt + off);
    act[k] = q.x != 0.0f;
    float v;
    if (MODE == SM_ZERO1) {
      v = b / q.x;
    } else if (!ghost) {
      v = (b - face_sum_regular(rc, ut, off, x, y, z, q)) / q.x;
    } else {
      const float ui = MODE == SM_ZERO2 ? 0.0f : __ldg(ut + off);
      const float mP = block_mean<MODE == SM_ZERO2>(a, t, x, y, z, colour);
      v = act[k] ? (b - face_sum<MODE == SM_ZERO2>(a, t, x, y, z, q, ui, mP, colour, 0.0f)) / q.x : 0.0f;
    }
    unew[k] = act[k] ? v : 0.0f;
  }
  __syncthreads();  // every pass-start read of this tile precedes the in-place writes
#pragma unroll
  for (int k = 0; k < CPT; ++k)
    if (act[k] || MODE == SM_ZERO1 || MODE == SM_ZERO2) ut[offs[k]] = unew[k];
}


// The colour pass, one colour row per thread (rowtile.cuh): thread j of a 64-thread tile
// CTA owns row (y, z) = (j & 7, j >> 3) of the pass colour, 13 float4 + 2 scalar loads for 4
// cells.  Regular tiles only read the other colour (and their own colour's b and record), so
// no barrier is needed before the in-place store.  Tiles with a T-junction face take the
// same row path with the Eq. 12 ghost values substituted (rowk::row_ghosts; snapshot reading
// 1 of DESIGN.md): u_i and m_P come from the pass-start values of the own row and, by
// shuffles of registers, of the rows y^1 / z^1 (lanes j^1 / j^8).  No thread reads another
// row's own-colour cells from memory, so no barrier is needed here either.
template <int MODE, bool GHOST>
__device__ __forceinline__ void pass_row_body(const SmoothArgs& a, int t, const int (&nb)[6]) {
  using namespace rowk;
  const int colour = a.stage[0] & 1;
  const RowGeo g = row_geo(colour, threadIdx.x);
  float* ut = tptr(a.u, t, a.NL);
  const float* ct = a.coef + ((size_t)t << 11);
  const float4 q0 = ld4(ct + g.own);
  const float4 bb = ld4(tptr(a.b, t, a.NL) + g.own);
  if (MODE == SM_ZERO1) {  // first pass of the cycle: u = 0, so u = b / c
    float4 r;
    r.x = q0.x != 0.0f ? bb.x / q0.x : 0.0f;
    r.y = q0.y != 0.0f ? bb.y / q0.y : 0.0f;
    r.z = q0.z != 0.0f ? bb.z / q0.z : 0.0f;
    r.w = q0.w != 0.0f ? bb.w / q0.w : 0.0f;
    *reinterpret_cast<float4*>(ut + g.own) = r;
    return;
  }
  int4 tv;
  int3 gl;
  if (GHOST) {  // the ghost path's tile origin and ghost-layer indices, issued first
    tv = __ldg(a.tile + t);
    gl = load_gl(a.glayer, t);
  }
  const float4 qx = ld4(ct + 512 + g.own), qy = ld4(ct + 1024 + g.own), qz = ld4(ct + 1536 + g.own);
  const Fld uf = a.u;
  const int NL = a.NL;
  auto tu = [uf, NL](int n) -> const float* { return tptr(uf, n, NL); };
  RowSt s;
  row_load(s, tu, a.coef, t, nb, g);
  if (GHOST) {
    const float4 Z4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    const float4 ui = MODE == SM_ZERO2 ? Z4 : ld4(ut + g.own);
    const float4 co = ld4(ct + g.oth);
    const float4 mP = row_block_mean<1, 8>(msk4(ui, q0), q0, msk4(s.ox, co), co);
    const Fld ucf = a.uc;
    auto uc_of = [ucf, NL](int C) -> const float* { return tptr(ucf, C, NL); };
    row_ghosts<MODE == SM_ZERO2>(s, g, t, nb, tv, a.coef, a.glayer_val, gl, uc_of, ui, mP);
  }
  const float4 f = row_sums(s, g, qx, qy, qz, make_float4(0.0f, 0.0f, 0.0f, 0.0f));
  float4 r;
  r.x = q0.x != 0.0f ? (bb.x - f.x) / q0.x : 0.0f;
  r.y = q0.y != 0.0f ? (bb.y - f.y) / q0.y : 0.0f;
  r.z = q0.z != 0.0f ? (bb.z - f.z) / q0.z : 0.0f;
  r.w = q0.w != 0.0f ? (bb.w - f.w) / q0.w : 0.0f;
  *reinterpret_cast<float4*>(ut + g.own) = r;
  if (MODE == SM_PLAIN_RZ) {
    // the last pass of M on a uniform tree (every leaf at this level): z is final here — this
    // colour's row just computed, the other colour's row (s.ox) untouched since the previous
    // pass — so (r, z) of Alg. 1 line 12 is summed here (r = the leaf b) instead of in a pass
    // of its own; one fp64 partial per warp (2 per tile), summed in fixed order afterwards
    const float4 bo = ld4(tptr(a.b, t, a.NL) + g.oth);
    double dd = (double)bb.x * (double)r.x + (double)bb.y * (double)r.y + (double)bb.z * (double)r.z +
                (double)bb.w * (double)r.w;
    dd += (double)bo.x * (double)s.ox.x + (double)bo.y * (double)s.ox.y + (double)bo.z * (double)s.ox.z +
          (double)bo.w * (double)s.ox.w;
    for (int o = 16; o; o >>= 1) dd += __shfl_down_sync(0xffffffffu, dd, o);
    if ((threadIdx.x & 31) == 0) a.rz_partial[2 * (size_t)blockIdx.x + (threadIdx.x >> 5)] = dd;
  }
}

// the ghost-tile body out of line: its extra registers (spilled to L1-resident local memory
// if need be) do not lower the occupancy of the regular-tile path
template <int MODE>
__device__ __noinline__ void pass_row_ghost(const SmoothArgs& a, int t, int n0, int n1, int n2, int n3, int n4,
                                            int n5) {
  const int nb[6] = {n0, n1, n2, n3, n4, n5};
  pass_row_body<MODE, true>(a, t, nb);
}

// INL: the ghost body inlined (1: at 12 CTAs/SM, 80 registers; 2: at 14 CTAs/SM, 72 registers)
// instead of out of line at 16 (the regular path's occupancy; the ghost body spills)
// (an instance without the ghost path for ghost-free levels — 61 registers, no call frame —
// measured slower: config 2 level-5 passes 2.77 vs 2.63 ms per solve; not kept)
template <int MODE, int INL>  // INL: 0 out of line (16 CTAs/SM), 1 inline at 12, 2 inline at 14
__global__ __launch_bounds__(64, INL == 1 ? 12 : (INL == 2 ? 14 : 16)) void k_pass_v3(const __grid_constant__ SmoothArgs a) {
  const int t = level_tile(a, blockIdx.x);
  int nb[6];
  rowk::load_nb(a.nbr, t, nb);
  bool ghost = false;
#pragma unroll
  for (int f = 0; f < 6; ++f) ghost |= nb[f] <= -2;
  if (MODE != SM_ZERO1 && ghost) {  // CTA-uniform
    if (INL != 0) pass_row_body<MODE, true>(a, t, nb);
    else pass_row_ghost<MODE>(a, t, nb[0], nb[1], nb[2], nb[3], nb[4], nb[5]);
    return;
  }
  pass_row_body<MODE, false>(a, t, nb);
}

// Residual r = b - A^l u and, per parent (inner, level l-1): u* = mean of the active
// children (Avg, Alg. 4 line 9), u^{l-1} := u*, b^{l-1} := beta * (R r), R = P^T / alpha
// (Alg. 4 lines 8-10; "residual computation and restriction step are fused").
// Thread j of a 256-thread tile CTA owns the x-pair (2 (j & 3), y, z); the lanes of one
// 2x2x2 block are 4 apart in a warp (bits 2, 3 = y & 1, z & 1), so block sums are two
// xor-shuffles.  Neighbour entries prefetched; on tiles without a ghost face the
// branch-free face sum (every load in flight at once, in-tile neighbours from L1).
template <int MINB>
__global__ __launch_bounds__(NT, MINB) void k_restrict_v2(SmoothArgs a) {
  const int t = level_tile(a, blockIdx.x);
  int nb[6];
  {
    const int2* np = reinterpret_cast<const int2*>(a.nbr + 6 * (size_t)t);
    const int2 n0 = __ldg(np), n1 = __ldg(np + 1), n2 = __ldg(np + 2);
    nb[0] = n0.x; nb[1] = n0.y; nb[2] = n1.x; nb[3] = n1.y; nb[4] = n2.x; nb[5] = n2.y;
  }
  // the tile's origin and parent (for the parent-cell stores at the end) are loaded up front,
  // with the neighbour entries, not after the face sums
  const int4 tv = __ldg(a.tile + t);
  const int P = __ldg(a.parent + t);
  const int j = threadIdx.x;
  const int x2 = j & 3;
  const int y = ((j >> 2) & 1) | (((j >> 4) & 3) << 1);
  const int z = ((j >> 3) & 1) | ((j >> 6) << 1);
  const int x0 = 2 * x2;
  const int off0 = loff(x0, y, z);
  const float* cb = a.coef + ((size_t)t << 11);
  const float2 qc = ldpair(cb, off0), qx = ldpair(cb + 512, off0), qy = ldpair(cb + 1024, off0),
               qz = ldpair(cb + 1536, off0);
  const float4 q0 = make_float4(qc.x, qx.x, qy.x, qz.x), q1 = make_float4(qc.y, qx.y, qy.y, qz.y);
  const float2 uu = ldpair(tptr(a.u, t, a.NL), off0);
  const float2 bb = ldpair(tptr(a.b, t, a.NL), off0);
  bool ghost = false;
#pragma unroll
  for (int f = 0; f < 6; ++f) ghost |= nb[f] <= -2;
  float f0, f1;
  if (!ghost) {
    const RowTiles rt = row_tiles(t, nb, y, z);
    FldVals vals;
#pragma unroll
    for (int f = 0; f < 6; ++f) vals.p[f] = tptr(a.u, rt.tf[f], a.NL);
    const float2 f = row2_faces(vals, rt, x2, y, z, uu, make_float2(q0.y, q1.y), make_float2(q0.z, q1.z),
                                make_float2(q0.w, q1.w), make_float2(q0.x * uu.x, q1.x * uu.y),
                                a.coef + ((size_t)rt.tf[1] << 11) + 512, a.coef + ((size_t)rt.tf[3] << 11) + 1024,
                                a.coef + ((size_t)rt.tf[5] << 11) + 1536);
    f0 = f.x;
    f1 = f.y;
  }
  // active u sum / count of the block (also the ghost m_P of its cells)
  float su = (q0.x != 0.0f ? uu.x : 0.0f) + (q1.x != 0.0f ? uu.y : 0.0f);
  int na = (q0.x != 0.0f) + (q1.x != 0.0f);
  su += __shfl_xor_sync(0xffffffffu, su, 4);
  na += __shfl_xor_sync(0xffffffffu, na, 4);
  su += __shfl_xor_sync(0xffffffffu, su, 8);
  na += __shfl_xor_sync(0xffffffffu, na, 8);
  const float mP = na ? su / (float)na : 0.0f;
  if (ghost) {
    f0 = q0.x != 0.0f ? face_sum<false>(a, t, x0, y, z, q0, uu.x, mP, 0, q0.x * uu.x) : 0.0f;
    f1 = q1.x != 0.0f ? face_sum<false>(a, t, x0 + 1, y, z, q1, uu.y, mP, 0, q1.x * uu.y) : 0.0f;
  }
  // (A u) summed as c*u, then faces x-, x+, y-, y+, z-, z+ (the staged / sub-cycle order)
  const float r0 = q0.x != 0.0f ? bb.x - f0 : 0.0f;
  const float r1 = q1.x != 0.0f ? bb.y - f1 : 0.0f;
  float rs = r0 + r1;
  rs += __shfl_xor_sync(0xffffffffu, rs, 4);
  rs += __shfl_xor_sync(0xffffffffu, rs, 8);
  if (((j >> 2) & 3) == 0) {
    const int pc = pcell_of(tv, x0, y, z);
    const size_t pi = (size_t)(P - a.NL) * TB3 + pc;
    a.u.inner[pi] = a.std_form ? 0.0f : mP;  // Alg. 2: zero coarse guess, u* = 0
    a.ustar_w[pi] = a.std_form ? 0.0f : mP;
    a.b.inner[pi] = a.beta * (rs / a.alpha);
  }
}

// Residual + restriction + Avg (Alg. 4 lines 8-10) in the row layout of k_apply_v6, for the
// levels that have T-junction (ghost) tiles: thread j of a 128-thread tile CTA owns row
// j >> 1 of colour j & 1.  r = b - A^l u per cell with the Eq. 12 ghosts substituted in the
// row (rowk::row_ghosts; m_P by shuffles), then per 2x2x2 block the residual sum r_own +
// r_oth (lane j^1), + the row y^1 (j^2), + the row z^1 (j^16) — k_restrict_v2's order — and
// the active-u mean m_P.  The rows with z even write the four parent cells of their block
// row, one each ((y & 1) * 2 + colour).  On ghost-free levels k_restrict_v2 (pairs of cells
// per thread) is faster (config 2: 0.94 vs 1.04 ms per solve); on ghost levels this one
// (config 3: 3.80 vs 4.18 ms) — the per-cell general ghost path is the slow part there.
template <bool GHOST>
__device__ __forceinline__ void restrict_row_body(const SmoothArgs& a, int t, const int (&nb)[6]) {
  using namespace rowk;
  const int4 tv = __ldg(a.tile + t);
  const int P = __ldg(a.parent + t);
  int3 gl;
  if (GHOST) gl = load_gl(a.glayer, t);
  const RowGeo g = row_geo(threadIdx.x & 1, threadIdx.x >> 1);
  const float* ut = tptr(a.u, t, a.NL);
  const float* ct = a.coef + ((size_t)t << 11);
  const float4 q0 = ld4(ct + g.own), qx = ld4(ct + 512 + g.own), qy = ld4(ct + 1024 + g.own),
               qz = ld4(ct + 1536 + g.own);
  const float4 uu = ld4(ut + g.own);
  const float4 bb = ld4(tptr(a.b, t, a.NL) + g.own);
  const float4 co = ld4(ct + g.oth);
  const Fld uf = a.u;
  const int NL = a.NL;
  auto tu = [uf, NL](int n) -> const float* { return tptr(uf, n, NL); };
  RowSt s;
  row_load(s, tu, a.coef, t, nb, g);
  const float4 mP = row_block_mean<2, 16>(msk4(uu, q0), q0, msk4(s.ox, co), co);
  if (GHOST) {
    const Fld ucf = a.uc;
    auto uc_of = [ucf, NL](int C) -> const float* { return tptr(ucf, C, NL); };
    row_ghosts<false>(s, g, t, nb, tv, a.coef, a.glayer_val, gl, uc_of, uu, mP);
  }
  const float4 f = row_sums(s, g, qx, qy, qz, make_float4(q0.x * uu.x, q0.y * uu.y, q0.z * uu.z, q0.w * uu.w));
  const unsigned FULL = 0xffffffffu;
  float rs[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const float c = e4(q0, m);
    float v = c != 0.0f ? e4(bb, m) - e4(f, m) : 0.0f;
    v += __shfl_xor_sync(FULL, v, 1);
    v += __shfl_xor_sync(FULL, v, 2);
    v += __shfl_xor_sync(FULL, v, 16);
    rs[m] = v;
  }
  if ((g.z & 1) == 0) {
    const int m = 2 * (g.y & 1) + (threadIdx.x & 1);
    const int pc = cslot(((tv.y & 1) << 2) + m, ((tv.z & 1) << 2) + (g.y >> 1), ((tv.w & 1) << 2) + (g.z >> 1));
    const size_t pi = (size_t)(P - a.NL) * TB3 + pc;
    const float mm = e4(mP, m);
    a.u.inner[pi] = a.std_form ? 0.0f : mm;  // Alg. 2: zero coarse guess, u* = 0
    a.ustar_w[pi] = a.std_form ? 0.0f : mm;
    a.b.inner[pi] = a.beta * ((m == 0 ? rs[0] : m == 1 ? rs[1] : m == 2 ? rs[2] : rs[3]) / a.alpha);
  }
}

__global__ __launch_bounds__(128, 6) void k_restrict_row(const __grid_constant__ SmoothArgs a) {
  const int t = level_tile(a, blockIdx.x);
  int nb[6];
  rowk::load_nb(a.nbr, t, nb);
  bool ghost = false;
#pragma unroll
  for (int f = 0; f < 6; ++f) ghost |= nb[f] <= -2;
  if (ghost) restrict_row_body<true>(a, t, nb);  // CTA-uniform
  else restrict_row_body<false>(a, t, nb);
}

// Residual + restriction + Avg on a level without T-junction tiles, right after the
// pre-smoothing's last pass (black): that pass set every black cell to u_B = (b_B - sum_f
// c_f u_f) / c_B from its red neighbours, which have not changed since, so r_B = b_B - c_B u_B
// - sum_f c_f u_f = 0 (in exact arithmetic; in fp32 a recomputation would only add the
// cancellation noise of b - c u - sum).  Only the red rows are computed: thread j of a
// 64-thread tile CTA owns red row (y, z) = (j & 7, j >> 3) — the colour pass's layout and
// loads, plus the black c plane for the Avg activity — and the block sums are the red
// residuals of the rows y, y^1 (lane j^1) and z^1 (lane j^8) (k_restrict_v2's pair / y / z
// order with a zero black term).  The rows with z even write the block row's four parents,
// two each.  22 B per cell instead of 25.5, and one stencil per two cells.
__global__ __launch_bounds__(64, 14) void k_restrict_red(const __grid_constant__ SmoothArgs a) {
  using namespace rowk;
  const int t = level_tile(a, blockIdx.x);
  int nb[6];
  load_nb(a.nbr, t, nb);
  const int4 tv = __ldg(a.tile + t);
  const int P = __ldg(a.parent + t);
  const RowGeo g = row_geo(0, threadIdx.x);
  const float* ut = tptr(a.u, t, a.NL);
  const float* ct = a.coef + ((size_t)t << 11);
  const float4 q0 = ld4(ct + g.own), qx = ld4(ct + 512 + g.own), qy = ld4(ct + 1024 + g.own),
               qz = ld4(ct + 1536 + g.own);
  const float4 uu = ld4(ut + g.own);
  const float4 bb = ld4(tptr(a.b, t, a.NL) + g.own);
  const float4 co = ld4(ct + g.oth);
  const Fld uf = a.u;
  const int NL = a.NL;
  auto tu = [uf, NL](int n) -> const float* { return tptr(uf, n, NL); };
  RowSt s;
  row_load(s, tu, a.coef, t, nb, g);
  const float4 mP = row_block_mean<1, 8>(msk4(uu, q0), q0, msk4(s.ox, co), co);
  const float4 f = row_sums(s, g, qx, qy, qz, make_float4(q0.x * uu.x, q0.y * uu.y, q0.z * uu.z, q0.w * uu.w));
  const unsigned FULL = 0xffffffffu;
  float rs[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const float c = e4(q0, m);
    float v = c != 0.0f ? e4(bb, m) - e4(f, m) : 0.0f;
    v += __shfl_xor_sync(FULL, v, 1);
    v += __shfl_xor_sync(FULL, v, 8);
    rs[m] = v;
  }
  if ((g.z & 1) == 0) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int m = 2 * (g.y & 1) + k;
      const int pc = cslot(((tv.y & 1) << 2) + m, ((tv.z & 1) << 2) + (g.y >> 1), ((tv.w & 1) << 2) + (g.z >> 1));
      const size_t pi = (size_t)(P - a.NL) * TB3 + pc;
      const float mm = e4(mP, m);
      a.u.inner[pi] = a.std_form ? 0.0f : mm;  // Alg. 2: zero coarse guess, u* = 0
      a.ustar_w[pi] = a.std_form ? 0.0f : mm;
      a.b.inner[pi] = a.beta * ((m == 0 ? rs[0] : m == 1 ? rs[1] : m == 2 ? rs[2] : rs[3]) / a.alpha);
    }
  }
}

// Prolongation of the coarse update, in place: u_i += u^{l-1}_P - u*_P for every active
// cell (Alg. 4 line 15; no beta).  4 cells per thread (float4).
__global__ __launch_bounds__(128) void k_prolong(SmoothArgs a) {
  const int t = level_tile(a, blockIdx.x);
  // thread j: the 4 same-q cells at slots j, j + 128 (red) and j + 256, j + 384 (black):
  // every access is a coalesced scalar per warp
  const int4 tv = __ldg(a.tile + t);
  const int P = __ldg(a.parent + t);
  float* ut = tptr(a.u, t, a.NL);
  const float* cc = a.coef + ((size_t)t << 11);
  const float* uc = tptr(a.uc, P, a.NL);
  const float* us = a.ustar + (size_t)(P - a.NL) * TB3;
  // the cells' u and activity do not depend on the parent: loaded before the parent values
  // arrive and unconditionally, so no load waits behind the activity branch
  float uo[4], cv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int sl = threadIdx.x + 128 * k;
    uo[k] = ut[sl];
    cv[k] = __ldg(cc + sl);
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int sl = threadIdx.x + 128 * k;
    int x, y, z;
    slot_xyz(sl, x, y, z);
    const int pc = pcell_of(tv, x, y, z);
    float c = a.pro_scale * (__ldg(uc + pc) - __ldg(us + pc));
    if (a.pro_active_only && __ldg(a.coef + ((size_t)P << 11) + pc) == 0.0f) c = 0.0f;
    if (cv[k] != 0.0f) ut[sl] = uo[k] + c;
  }
}

// FAS right-hand side of the inner rows of a coarse level (Alg. 4 line 10):
// b_I = beta R r (already in b) + (A^{l-1} u*)_I, with u* in u (inner rows) and the current
// u of the leaf rows.  Inner tiles never border a ghost (grading), so no reconstruction.
__global__ __launch_bounds__(NT, 8) void k_fasrhs(SmoothArgs a) {
  const int t = a.first_tile + blockIdx.x;
  const int j = threadIdx.x;
  const int y = (j >> 2) & 7, z = j >> 5, x0 = 2 * (j & 3);
  const int off0 = loff(x0, y, z), off1 = off0 ^ 256;
  const size_t base = (size_t)t * TB3;
  const float4 q0 = ldcoef(a.coef, base + off0), q1 = ldcoef(a.coef, base + off1);
  const float2 uu = ldpair(tptr(a.u, t, a.NL), off0);
  float* bt = a.b.inner + (size_t)(t - a.NL) * TB3;
  const float b0 = bt[off0], b1 = bt[off1];
  bt[off0] = q0.x != 0.0f ? b0 + face_sum<false>(a, t, x0, y, z, q0, 0.0f, 0.0f, 0, q0.x * uu.x) : 0.0f;
  bt[off1] = q1.x != 0.0f ? b1 + face_sum<false>(a, t, x0 + 1, y, z, q1, 0.0f, 0.0f, 0, q1.x * uu.y) : 0.0f;
}

// The FAS right-hand side in the row layout (thread j of a 128-thread tile CTA owns row j >> 1 of
// colour j & 1, rowtile.cuh): b_I += (A^{l-1} u*)_I summed as c*u, then faces x-, x+, y-, y+,
// z-, z+ (k_fasrhs's order, so bit-identical) from one float4 row of each neighbour instead
// of k_fasrhs's per-cell general path (config 2 level 4: 28 us -> ~8 us per visit, L2-resident)
__global__ __launch_bounds__(128, 8) void k_fasrhs_row(const __grid_constant__ SmoothArgs a) {
  using namespace rowk;
  const int t = a.first_tile + blockIdx.x;
  int nb[6];
  load_nb(a.nbr, t, nb);
  const RowGeo g = row_geo(threadIdx.x & 1, threadIdx.x >> 1);
  const float* ct = a.coef + ((size_t)t << 11);
  const float4 q0 = ld4(ct + g.own), qx = ld4(ct + 512 + g.own), qy = ld4(ct + 1024 + g.own),
               qz = ld4(ct + 1536 + g.own);
  const float4 uu = ld4(tptr(a.u, t, a.NL) + g.own);
  float* bt = a.b.inner + (size_t)(t - a.NL) * TB3 + g.own;
  const float4 bb = *reinterpret_cast<const float4*>(bt);
  const Fld uf = a.u;
  const int NL = a.NL;
  auto tu = [uf, NL](int n) -> const float* { return tptr(uf, n, NL); };
  RowSt st;
  row_load(st, tu, a.coef, t, nb, g);  // inner tiles never border a ghost (grading)
  const float4 f = row_sums(st, g, qx, qy, qz, make_float4(q0.x * uu.x, q0.y * uu.y, q0.z * uu.z, q0.w * uu.w));
  *reinterpret_cast<float4*>(bt) =
      make_float4(q0.x != 0.0f ? bb.x + f.x : 0.0f, q0.y != 0.0f ? bb.y + f.y : 0.0f,
                  q0.z != 0.0f ? bb.z + f.z : 0.0f, q0.w != 0.0f ? bb.w + f.w : 0.0f);
}

}  // namespace

// k_pass_v3's ghost body: inlined (80 registers, 12 CTAs/SM) on levels with ghost tiles,
// out of line (the regular path at 16 CTAs/SM) elsewhere; OCTMG_PASS_GHOST=inline / call
// forces one form on every level (measured: inline 10.2 vs 11.3 ms of passes per config-3
// solve; out of line 2.72 vs 3.15 ms on config 2, which has no ghost tile)
static bool pass_ghost_inline(bool level_has_ghosts) {
  int mode = -1;  // (env read per call: the variant tests switch it within one process)
  if (mode < 0) {
    const char* e = getenv("OCTMG_PASS_GHOST");
    mode = !e ? 0 : (std::string(e) == "inline" ? 1 : (std::string(e) == "call" ? 2 : 0));
  }
  return mode == 1 || (mode == 0 && level_has_ghosts);
}

// the inlined ghost body at 12 CTAs/SM (80 registers, no spills); OCTMG_PASS_GHOST_MINB=14 for
// 72 registers with 24 B of spills (measured late in round 2, after the ghost-row changes: 12
// is faster on configs 3 / 4 / 5 — 24.85 vs 25.49, 102.3 vs 104.1, 468.7 vs 479.7 ms per solve;
// earlier in the round 14 had measured better on config 3)
static int pass_ghost_minb() {
  int v = -1;
  if (v < 0) {
    const char* e = getenv("OCTMG_PASS_GHOST_MINB");
    v = e ? atoi(e) : 12;
  }
  return v;
}

// OCTMG_PASS_V=2: the scalar k_pass_v2 on big levels instead of the 128-bit k_pass_v3
bool pass_v3_on();
static bool pass_v3_enabled() { return pass_v3_on(); }
bool pass_v3_on() {
  int on = -1;
  if (on < 0) {
    const char* e = getenv("OCTMG_PASS_V");
    on = !(e && (std::string(e) == "2" || std::string(e) == "1"));
  }
  return on == 1;
}

// OCTMG_FASRHS=cell: the per-cell k_fasrhs instead of the row form
void launch_fasrhs(const SmoothArgs& a, int ninner, cudaStream_t s) {
  int cell = -1;
  if (cell < 0) {
    const char* e = getenv("OCTMG_FASRHS");
    cell = e && std::string(e) == "cell";
  }
  if (ninner <= 0) return;
  if (cell) k_fasrhs<<<ninner, NT, 0, s>>>(a);
  else k_fasrhs_row<<<ninner, 128, 0, s>>>(a);
}

template <int CPT>
static void launch_pass_cpt(const SmoothArgs& a, int mode, cudaStream_t s, bool v2, bool ghosts) {
  const int grid = a.n;
  if (CPT == 4 && v2 && pass_v3_enabled()) {  // 128-bit row form (CPT 4 = 64 threads per tile)
    switch (mode) {
      case SM_ZERO1: k_pass_v3<SM_ZERO1, 0><<<grid, 64, 0, s>>>(a); break;
      case SM_ZERO2:
        if (!pass_ghost_inline(ghosts)) k_pass_v3<SM_ZERO2, 0><<<grid, 64, 0, s>>>(a);
        else if (pass_ghost_minb() == 14) k_pass_v3<SM_ZERO2, 2><<<grid, 64, 0, s>>>(a);
        else k_pass_v3<SM_ZERO2, 1><<<grid, 64, 0, s>>>(a);
        break;
      case SM_PLAIN_RZ: k_pass_v3<SM_PLAIN_RZ, 0><<<grid, 64, 0, s>>>(a); break;  // (ghost-free levels only)
      default:
        if (!pass_ghost_inline(ghosts)) k_pass_v3<SM_PLAIN, 0><<<grid, 64, 0, s>>>(a);
        else if (pass_ghost_minb() == 14) k_pass_v3<SM_PLAIN, 2><<<grid, 64, 0, s>>>(a);
        else k_pass_v3<SM_PLAIN, 1><<<grid, 64, 0, s>>>(a);
        break;
    }
    return;
  }
  switch (mode) {
    case SM_ZERO1: k_pass_v2<SM_ZERO1, CPT><<<grid, NT / CPT, 0, s>>>(a); break;
    case SM_ZERO2: k_pass_v2<SM_ZERO2, CPT><<<grid, NT / CPT, 0, s>>>(a); break;
    default: k_pass_v2<SM_PLAIN, CPT><<<grid, NT / CPT, 0, s>>>(a); break;
  }
}

void launch_pass_direct(const SmoothArgs& a, cudaStream_t s, int cpt) {
  if (a.n == 0) return;
  const int mode = a.stage[0] >> 1;
  const bool v2 = cpt & 16, gh = cpt & 32;
  if ((cpt & 15) == 4) launch_pass_cpt<4>(a, mode, s, v2, gh);
  else if ((cpt & 15) == 2) launch_pass_cpt<2>(a, mode, s, v2, gh);
  else launch_pass_cpt<1>(a, mode, s, v2, gh);
}

void launch_restrict_direct(const SmoothArgs& a, cudaStream_t s, int v2) {
  if (!a.n) return;
  if (v2 & 64) {  // a level with ghost tiles: the row form
    k_restrict_row<<<a.n, 128, 0, s>>>(a);
    return;
  }
  if (v2 & 128) {  // a ghost-free level after a black pass: red rows only
    k_restrict_red<<<a.n, 64, 0, s>>>(a);
    return;
  }
  k_restrict_v2<6><<<a.n, NT, 0, s>>>(a);
}

void launch_prolong(const SmoothArgs& a, cudaStream_t s) {
  if (a.n) k_prolong<<<a.n, 128, 0, s>>>(a);
}

}  // namespace octmg
