// Fused red-black Gauss-Seidel iteration (sm_100a): one launch performs both colour passes
// of an RBGS iteration with ONE pass over HBM.  Each CTA stages its tile's u,
// coefficient records and right-hand side in shared memory, then
//   1. recomputes, redundantly, the first-colour values of the face layers of its same-level
//      neighbour tiles (the only cross-tile inputs of its second-colour cells) with the
//      generic stencil on the neighbour tile (same arithmetic, so bit-identical to what the
//      neighbour's own CTA computes),
//   2. updates its first-colour cells (in-tile inputs from shared memory, cross-tile inputs
//      are second-colour cells of other tiles, unchanged),
//   3. updates its second-colour cells from the new first-colour values,
//   4. writes the whole tile to the other buffer of a ping-pong pair (u_old is never written,
//      so cross-CTA reads are race-free).
// Ghost values use the snapshot of the pass they belong to (SURVEY c-5): old values in
// step 2 and step 1, (new first colour, old second colour) in step 3.
#include "stencil.cuh"

namespace octmg {

namespace {

constexpr int NT = 256;

struct RBSmem {
  float u[TB3];
  float4 c4[TB3];
  float b[TB3];
  float shell[6][64];
  int nb[6];
  int4 tv;
};

// face-layer index (p + 8q) of cell (x,y,z) on a face of axis ax
__device__ __forceinline__ int face_idx(int ax, int x, int y, int z) {
  return ax == 0 ? y + 8 * z : (ax == 1 ? x + 8 * z : x + 8 * y);
}

// sum of the six face terms of own cell (x,y,z), starting from s0; in-tile values from
// S.u, cross-tile values from `shell` (second-colour step) or from global u_old
template <bool ZERO>
__device__ __forceinline__ float fsum_tile(const SmoothArgs& a, const RBSmem& S, int t, int x, int y, int z,
                                           const float4& q, bool use_shell, float ui, float mP, float s0) {
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
      v = S.u[no];
      if (f & 1) cf = comp(S.c4[no], ax);
    } else {
      const int n = S.nb[f];
      nc[ax] &= 7;
      if (n >= 0) {
        const int no = loff(nc[0], nc[1], nc[2]);
        if (use_shell) v = S.shell[f][face_idx(ax, nc[0], nc[1], nc[2])];
        else v = ZERO ? 0.0f : __ldg(tptr(a.u, n, a.NL) + no);
        if (f & 1) cf = comp(ldcoef(a.coef, (size_t)n * TB3 + no), ax);
      } else if (n <= -2) {
        if (f & 1) cf = __ldg(a.glayer_val + (size_t)__ldg(a.glayer + 3 * t + ax) * 64 + face_idx(ax, x, y, z));
        const int C = -2 - n;
        int g[3] = {S.tv.y * 8 + c[0], S.tv.z * 8 + c[1], S.tv.w * 8 + c[2]};
        g[ax] += sg;
        const int co = loff((g[0] >> 1) & 7, (g[1] >> 1) & 7, (g[2] >> 1) & 7);
        if (ldcoef(a.coef, (size_t)C * TB3 + co).x != 0.0f) {
          const float uc = ZERO ? 0.0f : __ldg(tptr(a.uc, C, a.NL) + co);
          v = ui + 0.5f * (uc - mP);
        }
      }
    }
    s = fmaf(cf, v, s);
  }
  return s;
}

__device__ __forceinline__ float smem_block_mean(const RBSmem& S, int x, int y, int z) {
  float sm = 0.0f;
  int nn = 0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx) {
        const int bo = loff((x & ~1) + dx, (y & ~1) + dy, (z & ~1) + dz);
        if (S.c4[bo].x != 0.0f) { sm += S.u[bo]; nn++; }
      }
  return nn ? sm / (float)nn : 0.0f;
}

template <bool ZERO, bool SHELL>
__global__ __launch_bounds__(NT, 6) void k_rb_fused(SmoothArgs a) {
  __shared__ __align__(16) RBSmem S;
  const int t = a.order[blockIdx.x];
  const int c0 = a.stage[0] & 1;  // colour of the first pass
  const int j = threadIdx.x;
  const int y = (j >> 2) & 7, z = j >> 5, x0 = 2 * (j & 3);
  const int off0 = loff(x0, y, z);
  const size_t base = (size_t)t * TB3;
  // 1. stage the tile
  if (j < 6) S.nb[j] = __ldg(a.nbr + 6 * t + j);
  if (j == 6) S.tv = __ldg(a.tile + t);
  {
    const float2 uu = ZERO ? make_float2(0.f, 0.f) : __ldg(reinterpret_cast<const float2*>(tptr(a.u, t, a.NL) + off0));
    const float2 bb = __ldg(reinterpret_cast<const float2*>(tptr(a.b, t, a.NL) + off0));
    S.u[off0] = uu.x; S.u[off0 + 1] = uu.y;
    S.b[off0] = bb.x; S.b[off0 + 1] = bb.y;
    S.c4[off0] = ldcoef(a.coef, base + off0);
    S.c4[off0 + 1] = ldcoef(a.coef, base + off0 + 1);
  }
  __syncthreads();
  // 2. first-colour values of the neighbours' face layers (32 of the 64 cells per face)
  if (SHELL && j < 192) {
    const int f = j >> 5, k = j & 31;
    const int n = S.nb[f];
    if (n >= 0) {
      const int ax = f >> 1;
      const int lay = (f & 1) ? 0 : 7;           // the neighbour's layer that touches us
      const int q = k >> 2;                      // second face coordinate
      const int pp = 2 * (k & 3);
      // first face coordinate p chosen so the cell has colour c0
      int cc[3];
      int p = pp;
      {
        int tmp[3];
        tmp[ax] = lay;
        const int o1 = ax == 0 ? 1 : 0, o2 = ax == 2 ? 1 : 2;
        tmp[o1] = p; tmp[o2] = q;
        if (((tmp[0] + tmp[1] + tmp[2]) & 1) != c0) p += 1;
        tmp[o1] = p;
        cc[0] = tmp[0]; cc[1] = tmp[1]; cc[2] = tmp[2];
      }
      const int no = loff(cc[0], cc[1], cc[2]);
      const float4 qn = ldcoef(a.coef, (size_t)n * TB3 + no);
      float v = 0.0f;
      if (qn.x != 0.0f) {
        const float bn = __ldg(tptr(a.b, n, a.NL) + no);
        if (ZERO) {
          v = bn / qn.x;
        } else {
          float ui = 0.0f, mP = 0.0f;
          if (has_ghost(a, n)) {
            ui = __ldg(tptr(a.u, n, a.NL) + no);
            mP = block_mean<false, true>(a, n, cc[0], cc[1], cc[2], c0);
          }
          v = (bn - face_sum<false, true>(a, n, cc[0], cc[1], cc[2], qn, ui, mP, c0, 0.0f)) / qn.x;
        }
      }
      S.shell[f][face_idx(ax, cc[0], cc[1], cc[2])] = v;
    }
  }
  // 3. own first-colour cells (snapshot: all old values)
  const bool ghost = S.nb[0] <= -2 || S.nb[1] <= -2 || S.nb[2] <= -2 || S.nb[3] <= -2 || S.nb[4] <= -2 ||
                     S.nb[5] <= -2;
  const int sel1 = (c0 + y + z) & 1;  // which of the thread's two cells has colour c0
  const int x1 = x0 + sel1, xo = x0 + (sel1 ^ 1);
  const int o1 = off0 + sel1, oo = off0 + (sel1 ^ 1);
  float v1 = S.u[o1];
  {
    const float4 q = S.c4[o1];
    if (q.x != 0.0f) {
      if (ZERO) {
        v1 = S.b[o1] / q.x;
      } else {
        const float mP = ghost ? smem_block_mean(S, x1, y, z) : 0.0f;
        v1 = (S.b[o1] - fsum_tile<ZERO>(a, S, t, x1, y, z, q, false, S.u[o1], mP, 0.0f)) / q.x;
      }
    }
  }
  __syncthreads();  // first-colour reads done, shell complete
  S.u[o1] = v1;
  __syncthreads();
  // 4. own second-colour cells (snapshot: new first colour, old second colour)
  float v2 = S.u[oo];
  {
    const float4 q = S.c4[oo];
    if (q.x != 0.0f) {
      const float mP = ghost ? smem_block_mean(S, xo, y, z) : 0.0f;
      v2 = (S.b[oo] - fsum_tile<ZERO>(a, S, t, xo, y, z, q, true, S.u[oo], mP, 0.0f)) / q.x;
    } else if (ZERO) {
      v2 = 0.0f;
    }
  }
  // 5. whole tile to the other buffer (inactive cells keep 0)
  float2 out;
  out.x = sel1 ? v2 : v1;
  out.y = sel1 ? v1 : v2;
  *reinterpret_cast<float2*>(tptr(a.u2, t, a.NL) + off0) = out;
}

}  // namespace

void launch_rb_fused(const SmoothArgs& a, bool zero, cudaStream_t s, bool shell) {
  if (a.n == 0) return;
  if (!shell) {  // timing experiment only (OCTMG_RB=fused_noshell): wrong results
    k_rb_fused<false, false><<<a.n, NT, 0, s>>>(a);
    return;
  }
  if (zero) k_rb_fused<true, true><<<a.n, NT, 0, s>>>(a);
  else k_rb_fused<false, true><<<a.n, NT, 0, s>>>(a);
}

// copy a level's tiles from one buffer to the other (odd smoothing counts)
__global__ void k_copy_level(SmoothArgs a) {
  const int t = a.order[blockIdx.x];
  const int j = threadIdx.x;  // 128 threads x float4
  reinterpret_cast<float4*>(tptr(a.u2, t, a.NL))[j] = reinterpret_cast<const float4*>(tptr(a.u, t, a.NL))[j];
}

void launch_copy_level(const SmoothArgs& a, cudaStream_t s) {
  if (a.n) k_copy_level<<<a.n, 128, 0, s>>>(a);
}

}  // namespace octmg
