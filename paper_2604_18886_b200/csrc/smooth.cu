// Smoother stage kernel (sm_100a): one launch = one stage over all tiles of a level — a
// red-black Gauss-Seidel colour pass done IN PLACE, or the fused residual +
// restriction + Avg of Alg. 4 lines 8-9 ("fused into one kernel").
// An in-place colour-c pass is race-free: it reads only colour-(1-c) cells of other tiles
// (the face neighbours of its colour-c cells) and its own tile, and writes only its own
// colour-c cells; ghost values use the pass-start snapshot of the own tile (SURVEY c-5).
//
// Each CTA walks a contiguous run of tiles of the level in slab-major rank order (z, then
// Morton of (x, y), so consecutive tiles share faces) with a two-deep software pipeline:
// while tile i is computed, TMA bulk copies (cp.async.bulk + mbarrier) bring tile i+1's
// u (2 KB), coefficient record (8 KB) and right-hand side (2 KB) into the other shared
// buffer, and its face halos / ghost sources / prolongation parents are loaded into
// registers.  The run length is sized so the grid is one wave of resident CTAs.
#include "octmg_internal.cuh"

namespace octmg {

// stage descriptor: bit0 colour, bits 1..3 mode
enum { SM_PLAIN = 0, SM_ZERO1 = 1, SM_ZERO2 = 2, SM_PRO1 = 3, SM_PRO2 = 4, SM_RESTRICT = 5 };

namespace {

constexpr int NT = 256;

__device__ __forceinline__ int su_idx(int x, int y, int z) { return (z + 1) * 100 + (y + 1) * 10 + (x + 1); }
__device__ __forceinline__ int loff(int x, int y, int z) { return x + 8 * y + 64 * z; }
__device__ __forceinline__ float comp(const float4& v, int a) { return a == 0 ? v.y : (a == 1 ? v.z : v.w); }
__device__ __forceinline__ int pcell_of(int4 tv, int x, int y, int z) {
  return loff(((tv.y & 1) << 2) + (x >> 1), ((tv.z & 1) << 2) + (y >> 1), ((tv.w & 1) << 2) + (z >> 1));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}

struct Meta {
  int4 tv;
  int nb[6];
  int par;
  int4 ntv[6];   // neighbour tile coords (PROLONG1 halo correction)
  int npar[6];   // neighbour parents
  int gl[3];     // ghost layers of the +x/+y/+z faces
};

struct Smem {
  float4 coef[2][512];
  float b[2][512];
  float ub[2][512];  // own u (bulk copy)
  float u[1000];     // own u + halo, the pass-start snapshot
  float cp[3][64];   // +face coefficients of the neighbour layer (x+, y+, z+)
  float r[512];      // residual (restrict stage)
  Meta meta[3];
  uint64_t bar[2];
};

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

__device__ __forceinline__ float cxm_at(const Smem& S, int buf, int x, int y, int z) {
  return x < 8 ? S.coef[buf][loff(x, y, z)].y : S.cp[0][y + 8 * z];
}
__device__ __forceinline__ float cym_at(const Smem& S, int buf, int x, int y, int z) {
  return y < 8 ? S.coef[buf][loff(x, y, z)].z : S.cp[1][x + 8 * z];
}
__device__ __forceinline__ float czm_at(const Smem& S, int buf, int x, int y, int z) {
  return z < 8 ? S.coef[buf][loff(x, y, z)].w : S.cp[2][x + 8 * y];
}

// sum of the six face terms in the oracle's order x-, x+, y-, y+, z-, z+, starting from s0
__device__ __forceinline__ float faces(const Smem& S, int buf, int x, int y, int z, float s0) {
  int iu = su_idx(x, y, z);
  const float4 me = S.coef[buf][loff(x, y, z)];
  float s = s0;
  s = fmaf(me.y, S.u[iu - 1], s);
  s = fmaf(cxm_at(S, buf, x + 1, y, z), S.u[iu + 1], s);
  s = fmaf(me.z, S.u[iu - 10], s);
  s = fmaf(cym_at(S, buf, x, y + 1, z), S.u[iu + 10], s);
  s = fmaf(me.w, S.u[iu - 100], s);
  s = fmaf(czm_at(S, buf, x, y, z + 1), S.u[iu + 100], s);
  return s;
}

__device__ __forceinline__ float block_mean(const Smem& S, int buf, const int o[3]) {
  int bx = o[0] & ~1, by = o[1] & ~1, bz = o[2] & ~1;
  float s = 0.0f;
  int n = 0;
  for (int dz = 0; dz < 2; ++dz)
    for (int dy = 0; dy < 2; ++dy)
      for (int dx = 0; dx < 2; ++dx)
        if (S.coef[buf][loff(bx + dx, by + dy, bz + dz)].x != 0.0f) {
          s += S.u[su_idx(bx + dx, by + dy, bz + dz)];
          n++;
        }
  return n ? s / (float)n : 0.0f;
}

__device__ __forceinline__ void load_meta(Meta& m, const SmoothArgs& a, int t, bool prolong) {
  // executed by threads 0..7 of warp 1
  int k = threadIdx.x - 32;
  if (k < 6) {
    int n = a.nbr[6 * t + k];
    m.nb[k] = n;
    if (prolong && n >= 0) { m.ntv[k] = a.tile[n]; m.npar[k] = a.parent[n]; }
  } else if (k == 6) {
    m.tv = a.tile[t];
    m.par = a.parent[t];
  } else if (k == 7) {
    if (t < a.NL) {
      m.gl[0] = a.glayer[3 * t]; m.gl[1] = a.glayer[3 * t + 1]; m.gl[2] = a.glayer[3 * t + 2];
    } else {
      m.gl[0] = m.gl[1] = m.gl[2] = -1;
    }
  }
}

__device__ __forceinline__ void issue_tile(Smem& S, int buf, const SmoothArgs& a, int t, bool with_u) {
  // one elected thread: coefficient record (8 KB) + right-hand side (2 KB) + u (2 KB)
  mbar_expect_tx(&S.bar[buf], TB3 * 16 + TB3 * 4 + (with_u ? TB3 * 4 : 0));
  bulk_g2s(&S.coef[buf][0], a.coef + (size_t)t * TB3, TB3 * 16, &S.bar[buf]);
  bulk_g2s(&S.b[buf][0], tptr(a.b, t, a.NL), TB3 * 4, &S.bar[buf]);
  if (with_u) bulk_g2s(&S.ub[buf][0], tptr(a.u, t, a.NL), TB3 * 4, &S.bar[buf]);
}

// halo sources of one tile held in registers between prefetch and staging
struct Halo {
  float v[2], c[2], uc[2];
  int kind[2];  // 0 zero, 1 value, 2 ghost (uc = coarse value)
  float corr;   // prolongation correction of the thread's own cells
};

__device__ __forceinline__ void load_halo(Halo& H, const Meta& M, const SmoothArgs& a, int mode) {
  const int tid = threadIdx.x;
  const int x2 = tid & 3, y = (tid >> 2) & 7, z = tid >> 5, x0 = 2 * x2;
  H.corr = 0.0f;
  if (mode == SM_PRO1 || mode == SM_PRO2) {
    int pc = pcell_of(M.tv, x0, y, z);
    H.corr = __ldcg(tptr(a.u, M.par, a.NL) + pc) - a.ustar[(size_t)(M.par - a.NL) * TB3 + pc];
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    H.v[k] = 0.0f; H.c[k] = 0.0f; H.uc[k] = 0.0f; H.kind[k] = 0;
    int w = tid + k * NT;
    if (w >= 384) break;
    int f = w >> 6, p = w & 7, q = (w >> 3) & 7;
    int own[3], src[3], halo[3];
    face_cells(f, p, q, own, src, halo);
    int n = M.nb[f];
    if (n >= 0) {
      int so = loff(src[0], src[1], src[2]);
      if (mode != SM_ZERO1) {
        H.v[k] = __ldcg(tptr(a.u, n, a.NL) + so);
        H.kind[k] = 1;
      }
      if ((f & 1) || mode == SM_PRO1) {
        float4 r = a.coef[(size_t)n * TB3 + so];
        H.c[k] = comp(r, f >> 1);
        if (mode == SM_PRO1 && r.x != 0.0f) {
          int P = M.npar[f];
          int pc = pcell_of(M.ntv[f], src[0], src[1], src[2]);
          H.v[k] += __ldcg(tptr(a.u, P, a.NL) + pc) - a.ustar[(size_t)(P - a.NL) * TB3 + pc];
        }
      }
    } else if (n <= -2) {
      int C = -2 - n;
      int g0 = M.tv.y * 8 + halo[0], g1 = M.tv.z * 8 + halo[1], g2 = M.tv.w * 8 + halo[2];
      int co = loff((g0 >> 1) & 7, (g1 >> 1) & 7, (g2 >> 1) & 7);
      if (mode != SM_ZERO1 && a.coef[(size_t)C * TB3 + co].x != 0.0f) {
        H.uc[k] = __ldcg(tptr(a.u, C, a.NL) + co);
        H.kind[k] = 2;
      }
      if (f & 1) H.c[k] = a.glayer_val[(size_t)M.gl[f >> 1] * 64 + p + 8 * q];
    }
  }
}

}  // namespace

__global__ __launch_bounds__(NT, 7) void k_stage(SmoothArgs a) {
  __shared__ __align__(128) Smem S;
  const int tid = threadIdx.x;
  const int x2 = tid & 3, y = (tid >> 2) & 7, z = tid >> 5, x0 = 2 * x2;
  const int off0 = loff(x0, y, z);
  const int desc = a.stage[0];
  const int colour = desc & 1, mode = desc >> 1;
  const bool pro = mode == SM_PRO1;
  const int r0 = blockIdx.x * a.run;
  const int r1 = min(a.n, r0 + a.run);
  if (r0 >= r1) return;
  if (tid == 0) {
    mbar_init(&S.bar[0]);
    mbar_init(&S.bar[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    issue_tile(S, 0, a, a.order[r0], mode != SM_ZERO1);
  }
  if (tid >= 32 && tid < 40) {
    load_meta(S.meta[0], a, a.order[r0], pro);
    if (r0 + 1 < r1) load_meta(S.meta[1], a, a.order[r0 + 1], pro);
  }
  __syncthreads();
  Halo H, Hn;
  load_halo(H, S.meta[0], a, mode);
  uint32_t phase[2] = {0u, 0u};
  for (int i = r0; i < r1; ++i) {
    const int k = i - r0;
    const int cur = k & 1;
    const Meta& M = S.meta[k % 3];
    const int t = a.order[i];
    // (b) prefetch tile i+1 (its buffers were freed by the sync that ended tile i-1)
    if (i + 1 < r1) {
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_tile(S, cur ^ 1, a, a.order[i + 1], mode != SM_ZERO1);
      }
      load_halo(Hn, S.meta[(k + 1) % 3], a, mode);
      if (i + 2 < r1 && tid >= 32 && tid < 40) load_meta(S.meta[(k + 2) % 3], a, a.order[i + 2], pro);
    }
    // (c) own values: snapshot of this pass with the stage's transforms
    mbar_wait(&S.bar[cur], phase[cur]);
    phase[cur] ^= 1u;
    const float4 q0 = S.coef[cur][off0], q1 = S.coef[cur][off0 + 1];
    float u0 = 0.0f, u1 = 0.0f;
    if (mode != SM_ZERO1) { u0 = S.ub[cur][off0]; u1 = S.ub[cur][off0 + 1]; }
    if (mode == SM_PRO1) {
      if (q0.x != 0.0f) u0 += H.corr;
      if (q1.x != 0.0f) u1 += H.corr;
    } else if (mode == SM_PRO2 || mode == SM_ZERO2) {
      const int selc = (colour + y + z) & 1;
      float& uc = selc ? u1 : u0;
      const float qc = selc ? q1.x : q0.x;
      if (mode == SM_ZERO2) uc = 0.0f;
      else if (qc != 0.0f) uc += H.corr;
    }
    S.u[su_idx(x0, y, z)] = u0;
    S.u[su_idx(x0 + 1, y, z)] = u1;
    __syncthreads();  // own snapshot visible (ghosts need it)
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      int w = tid + kk * NT;
      if (w >= 384) break;
      int f = w >> 6, p = w & 7, q = (w >> 3) & 7;
      int own[3], src[3], halo[3];
      face_cells(f, p, q, own, src, halo);
      float v = H.v[kk];
      if (H.kind[kk] == 2) v = S.u[su_idx(own[0], own[1], own[2])] + 0.5f * (H.uc[kk] - block_mean(S, cur, own));
      else if (H.kind[kk] == 0) v = 0.0f;
      S.u[su_idx(halo[0], halo[1], halo[2])] = v;
      if (f & 1) S.cp[f >> 1][p + 8 * q] = H.c[kk];
    }
    __syncthreads();  // halo visible
    if (mode != SM_RESTRICT) {
      const int sel = (colour + y + z) & 1;
      const int xc = x0 + sel;
      const float cc = sel ? q1.x : q0.x;
      if (cc != 0.0f) {
        float bc = S.b[cur][off0 + sel];
        tptr(a.u, t, a.NL)[off0 + sel] = (bc - faces(S, cur, xc, y, z, 0.0f)) / cc;
      } else if (mode == SM_ZERO1 || mode == SM_ZERO2) {
        tptr(a.u, t, a.NL)[off0 + sel] = 0.0f;  // memory may hold a previous cycle's data
      }
    } else {
      // r = b - A^l u; per parent: u* = mean of active children, u^{l-1} := u*,
      // b^{l-1} := beta * (R r), R = P^T / alpha
      S.r[off0] = q0.x != 0.0f ? S.b[cur][off0] - faces(S, cur, x0, y, z, q0.x * u0) : 0.0f;
      S.r[off0 + 1] = q1.x != 0.0f ? S.b[cur][off0 + 1] - faces(S, cur, x0 + 1, y, z, q1.x * u1) : 0.0f;
      __syncthreads();
      if (tid < 64) {
        int bx = (tid & 3) * 2, by = ((tid >> 2) & 3) * 2, bz = (tid >> 4) * 2;
        float su = 0.0f, rs = 0.0f;
        int nact = 0;
        for (int dz = 0; dz < 2; ++dz)
          for (int dy = 0; dy < 2; ++dy)
            for (int dx = 0; dx < 2; ++dx) {
              int o = loff(bx + dx, by + dy, bz + dz);
              if (S.coef[cur][o].x != 0.0f) { nact++; su += S.u[su_idx(bx + dx, by + dy, bz + dz)]; rs += S.r[o]; }
            }
        float us = nact ? su / (float)nact : 0.0f;
        int P = M.par;
        int pc = pcell_of(M.tv, bx, by, bz);
        size_t pi = (size_t)(P - a.NL) * TB3 + pc;
        a.u.inner[pi] = us;
        a.ustar_w[pi] = us;
        a.b.inner[pi] = a.beta * (rs / a.alpha);
      }
    }
    H = Hn;
    __syncthreads();  // buffers of `cur`, S.u and meta slot k%3 free for reuse
  }
}

// FAS right-hand side of the inner rows of a coarse level (Alg. 4 line 10):
// b_I = beta R r (already in b) + (A^{l-1} u*)_I, u* in u (inner) and current u (leaves).
__global__ __launch_bounds__(NT) void k_fasrhs(SmoothArgs a) {
  __shared__ __align__(128) Smem S;
  const int tid = threadIdx.x;
  const int t = a.first_tile + blockIdx.x;  // inner tiles of the level (contiguous)
  const int x2 = tid & 3, y = (tid >> 2) & 7, z = tid >> 5, x0 = 2 * x2;
  const int off0 = loff(x0, y, z);
  if (tid >= 32 && tid < 40) load_meta(S.meta[0], a, t, false);
  const float4* cf = a.coef + (size_t)t * TB3;
  float4 q0 = cf[off0], q1 = cf[off0 + 1];
  S.coef[0][off0] = q0;
  S.coef[0][off0 + 1] = q1;
  float2 uu = __ldcg(reinterpret_cast<const float2*>(tptr(a.u, t, a.NL) + off0));
  S.u[su_idx(x0, y, z)] = uu.x;
  S.u[su_idx(x0 + 1, y, z)] = uu.y;
  __syncthreads();
  const Meta& M = S.meta[0];
  for (int w = tid; w < 384; w += NT) {
    int f = w >> 6, p = w & 7, q = (w >> 3) & 7;
    int own[3], src[3], halo[3];
    face_cells(f, p, q, own, src, halo);
    int n = M.nb[f];  // inner tiles never border ghosts (grading)
    float v = 0.0f, c = 0.0f;
    if (n >= 0) {
      int so = loff(src[0], src[1], src[2]);
      v = __ldcg(tptr(a.u, n, a.NL) + so);
      if (f & 1) c = comp(a.coef[(size_t)n * TB3 + so], f >> 1);
    }
    S.u[su_idx(halo[0], halo[1], halo[2])] = v;
    if (f & 1) S.cp[f >> 1][p + 8 * q] = c;
  }
  __syncthreads();
  float* bi = a.b.inner + (size_t)(t - a.NL) * TB3 + off0;
  float2 bb = *reinterpret_cast<float2*>(bi);
  float b0 = q0.x != 0.0f ? bb.x + faces(S, 0, x0, y, z, q0.x * uu.x) : 0.0f;
  float b1 = q1.x != 0.0f ? bb.y + faces(S, 0, x0 + 1, y, z, q1.x * uu.y) : 0.0f;
  *reinterpret_cast<float2*>(bi) = make_float2(b0, b1);
}

const void* smooth_kernel_ptr() { return (const void*)k_stage; }

void launch_smooth(const SmoothArgs& a, int grid, cudaStream_t s) {
  k_stage<<<grid, NT, 0, s>>>(a);
}

void launch_fasrhs(const SmoothArgs& a, int ninner, cudaStream_t s) {
  if (ninner > 0) k_fasrhs<<<ninner, NT, 0, s>>>(a);
}

}  // namespace octmg
