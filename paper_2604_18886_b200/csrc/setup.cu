// Coefficient setup: leaf assembly (Eq. 3; ghost-fluid kinds P:L318-337;
// T-junction faces Eqs. 9-10) and Galerkin coarsening (Alg. 3)
// of the compact record (c, c_x-, c_y-, c_z-) held as one float4 per cell.
#include <algorithm>
#include <vector>

#include "nbref.cuh"

namespace octmg {

namespace {

struct AsmArgs {
  const int4* tile;
  const int* nbr;
  const int* child;
  const int* glayer;
  const uint8_t* kind;
  WIn w;
  float* coef;  // SoA per tile (cidx)
  float* glayer_val;
  int NL;
  uint8_t wall[6];
};

// pass 1: diagonal of every leaf cell from geometry (SURVEY c-2)
__global__ __launch_bounds__(256) void k_assemble_diag(AsmArgs a) {
  int t = blockIdx.x;
  int4 tv = a.tile[t];
  float h = ldexpf(1.0f, -tv.x) * 0.125f;
  for (int off = threadIdx.x; off < TB3; off += blockDim.x) {
    int x, y, z;
    slot_xyz(off, x, y, z);
    size_t i = (size_t)t * TB3 + off;
    float c = 0.0f;
    if (a.kind[i] == KF) {
      for (int f = 0; f < 6; ++f) {
        NbRef nb = nb_ref(a.nbr, tv, t, a.NL, x, y, z, f);
        if (nb.what == NB_WALL) {
          if (a.wall[f]) c += a.w.w(f, i) * h;
        } else if (nb.what == NB_LEAF) {
          size_t j = (size_t)nb.tile * TB3 + nb.off;
          if (a.kind[j] != KN) c += ((f & 1) ? a.w.w(f ^ 1, j) : a.w.w(f, i)) * h;
        } else if (nb.what == NB_INNER) {
          size_t sub[4];
          fine_subs(a.child, a.NL, nb, f, sub);
          for (int k = 0; k < 4; ++k)
            if (a.kind[sub[k]] != KN) c += 0.5f * a.w.w(f ^ 1, sub[k]) * (0.5f * h);
        } else {
          size_t C = (size_t)nb.tile * TB3 + nb.off;
          if (a.kind[C] != KN) c += a.w.w(f, i) * h;
        }
      }
    }
    stcoef(a.coef, i, make_float4(c, 0.f, 0.f, 0.f));
  }
}

// pass 2: -face off-diagonals and the +face ghost-layer coefficients
__global__ __launch_bounds__(256) void k_assemble_offdiag(AsmArgs a) {
  int t = blockIdx.x;
  int4 tv = a.tile[t];
  float h = ldexpf(1.0f, -tv.x) * 0.125f;
  for (int off = threadIdx.x; off < TB3; off += blockDim.x) {
    int x, y, z;
    slot_xyz(off, x, y, z);
    size_t i = (size_t)t * TB3 + off;
    if (a.kind[i] == KN) continue;  // Neumann: all-zero record (already zero)
    float cm[3];
    for (int ax = 0; ax < 3; ++ax) {
      int f = 2 * ax;
      NbRef nb = nb_ref(a.nbr, tv, t, a.NL, x, y, z, f);
      float v = 0.0f;
      if (nb.what == NB_LEAF) {
        if (a.kind[(size_t)nb.tile * TB3 + nb.off] != KN) v = -a.w.w(f, i) * h;
      } else if (nb.what == NB_INNER) {
        size_t sub[4];
        fine_subs(a.child, a.NL, nb, f, sub);
        float acc = 0.0f;
        for (int k = 0; k < 4; ++k)
          if (a.coef[cidx(sub[k], 0)] != 0.0f) acc += a.w.w(f ^ 1, sub[k]) * (0.5f * h);
        v = -0.5f * acc;
      } else if (nb.what == NB_GHOST) {
        if (a.kind[(size_t)nb.tile * TB3 + nb.off] != KN) v = -a.w.w(f, i) * h;
      }
      cm[ax] = v;
      // +face toward a ghost: coefficient of the ghost cell's -face (c_{6,x-})
      int cc[3] = {x, y, z};
      if (cc[ax] == 7) {
        int gl = a.glayer[3 * t + ax];
        if (gl >= 0) {
          NbRef g = nb_ref(a.nbr, tv, t, a.NL, x, y, z, f + 1);
          float gv = a.kind[(size_t)g.tile * TB3 + g.off] != KN ? -a.w.w(f + 1, i) * h : 0.0f;
          int p = ax == 0 ? y + 8 * z : (ax == 1 ? x + 8 * z : x + 8 * y);
          a.glayer_val[(size_t)gl * 64 + p] = gv;
        }
      }
    }
    a.coef[cidx(i, 1)] = cm[0];
    a.coef[cidx(i, 2)] = cm[1];
    a.coef[cidx(i, 3)] = cm[2];
  }
}

// Row sums of the leaf operator as the apply evaluates it, d_i = c_i + sum_f c_f (the
// exact, fp64 diagonal of Eq. 3 plus the six stored fp32 couplings the apply uses: own -face
// entries, the +face neighbour's -face entry (same-level leaf or inner cell), the ghost
// layer toward a coarse leaf, 0 at a domain wall).  The apply evaluates the operator in
// flux form, (A p)_i = d_i p_i + sum_f c_f (v_f - p_i) (kernels.cu k_apply_v6), so its
// diagonal is the exact c_i even though the stored c is fp32, and the operator's rows sum
// exactly to d_i (0 away from Dirichlet walls).  Runs after the coarsening (the +faces of
// inner neighbours are their Alg. 3 records).  flag[t] = 1 if any d of tile t is nonzero.
__global__ __launch_bounds__(256) void k_leaf_rowsum(AsmArgs a, float* d, int* flag) {
  const int t = blockIdx.x;
  const int4 tv = a.tile[t];
  const double h = ldexp(1.0, -tv.x) * 0.125;
  int any = 0;
  for (int off = threadIdx.x; off < TB3; off += blockDim.x) {
    int x, y, z;
    slot_xyz(off, x, y, z);
    const size_t i = (size_t)t * TB3 + off;
    double dv = 0.0;
    if (a.coef[cidx(i, 0)] != 0.0f) {
      // the exact diagonal (k_assemble_diag's terms in fp64)
      double c = 0.0;
      for (int f = 0; f < 6; ++f) {
        NbRef nb = nb_ref(a.nbr, tv, t, a.NL, x, y, z, f);
        if (nb.what == NB_WALL) {
          if (a.wall[f]) c += (double)a.w.w(f, i) * h;
        } else if (nb.what == NB_LEAF) {
          size_t j = (size_t)nb.tile * TB3 + nb.off;
          if (a.kind[j] != KN) c += (double)((f & 1) ? a.w.w(f ^ 1, j) : a.w.w(f, i)) * h;
        } else if (nb.what == NB_INNER) {
          size_t sub[4];
          fine_subs(a.child, a.NL, nb, f, sub);
          for (int k = 0; k < 4; ++k)
            if (a.kind[sub[k]] != KN) c += 0.5 * (double)a.w.w(f ^ 1, sub[k]) * (0.5 * h);
        } else {
          size_t C = (size_t)nb.tile * TB3 + nb.off;
          if (a.kind[C] != KN) c += (double)a.w.w(f, i) * h;
        }
      }
      // + the couplings the apply uses
      for (int f = 0; f < 6; ++f) {
        const int ax = f >> 1;
        if (!(f & 1)) {
          c += (double)a.coef[cidx(i, 1 + ax)];
          continue;
        }
        NbRef nb = nb_ref(a.nbr, tv, t, a.NL, x, y, z, f);
        if (nb.what == NB_LEAF || nb.what == NB_INNER) {
          c += (double)a.coef[cidx((size_t)nb.tile * TB3 + nb.off, 1 + ax)];
        } else if (nb.what == NB_GHOST) {
          const int p = ax == 0 ? y + 8 * z : (ax == 1 ? x + 8 * z : x + 8 * y);
          c += (double)a.glayer_val[(size_t)a.glayer[3 * t + ax] * 64 + p];
        }
      }
      dv = c;
    }
    d[i] = (float)dv;
    any |= (float)dv != 0.0f;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) flag[t] = any;
}

__global__ void k_compact_rowsum(const float* d, const int* dtile, int NL, float* dval) {
  const int t = blockIdx.x;
  const int k = dtile[t];
  if (k < 0) return;
  for (int o = threadIdx.x; o < TB3; o += blockDim.x) dval[(size_t)k * TB3 + o] = d[(size_t)t * TB3 + o];
}

struct CoarsenArgs {
  const int4* tile;
  const int* nbr;
  const int* child;
  float* coef;  // SoA per tile (cidx)
  int NL;
  int toff;  // first inner tile of level l-1
  float alpha;
  int literal;  // Alg. 3 as printed: no activity test on the non-diagonal branch
};

__device__ __forceinline__ float comp(const float4& v, int a) { return a == 0 ? v.y : (a == 1 ? v.z : v.w); }

// Alg. 3 with the activity test on the off-diagonal branch (SURVEY c-3)
__global__ __launch_bounds__(256) void k_coarsen(CoarsenArgs a) {
  int P = a.toff + blockIdx.x;
  const int* ch8 = a.child + 8 * (P - a.NL);
  for (int off = threadIdx.x; off < TB3; off += blockDim.x) {
    int x, y, z;
    slot_xyz(off, x, y, z);
    int ct = ch8[(x >> 2) + 2 * (y >> 2) + 4 * (z >> 2)];
    int4 ctv = a.tile[ct];
    float cI = 0.0f, cIm[3] = {0.f, 0.f, 0.f};
    int cnt = 0;
    for (int dz = 0; dz < 2; ++dz)
      for (int dy = 0; dy < 2; ++dy)
        for (int dx = 0; dx < 2; ++dx) {
          int d[3] = {dx, dy, dz};
          int cx[3] = {(2 * x + dx) & 7, (2 * y + dy) & 7, (2 * z + dz) & 7};
          float4 ci = rdcoef(a.coef, (size_t)ct * TB3 + loff(cx[0], cx[1], cx[2]));
          bool act = ci.x != 0.0f;
          if (act) { cnt++; cI += ci.x / a.alpha; }
          for (int ax = 0; ax < 3; ++ax) {
            if (d[ax] == 1) {
              int sx[3] = {cx[0], cx[1], cx[2]};
              sx[ax] -= 1;
              bool sact = a.coef[cidx((size_t)ct * TB3 + loff(sx[0], sx[1], sx[2]), 0)] != 0.0f;
              if (act && sact) cI += (2.0f / a.alpha) * comp(ci, ax);
            } else {
              NbRef nb = nb_ref(a.nbr, ctv, ct, a.NL, cx[0], cx[1], cx[2], 2 * ax);
              bool nact = nb.what != NB_WALL && a.coef[cidx((size_t)nb.tile * TB3 + nb.off, 0)] != 0.0f;
              if (a.literal || (act && nact)) cIm[ax] += comp(ci, ax) / a.alpha;
            }
          }
        }
    stcoef(a.coef, (size_t)P * TB3 + off, make_float4(cnt ? cI : 0.0f, cIm[0], cIm[1], cIm[2]));
  }
}

__global__ void k_count_active(const float* coef, int64_t n, unsigned long long* cnt) {
  unsigned long long c = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    c += coef[cidx(i, 0)] != 0.0f;
  for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

__global__ void k_any_dirichlet(const uint8_t* kind, int64_t n, int* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (kind[i] == KD) { *flag = 1; return; }
}

// GMG comparison mode: the cycle's coarse records "given directly by the grid
// discretization" — Eq. 3 (kinds P:L318-335) on every inner cell at its
// own level, from its own kind / face weights and those of its same-level neighbours (an
// inner tile never borders a ghost), in place of Alg. 3.  Written into the cycle's copy of
// the store; the leaf records (the composite operator) are untouched.  Same fp32 terms and
// order as k_assemble_diag / offdiag.
struct GmgArgs {
  const int4* tile;
  const int* nbr;
  const uint8_t* kind;    // leaf cells (slot order)
  WIn w;
  const uint8_t* kind_i;  // inner cells (slot order)
  WIn wi;
  float* coef;            // the cycle's store
  int NL;
  uint8_t wall[6];
};
__global__ __launch_bounds__(256) void k_gmg_inner(GmgArgs a) {
  const int t = a.NL + blockIdx.x;
  const int4 tv = a.tile[t];
  const float h = ldexpf(1.0f, -tv.x) * 0.125f;
  const size_t NL3 = (size_t)a.NL * TB3;
  auto kind_of = [&](size_t j) -> int { return j < NL3 ? a.kind[j] : a.kind_i[j - NL3]; };
  auto w_of = [&](int f, size_t j) -> float { return j < NL3 ? a.w.w(f, j) : a.wi.w(f, j - NL3); };
  for (int off = threadIdx.x; off < TB3; off += blockDim.x) {
    int x, y, z;
    slot_xyz(off, x, y, z);
    const size_t i = (size_t)t * TB3 + off;
    const int k = kind_of(i);
    float c = 0.0f, cm[3] = {0.0f, 0.0f, 0.0f};
    if (k != KN) {
      for (int f = 0; f < 6; ++f) {
        const NbRef nb = nb_ref(a.nbr, tv, t, a.NL, x, y, z, f);
        if (nb.what == NB_WALL) {
          if (k == KF && a.wall[f]) c += w_of(f, i) * h;
        } else if (nb.what == NB_LEAF || nb.what == NB_INNER) {
          const size_t j = (size_t)nb.tile * TB3 + nb.off;
          if (kind_of(j) != KN) {
            if (k == KF) c += ((f & 1) ? w_of(f ^ 1, j) : w_of(f, i)) * h;
            if (!(f & 1)) cm[f >> 1] = -w_of(f, i) * h;
          }
        }
      }
    }
    stcoef(a.coef, i, make_float4(c, cm[0], cm[1], cm[2]));
  }
}

}  // namespace

octmg_status assemble_leaf_coefs(Hier& h, const uint8_t* kind, const float* fbeta, const float* ffrac,
                                 cudaStream_t s) {
  Tree& T = *h.tree;
  const int64_t Nc = (int64_t)T.NL * TB3;
  // the caller's per-cell inputs (natural cell order) -> slot order, in temporaries
  uint8_t* kind_s = nullptr;
  float* beta_s = nullptr;
  float* frac_s = nullptr;
  OCTMG_CUDA(cudaMallocAsync(&kind_s, std::max<int64_t>(Nc, 1), s));
  launch_permute_u8(kind, kind_s, Nc, true, s);
  if (fbeta) {
    OCTMG_CUDA(cudaMallocAsync(&beta_s, sizeof(float) * 6 * std::max<int64_t>(Nc, 1), s));
    launch_permute_f32(fbeta, beta_s, Nc, 6, true, s);
  }
  if (ffrac) {
    OCTMG_CUDA(cudaMallocAsync(&frac_s, sizeof(float) * 6 * std::max<int64_t>(Nc, 1), s));
    launch_permute_f32(ffrac, frac_s, Nc, 6, true, s);
  }
  kind = kind_s;
  AsmArgs a;
  a.tile = T.tile;
  a.nbr = T.nbr;
  a.child = T.child;
  a.glayer = T.glayer;
  a.kind = kind;
  a.w = WIn{beta_s, frac_s, (size_t)T.NL * TB3};
  a.coef = h.coef;
  a.glayer_val = h.glayer_val;
  a.NL = T.NL;
  for (int f = 0; f < 6; ++f) a.wall[f] = T.wall[f];
  if (T.n_glayers) OCTMG_CUDA(cudaMemsetAsync(h.glayer_val, 0, (size_t)T.n_glayers * 64 * sizeof(float), s));
  k_assemble_diag<<<T.NL, 256, 0, s>>>(a);
  k_assemble_offdiag<<<T.NL, 256, 0, s>>>(a);
  OCTMG_CUDA(cudaGetLastError());
  OCTMG_TRY(coarsen_all(h, s));  // Alg. 3 (the +face records of inner neighbours feed the row sums)
  {
    // leaf row sums d (flux-form apply), kept for the tiles where some d != 0
    float* dfull = nullptr;
    int* dflag = nullptr;
    OCTMG_CUDA(cudaMallocAsync(&dfull, sizeof(float) * std::max<int64_t>(Nc, 1), s));
    OCTMG_CUDA(cudaMallocAsync(&dflag, sizeof(int) * std::max(T.NL, 1), s));
    if (T.NL) k_leaf_rowsum<<<T.NL, 256, 0, s>>>(a, dfull, dflag);
    OCTMG_CUDA(cudaGetLastError());
    std::vector<int> fl(T.NL);
    if (T.NL) OCTMG_CUDA(cudaMemcpyAsync(fl.data(), dflag, sizeof(int) * T.NL, cudaMemcpyDeviceToHost, s));
    OCTMG_CUDA(cudaStreamSynchronize(s));
    int nd = 0;
    for (int t = 0; t < T.NL; ++t) fl[t] = fl[t] ? nd++ : -1;
    OCTMG_CUDA(cudaMemcpyAsync(dflag, fl.data(), sizeof(int) * T.NL, cudaMemcpyHostToDevice, s));
    h.dtile = (int*)dev_malloc(sizeof(int) * std::max(T.NL, 1));
    h.dval = (float*)dev_malloc(sizeof(float) * (size_t)std::max(nd, 1) * TB3);
    if (!h.dtile || !h.dval) {
      set_error("device allocation failed (leaf row sums)");
      return OCTMG_E_OOM;
    }
    h.allocs.push_back(h.dtile);
    h.allocs.push_back(h.dval);
    h.n_dtiles = nd;
    OCTMG_CUDA(cudaMemcpyAsync(h.dtile, dflag, sizeof(int) * T.NL, cudaMemcpyDeviceToDevice, s));
    if (T.NL) k_compact_rowsum<<<T.NL, 128, 0, s>>>(dfull, dflag, T.NL, h.dval);
    OCTMG_CUDA(cudaGetLastError());
    OCTMG_CUDA(cudaFreeAsync(dfull, s));
    OCTMG_CUDA(cudaFreeAsync(dflag, s));
  }
  h.ccoef = h.coef;
  if (h.gmg_kind && T.NI > 0) {
    // GMG comparison mode: the cycle's own store, inner records from the grid
    const int64_t Ni = (int64_t)T.NI * TB3;
    float* cc = (float*)dev_malloc(sizeof(float) * (size_t)T.T * TB3 * 4);
    if (!cc) { set_error("device allocation failed (GMG cycle coefficients)"); return OCTMG_E_OOM; }
    h.allocs.push_back(cc);
    OCTMG_CUDA(cudaMemcpyAsync(cc, h.coef, sizeof(float) * (size_t)T.T * TB3 * 4, cudaMemcpyDeviceToDevice, s));
    uint8_t* ki = nullptr;
    float *bi = nullptr, *fi = nullptr;
    OCTMG_CUDA(cudaMallocAsync(&ki, Ni, s));
    launch_permute_u8(h.gmg_kind, ki, Ni, true, s);
    if (h.gmg_beta) {
      OCTMG_CUDA(cudaMallocAsync(&bi, sizeof(float) * 6 * Ni, s));
      launch_permute_f32(h.gmg_beta, bi, Ni, 6, true, s);
    }
    if (h.gmg_frac) {
      OCTMG_CUDA(cudaMallocAsync(&fi, sizeof(float) * 6 * Ni, s));
      launch_permute_f32(h.gmg_frac, fi, Ni, 6, true, s);
    }
    GmgArgs g;
    g.tile = T.tile;
    g.nbr = T.nbr;
    g.kind = kind;
    g.w = a.w;
    g.kind_i = ki;
    g.wi = WIn{bi, fi, (size_t)Ni};
    g.coef = cc;
    g.NL = T.NL;
    for (int f = 0; f < 6; ++f) g.wall[f] = T.wall[f];
    k_gmg_inner<<<T.NI, 256, 0, s>>>(g);
    OCTMG_CUDA(cudaGetLastError());
    OCTMG_CUDA(cudaFreeAsync(ki, s));
    if (bi) OCTMG_CUDA(cudaFreeAsync(bi, s));
    if (fi) OCTMG_CUDA(cudaFreeAsync(fi, s));
    h.ccoef = cc;
  }
  // active leaf-cell count and whether any Dirichlet kind exists (null-space auto)
  unsigned long long* d_cnt;
  int* d_flag;
  OCTMG_CUDA(cudaMallocAsync(&d_cnt, sizeof(unsigned long long) + sizeof(int) * 2, s));
  d_flag = (int*)(d_cnt + 1);
  OCTMG_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) + sizeof(int) * 2, s));
  int64_t N = (int64_t)T.NL * TB3;
  k_count_active<<<592, 256, 0, s>>>(h.coef, N, d_cnt);
  k_any_dirichlet<<<592, 256, 0, s>>>(kind, N, d_flag);
  unsigned long long cnt = 0;
  int flag = 0;
  OCTMG_CUDA(cudaMemcpyAsync(&cnt, d_cnt, sizeof(cnt), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaMemcpyAsync(&flag, d_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  OCTMG_CUDA(cudaFreeAsync(d_cnt, s));
  OCTMG_CUDA(cudaFreeAsync(kind_s, s));
  if (beta_s) OCTMG_CUDA(cudaFreeAsync(beta_s, s));
  if (frac_s) OCTMG_CUDA(cudaFreeAsync(frac_s, s));
  OCTMG_CUDA(cudaStreamSynchronize(s));
  h.n_active = (double)cnt;
  int wall_d = 0;
  for (int f = 0; f < 6; ++f) wall_d |= T.wall[f];
  h.any_dirichlet = flag || wall_d;
  return OCTMG_OK;
}

octmg_status coarsen_all(Hier& h, cudaStream_t s) {
  Tree& T = *h.tree;
  for (int l = T.L; l >= 1; --l) {
    int lc = l - 1;
    if (T.ic[lc] == 0) continue;
    CoarsenArgs a{T.tile, T.nbr, T.child, h.coef, T.NL, T.ib[lc], h.prm.alpha, h.prm.coarsen_literal};
    k_coarsen<<<T.ic[lc], 256, 0, s>>>(a);
  }
  OCTMG_CUDA(cudaGetLastError());
  return OCTMG_OK;
}

}  // namespace octmg
