// C-ABI entry points (include/octmg.h), hierarchy management, the unrolled mu-cycle
// schedule (captured once into a CUDA graph) and the PCG driver (Alg. 1).
#include <mutex>
#include <cstddef>
#include <cmath>
#include <unordered_map>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <nvtx3/nvToolsExt.h>

#include "comm.h"
#include "octmg_internal.cuh"
#include "partition.h"

namespace octmg {

static thread_local std::string g_err = "no error";

void set_error(const std::string& msg) { g_err = msg; }

octmg_status cuda_status(cudaError_t e, const char* what) {
  cudaGetLastError();
  g_err = std::string("CUDA error ") + cudaGetErrorString(e) + " in " + what;
  return e == cudaErrorMemoryAllocation ? OCTMG_E_OOM : OCTMG_E_CUDA;
}

const char* kclass_name[KC_COUNT] = {"rbgs_pass", "prolong", "residual_restrict", "coarsest",
                                     "fas_rhs", "coarse_levels", "apply", "pcg_update", "dot_rz", "project",
                                     "init", "setup", "memset", "coarse_subcycle", "rbgs_fused_iteration",
                                     "copy_level", "coarse_grid", "p_update"};

// ------------------------------------------------------------------------------------
// allocator hook (octmg_set_allocator)
// ------------------------------------------------------------------------------------
namespace {
struct Allocator {
  octmg_alloc_fn alloc = nullptr;
  octmg_free_fn release = nullptr;
  void* ctx = nullptr;
};
std::mutex g_alloc_mu;
Allocator g_alloc;                                  // current (nullptr: cudaMalloc)
std::unordered_map<void*, Allocator> g_alloc_owner;  // who made each live pointer
}  // namespace

void* dev_malloc(size_t bytes) {
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  void* q = nullptr;
  if (g_alloc.alloc) {
    q = g_alloc.alloc(bytes, nullptr, g_alloc.ctx);
  } else if (cudaMalloc(&q, bytes) != cudaSuccess) {
    cudaGetLastError();
    q = nullptr;
  }
  if (q) g_alloc_owner[q] = g_alloc;
  return q;
}

void dev_free(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  auto it = g_alloc_owner.find(p);
  Allocator a = it == g_alloc_owner.end() ? Allocator{} : it->second;
  if (it != g_alloc_owner.end()) g_alloc_owner.erase(it);
  if (a.release) a.release(p, nullptr, a.ctx);
  else cudaFree(p);
}

template <class T>
static octmg_status halloc(std::vector<void*>& list, T** p, size_t count) {
  if (count == 0) count = 1;
  void* q = dev_malloc(count * sizeof(T));
  if (!q) {
    set_error("device allocation failed (" + std::to_string(count * sizeof(T)) + " bytes)");
    return OCTMG_E_OOM;
  }
  list.push_back(q);
  *p = (T*)q;
  return OCTMG_OK;
}

Hier::~Hier() {
  // work issued on any stream may still read these buffers; a caching allocator hook (unlike
  // cudaFree) would hand them out again at once
  if (!allocs.empty()) cudaDeviceSynchronize();
  for (auto e : event_pool) cudaEventDestroy(e);
  for (void* p : allocs) dev_free(p);
  if (sc_host) cudaFreeHost(sc_host);
}

Group::~Group() {
  cudaDeviceSynchronize();
  if (graph) cudaGraphExecDestroy(graph);
  if (loop_graph) cudaGraphExecDestroy(loop_graph);
  if (loop) dev_free(loop);
  if (loop_host) cudaFreeHost(loop_host);
  if (graph_stream) cudaStreamDestroy(graph_stream);
  for (Hier* h : parts) delete h;
  delete comm;
  delete plan;
}

// ------------------------------------------------------------------------------------
// schedule of one preconditioner application M (Alg. 4; SURVEY c-6)
// ------------------------------------------------------------------------------------
namespace {

enum { SM_PLAIN = 0, SM_ZERO1 = 1, SM_ZERO2 = 2, SM_PRO1 = 3, SM_PRO2 = 4, SM_RESTRICT = 5, SM_PLAIN_RZ = 6 };

inline int stage_desc(int colour, int mode) { return colour | (mode << 1); }

// Tiles of each level in rank order (slab-major: z, then Morton of (x, y)), so that the
// consecutive tiles of a CTA's run share faces (host, once per hierarchy).
octmg_status build_orders(Hier& h) {
  const Tree& T = *h.tree;
  std::vector<int4> tile(T.T);
  OCTMG_CUDA(cudaMemcpy(tile.data(), T.tile, sizeof(int4) * T.T, cudaMemcpyDeviceToHost));
  std::vector<int> nbr((size_t)T.T * 6);
  OCTMG_CUDA(cudaMemcpy(nbr.data(), T.nbr, sizeof(int) * nbr.size(), cudaMemcpyDeviceToHost));
  {
    // levels with a T-junction (ghost) face anywhere (all parts decide alike)
    for (int l = 0; l <= MAXL; ++l) h.lvl_ghost[l] = false;
    for (int t = 0; t < T.T; ++t)
      for (int f = 0; f < 6; ++f)
        if (nbr[6 * (size_t)t + f] <= -2) h.lvl_ghost[tile[t].x] = true;
    // the face layers of inner tiles that are same-level neighbours of this part's leaf
    // tiles: the apply reads their active-children means from pbar (k_inner_face_means)
    if (!h.ifaces) {
      std::vector<int2> fl;
      for (int l = 0; l <= T.L; ++l)
        for (int t = h.own_lb[l]; t < h.own_lb[l] + h.own_lc[l]; ++t)
          for (int f = 0; f < 6; ++f) {
            const int n = nbr[6 * (size_t)t + f];
            if (n >= T.NL) fl.push_back(make_int2(n, f ^ 1));
          }
      h.n_ifaces = (int)fl.size();
      OCTMG_TRY(halloc(h.allocs, &h.ifaces, std::max<size_t>(fl.size(), 1)));
      if (!fl.empty()) {
        OCTMG_CUDA(cudaMemcpy(h.ifaces, fl.data(), sizeof(int2) * fl.size(), cudaMemcpyHostToDevice));
        OCTMG_TRY(halloc(h.allocs, &h.pbar, (size_t)T.NI * TB3));
      }
    }
  }
  auto m2 = [](uint32_t x, uint32_t y) {
    uint64_t m = 0;
    for (int b = 0; b < 21; ++b) m |= ((uint64_t)((x >> b) & 1) << (2 * b)) | ((uint64_t)((y >> b) & 1) << (2 * b + 1));
    return m;
  };
  std::vector<int> order;
  order.reserve(T.T);
  for (int l = 0; l <= T.L; ++l) {
    std::vector<int> ts;
    for (int t = h.own_lb[l]; t < h.own_lb[l] + h.own_lc[l]; ++t) ts.push_back(t);
    for (int t = h.own_ib[l]; t < h.own_ib[l] + h.own_ic[l]; ++t) ts.push_back(t);
    std::sort(ts.begin(), ts.end(), [&](int a, int b) {
      if (tile[a].w != tile[b].w) return tile[a].w < tile[b].w;
      return m2(tile[a].y, tile[a].z) < m2(tile[b].y, tile[b].z);
    });
    // tiles without a ghost face first (each group keeps that order): kernels with a
    // ghost-free fast path can be launched on the two groups separately
    auto regular = [&](int t) {
      for (int f = 0; f < 6; ++f)
        if (nbr[6 * (size_t)t + f] <= -2) return false;
      return true;
    };
    const auto mid = std::stable_partition(ts.begin(), ts.end(), regular);
    h.lvl_nreg[l] = (int)(mid - ts.begin());
    h.lvl_order_off[l] = (int)order.size();
    h.lvl_n[l] = (int)ts.size();
    order.insert(order.end(), ts.begin(), ts.end());
  }
  int* d;
  OCTMG_TRY(halloc(h.allocs, &d, order.size()));
  OCTMG_CUDA(cudaMemcpy(d, order.data(), sizeof(int) * order.size(), cudaMemcpyHostToDevice));
  h.order = d;
  return OCTMG_OK;
}

struct Builder {
  Group& g;
  Hier& h;  // part 0 (every part has the same schedule)
  void push(const Op& op) { g.ops.push_back(op); }
  void xchg(int l) {  // halo exchange of level l after a kernel changed it
    if (h.nranks > 1 && l >= h.lg) push(Op{7, l, 0});
  }
  void stage(int l, int desc) {
    push(Op{0, l, desc});
    if ((desc >> 1) == SM_RESTRICT) {
      if (h.nranks > 1 && l == h.lg && l >= 1) push(Op{8, l - 1, 0});  // parents -> all ranks
      else xchg(l - 1);
    } else {
      xchg(l);
    }
  }
  void passes(int l, int iters, bool red_first, int m1, int m2) {
    for (int k = 0; k < iters; ++k) {
      stage(l, stage_desc(red_first ? 0 : 1, k == 0 ? m1 : SM_PLAIN));
      stage(l, stage_desc(red_first ? 1 : 0, k == 0 ? m2 : SM_PLAIN));
    }
  }
  // Alg. 4 at level l; fas_first: first of the mu calls from level l+1 (forms the FAS rhs)
  void fas(int l, bool fas_first) {
    const Tree& T = *h.tree;
    if (l <= h.sub_K) {  // the rest of the cycle runs on chip in one CTA
      push(Op{4, l, fas_first ? 1 : 0});
      return;
    }
    if (l < T.L && fas_first && T.ic[l] > 0 && h.prm.form == 0) push(Op{1, l, 0});
    const bool finest = l == T.L;
    if (l == 0 && h.c0n > 0) {  // direct coarsest solve (Alg. 4 line 4)
      push(Op{10, 0, 0});
      return;
    }
    if (l == 0) {
      int nb = h.prm.nu_coarsest;
      int h1 = nb / 2;
      passes(0, h1, true, finest ? SM_ZERO1 : SM_PLAIN, finest ? SM_ZERO2 : SM_PLAIN);
      bool z = finest && h1 == 0;
      passes(0, nb - h1, false, z ? SM_ZERO1 : SM_PLAIN, z ? SM_ZERO2 : SM_PLAIN);
      return;
    }
    passes(l, h.prm.nu_pre, true, finest ? SM_ZERO1 : SM_PLAIN, finest ? SM_ZERO2 : SM_PLAIN);
    stage(l, stage_desc(0, SM_RESTRICT));
    for (int k = 0; k < h.prm.mu; ++k) fas(l - 1, k == 0);
    push(Op{3, l, 0});  // prolongation u += P(u^{l-1} - u*), in place
    xchg(l);
    passes(l, h.prm.nu_post, false, SM_PLAIN, SM_PLAIN);
  }
};

void read_env(Hier& h) {
  const char* pc = getenv("OCTMG_PASS_CPT");
  h.pass_cpt = pc ? (atoi(pc) >= 4 ? 4 : std::max(1, std::min(2, atoi(pc)))) : 4;
  const char* pb = getenv("OCTMG_PASS_BIG");
  h.pass_big = pb ? std::max(1, atoi(pb)) : 512;  // levels with >= this many tiles take pass_cpt (1024 before: config 5 469.8 vs 468.2 ms, config 2 5.52 vs 5.48 ms)
  h.pass_v2 = true;
  h.restrict_v2 = 6;  // k_restrict_v2 at >= 6 CTAs/SM
  const char* to = getenv("OCTMG_TILE_ORDER");  // slab: the slab-major order array
  h.direct_order = !(to && std::string(to) == "slab");
  const char* rd = getenv("OCTMG_RESTRICT_RED");
  h.restrict_red = !(rd && atoi(rd) == 0);
  const char* rw = getenv("OCTMG_RESTRICT_ROW");
  h.restrict_row = rw ? (atoi(rw) != 0 ? 1 : 0) : -1;
  const Tree& T = *h.tree;
  const char* sc = getenv("OCTMG_SUBCYCLE");
  const int sub_cap = subcycle_max_tiles();
  h.sub_K = -1;
  if (!(sc && std::string(sc) == "0"))
    for (int l = 0; l <= std::min(T.L, subcycle_max_level()); ++l) {
      if (h.lvl_n[l] > sub_cap) break;
      if (h.nranks > 1 && l >= h.lg) break;  // only replicated levels run on chip
      h.sub_K = l;
    }
}

bool split_pass(const Hier& h, int l, int mode);

octmg_status build_schedule(Group& g) {
  g.ops.clear();
  for (Hier* p : g.parts) {
    OCTMG_TRY(build_orders(*p));
    read_env(*p);
    // the on-chip sub-cycle levels as dense shared-memory grids when they are complete
    // inner levels (coarse_dense.cu); otherwise the tile-layout k_subcycle
    // (not in the GMG comparison mode: its prolongation skips inactive parents, which the
    // dense and cluster kernels do not test)
    if (p->sub_K >= 0 && p->c0n == 0 && p->ccoef == p->coef) {
      OCTMG_TRY(build_coarse_dense(*p, p->nranks > 1 ? p->lg - 1 : MAXL, nullptr));
      OCTMG_CUDA(cudaDeviceSynchronize());
      if (p->cd_K >= p->sub_K) p->sub_K = p->cd_K;
      else p->cd_K = -1;
      // level 2 too, in a thread-block cluster, when it is a replicated complete level
      if (p->cd_K == 1 && (p->nranks == 1 || p->lg > 2)) {
        OCTMG_TRY(build_coarse_cluster(*p, nullptr));
        OCTMG_CUDA(cudaDeviceSynchronize());
        if (p->cc_K == 2) p->sub_K = 2;
      }
    }
  }
  Hier& h = *g.parts[0];
  const Tree& T = *h.tree;
  if (T.NL > T.lc[T.L]) g.ops.push_back(Op{2, 0, 0});  // coarse leaves start the cycle at 0
  Builder b{g, h};
  b.fas(T.L, false);
  // (r, z) fused into the last pass of M when every leaf is at the finest level and that level
  // runs the 128-bit row pass (OCTMG_RZ_FUSED=0: the separate k_dot_rz pass)
  g.rz_fused = false;
  const char* rf = getenv("OCTMG_RZ_FUSED");
  const int lt = T.lc[T.L] + T.ic[T.L];
  if (!(rf && atoi(rf) == 0) && T.NL == T.lc[T.L] && T.L > h.sub_K && lt >= h.pass_big && h.pass_cpt == 4 &&
      h.pass_v2 && pass_v3_on() && !h.lvl_ghost[T.L] && h.prm.form == 0)
    for (auto it = g.ops.rbegin(); it != g.ops.rend(); ++it)
      if (it->kind == 0 && it->level == T.L) {
        if ((it->stage >> 1) == SM_PLAIN && !split_pass(h, T.L, SM_PLAIN)) {
          it->stage = stage_desc(it->stage & 1, SM_PLAIN_RZ);
          g.rz_fused = true;
        }
        break;
      }
  return OCTMG_OK;
}

// parts whose apply first forms the inner-face children means (one more kernel per apply)
int inner_mean_kernels(const Group& g) {
  int n = 0;
  for (const Hier* h : g.parts) n += h->n_ifaces > 0;
  return n;
}

// restrictions launched as two kernels (big ghost level: ghost-free tiles + ghost tiles)
// (every ghost level with ghost-free tiles: they take the red-row kernel; OCTMG_RESTRICT_SPLIT=
// big: only levels of >= 32768 tiles)
bool split_restrict(const Hier& h, int l) {
  int all = -1;  // (read per call: the variant tests switch it within one process)
  if (all < 0) {
    const char* e = getenv("OCTMG_RESTRICT_SPLIT");
    all = !(e && std::string(e) == "big");
  }
  const Tree& T = *h.tree;
  const bool big_ghost = h.lvl_ghost[l] && T.lc[l] + T.ic[l] >= 32768;
  const bool ok = all ? h.lvl_ghost[l] : big_ghost;
  return ok && h.restrict_red && h.restrict_v2 && h.restrict_row != 0 && h.lvl_nreg[l] > 0 && h.lvl_nreg[l] < h.lvl_n[l];
}

// colour passes launched as two kernels on big ghost levels (OCTMG_PASS_SPLIT=1; measured
// slower than one launch with the inlined ghost body: config 3 10.28 vs 10.02 ms, config 5
// level 9 111.7 vs 108.7 ms of passes per solve — the second launch's ramp and tail)
bool split_pass(const Hier& h, int l, int mode) {
  int on = -1;
  if (on < 0) {
    const char* e = getenv("OCTMG_PASS_SPLIT");
    on = e && atoi(e) == 1;
  }
  const Tree& T = *h.tree;
  return on && mode != SM_ZERO1 && h.pass_v2 && h.pass_cpt == 4 && h.lvl_ghost[l] &&
         T.lc[l] + T.ic[l] >= std::max(32768, h.pass_big) && h.lvl_nreg[l] > 0 && h.lvl_nreg[l] < h.lvl_n[l];
}

int64_t schedule_kernels(const Group& g) {
  int64_t n = 0;
  for (const Hier* h : g.parts)
    for (const Op& op : g.ops) {
      if (op.kind == 2 || op.kind == 7 || op.kind == 8) continue;
      n += 1;
      if (op.kind == 0 && (op.stage >> 1) == SM_PLAIN_RZ) n += 2;  // + the (r, z) chunk sums and finish
      if (op.kind == 0 && (op.stage >> 1) == SM_RESTRICT && split_restrict(*h, op.level)) n += 1;
      if (op.kind == 0 && (op.stage >> 1) != SM_RESTRICT && split_pass(*h, op.level, op.stage >> 1)) n += 1;
    }
  return n;
}

Fld ubuf(const Hier& h) { return Fld{h.z, h.uinA}; }

cudaEvent_t next_event(Hier& h) {
  if (h.event_next == h.event_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    h.event_pool.push_back(e);
  }
  return h.event_pool[h.event_next++];
}

// CUDA events around a launch (and an NVTX range "class Ll" for nsys timelines) while the
// hierarchy profiles; nothing otherwise
struct ProfScope {
  Hier& h;
  int cls;
  cudaStream_t s;
  cudaEvent_t b = nullptr;
  ProfScope(Hier& hh, int c, cudaStream_t ss, double bytes, int level = -1) : h(hh), cls(c), s(ss) {
    if (h.profiling) {
      char nm[48];
      if (level >= 0) snprintf(nm, sizeof nm, "%s L%d", kclass_name[cls], level);
      else snprintf(nm, sizeof nm, "%s", kclass_name[cls]);
      nvtxRangePushA(nm);
      cudaEvent_t a = next_event(h);
      b = next_event(h);
      cudaEventRecord(a, s);
      h.events.push_back({cls, bytes, a, b, level});
    }
  }
  ~ProfScope() {
    if (h.profiling) {
      cudaEventRecord(b, s);
      nvtxRangePop();
    }
  }
};

void launch_op(Hier& h, const Op& op, cudaStream_t s) {
  const Tree& T = *h.tree;
  if (op.kind == 2) {
    size_t first = (size_t)T.lc[T.L] * TB3;
    ProfScope ps(h, KC_MEMSET, s, 4.0 * ((double)T.NL * TB3 - first), op.level);
    cudaMemsetAsync(h.z + first, 0, ((size_t)T.NL * TB3 - first) * sizeof(float), s);
    return;
  }
  const int l = op.level;
  SmoothArgs a;
  a.tile = T.tile; a.nbr = T.nbr; a.parent = T.parent; a.coef = h.ccoef; a.glayer_val = h.glayer_val;
  a.glayer = T.glayer; a.u = ubuf(h); a.uc = ubuf(h); a.ustar = h.ustar; a.ustar_w = h.ustar;
  a.b = Fld{h.r, h.binner};
  a.alpha = h.prm.alpha; a.NL = T.NL;
  // FAS form (Alg. 4): beta at restriction, prolongation of u^{l-1} - u*; standard form
  // (Alg. 2): R r as the coarse rhs, zero coarse guess (u* = 0), beta at prolongation
  a.std_form = h.prm.form == 1;
  a.beta = a.std_form ? 1.0f : h.prm.beta_overshoot;
  a.pro_scale = a.std_form ? h.prm.beta_overshoot : 1.0f;
  a.pro_active_only = h.ccoef != h.coef;  // GMG comparison mode (reading 20)
  a.order = h.order + h.lvl_order_off[l];
  a.ord_leaf0 = h.own_lb[l];
  a.ord_nleaf = h.own_lc[l];
  a.ord_inner0 = h.own_ib[l];
  if (h.direct_order) a.order = nullptr;  // tiles by index (Morton within leaves, inners)
  a.n = h.lvl_n[l];
  a.first_tile = T.ib[l];
  a.stage[0] = op.stage;
  a.c0M = h.c0M;
  a.c0tile = h.c0tile;
  a.c0n = h.c0n;
  if (op.kind == 10) {
    // read M0 (4 n0^2 B) and b^0, write u^0
    ProfScope ps(h, KC_COARSEST, s, 4.0 * (double)h.c0n * h.c0n + 8.0 * h.c0n, op.level);
    launch_coarse_direct(a, s);
    return;
  }

  if (op.kind == 4 && h.cc_K == 2 && l == 2) {
    ProfScope ps(h, KC_SUBCYCLE, s, 0.0, op.level);
    launch_coarse_cluster(h, op.stage, h.uinA, h.binner, s);
    return;
  }
  if (op.kind == 4 && h.cd_K >= 0) {
    ProfScope ps(h, KC_SUBCYCLE, s, 0.0, op.level);
    launch_coarse_dense(h, l, op.stage, h.uinA, h.binner, s);
    return;
  }
  if (op.kind == 4) {
    ProfScope ps(h, KC_SUBCYCLE, s, 0.0, op.level);
    launch_subcycle(a, T.L, l, op.stage, h.prm, h.order, h.lvl_order_off, h.lvl_n, T.ib, T.ic, s);
    return;
  }
  if (op.kind == 3) {
    // read u and the c plane, write u (12 B/cell) + the parents' u, u* (1 B/cell)
    ProfScope ps(h, KC_PROLONG, s, 13.0 * a.n * TB3, op.level);
    launch_prolong(a, s);
    return;
  }
  if (op.kind == 1) {
    // read u, b, record; write b (inner cells of the level, this part's)
    a.first_tile = h.own_ib[l];
    ProfScope ps(h, KC_FASRHS, s, 28.0 * h.own_ic[l] * TB3, op.level);
    launch_fasrhs(a, h.own_ic[l], s);
    return;
  }
  const int mode = op.stage >> 1;
  // algorithmic bytes per cell of the level (colour-split slot order): a colour pass reads
  // the other colour's u (2 B), its own colour's b (2 B) and 4 coefficient planes (8 B), the
  // other colour's 3 coupling planes (6 B) and writes its own u (2 B): 20 B; the first pass
  // of a cycle (u known 0: u = b / c) 6 B; restrict = read u, b, record (24 B) + the
  // parents' u, u*, b (1.5 B); prolongation-fused passes read the parents' u, u* (+1 B)
  const double cells = (double)a.n * TB3;
  double bytes = cells * (mode == SM_RESTRICT ? 25.5 : (mode == SM_ZERO1 ? 6.0 : 20.0));
  if (mode == SM_PLAIN_RZ) bytes += 2.0 * cells;  // the other colour's r
  if (mode == SM_PRO1 || mode == SM_PRO2) bytes += cells;
  int cls = mode == SM_RESTRICT ? KC_RESTRICT
          : (l == 0 ? KC_COARSEST : (l < T.L ? KC_SMOOTH_COARSE : KC_PASS));
  ProfScope ps(h, cls, s, bytes, op.level);
  if (mode == SM_RESTRICT) {
    // levels with T-junction tiles: the row-form restriction (its ghost path in the row);
    // OCTMG_RESTRICT_ROW=0 keeps k_restrict_v2 everywhere, =1 takes the row form everywhere
    // (measured: faster on config 3's 85696-tile level 7 — 3.86 vs 4.13 ms per solve — slower on
    // config 4's smaller ghost levels, so only on ghost levels of >= 32768 tiles)
    const bool big_ghost = h.lvl_ghost[l] && T.lc[l] + T.ic[l] >= 32768;
    int rr = h.restrict_row < 0 ? (big_ghost ? 64 : 0) : (h.restrict_row ? 64 : 0);
    // ghost-free levels: the red-row restriction (the black residual is zero after the black
    // pass that ends the pre-smoothing); OCTMG_RESTRICT_RED=0 keeps k_restrict_v2
    if (!rr && !h.lvl_ghost[l] && h.restrict_red) rr = 128;
    if (split_restrict(h, l)) {
      // ghost level: the ghost-free tiles (first in the order) with the red-row kernel, the
      // ghost tiles with the row form (big levels) or k_restrict_v2
      SmoothArgs ar = a, ag = a;
      ar.order = h.order + h.lvl_order_off[l];
      ar.n = h.lvl_nreg[l];
      ag.order = ar.order + h.lvl_nreg[l];
      ag.n = a.n - h.lvl_nreg[l];
      launch_restrict_direct(ar, s, h.restrict_v2 | 128);
      launch_restrict_direct(ag, s, h.restrict_v2 | rr);
    } else {
      launch_restrict_direct(a, s, h.restrict_v2 ? (h.restrict_v2 | rr) : 0);
    }
  } else {
    // kernel chosen by the level's total tile count, so every part of a partitioned solve runs
    // the same per-tile arithmetic as the single-part solve
    const int level_tiles = T.lc[l] + T.ic[l];
    const int cpt = (level_tiles >= h.pass_big ? h.pass_cpt : 1) | (h.pass_v2 ? 16 : 0);
    if (split_pass(h, l, mode)) {
      // big ghost level: the ghost-free tiles (first in the order) with the regular-path
      // kernel at 16 CTAs/SM, the ghost tiles with the inlined ghost body
      SmoothArgs ar = a, ag = a;
      ar.order = h.order + h.lvl_order_off[l];
      ar.n = h.lvl_nreg[l];
      ag.order = ar.order + h.lvl_nreg[l];
      ag.n = a.n - h.lvl_nreg[l];
      launch_pass_direct(ar, s, cpt);
      launch_pass_direct(ag, s, cpt | 32);
    } else {
      a.rz_partial = h.partial;
      launch_pass_direct(a, s, cpt | (h.lvl_ghost[l] ? 32 : 0));
      if (mode == SM_PLAIN_RZ) launch_rz_finish(h.partial, 2 * (int64_t)a.n, h.partial + 2 * (size_t)a.n, h.sc, s);
    }
  }
}

std::vector<Fld> ubufs(const Group& g) {
  std::vector<Fld> f;
  for (const Hier* h : g.parts) f.push_back(ubuf(*h));
  return f;
}

octmg_status launch_ops(Group& g, cudaStream_t s) {
  for (const Op& op : g.ops) {
    if (op.kind == 7) OCTMG_TRY(g.comm->exchange(g, op.level, 0, ubufs(g), s));
    else if (op.kind == 8) OCTMG_TRY(g.comm->bcast_parents(g, s));
    else
      for (Hier* h : g.parts) launch_op(*h, op, s);
  }
  return OCTMG_OK;
}

bool profiling(const Group& g) { return g.parts[0]->profiling; }

octmg_status run_M(Group& g, cudaStream_t s) {
  if (profiling(g)) {
    OCTMG_TRY(launch_ops(g, s));
    OCTMG_CUDA(cudaGetLastError());
    g.launches += schedule_kernels(g);
    return OCTMG_OK;
  }
  if (!g.graph) {
    if (!g.graph_stream) OCTMG_CUDA(cudaStreamCreateWithFlags(&g.graph_stream, cudaStreamNonBlocking));
    cudaGraph_t gr;
    OCTMG_CUDA(cudaStreamBeginCapture(g.graph_stream, cudaStreamCaptureModeThreadLocal));
    octmg_status st = launch_ops(g, g.graph_stream);
    cudaError_t e = cudaStreamEndCapture(g.graph_stream, &gr);
    if (st != OCTMG_OK) return st;
    if (e != cudaSuccess) return cuda_status(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&g.graph, gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) return cuda_status(e, "cudaGraphInstantiate");
  }
  OCTMG_CUDA(cudaGraphLaunch(g.graph, s));
  g.launches += schedule_kernels(g);
  return OCTMG_OK;
}

octmg_status allreduce(Group& g, int first, int count, cudaStream_t s) {
  if (g.comm) return g.comm->allreduce(g, first, count, s);
  return OCTMG_OK;
}

int vec_grid() { return 148 * 4; }

}  // namespace

}  // namespace octmg

using namespace octmg;

extern "C" {

const char* octmg_last_error(void) { return g_err.c_str(); }

const char* octmg_version(void) { return "octmg 0.1.0 (sm_100a, fp32 fields / fp64 dots)"; }

octmg_status octmg_set_allocator(octmg_alloc_fn alloc, octmg_free_fn release, void* ctx) {
  if ((alloc == nullptr) != (release == nullptr)) {
    set_error("alloc and release must both be set or both be NULL");
    return OCTMG_E_INVALID;
  }
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  g_alloc.alloc = alloc;
  g_alloc.release = release;
  g_alloc.ctx = ctx;
  return OCTMG_OK;
}

octmg_status octmg_build_tree(const octmg_tree_desc* desc, const octmg_tile* leaf_tiles_host, int64_t n,
                              octmg_stream stream, octmg_tree** out) {
  if (!desc || !leaf_tiles_host || !out) { set_error("null argument"); return OCTMG_E_INVALID; }
  *out = nullptr;
  auto* t = new (std::nothrow) octmg_tree();
  if (!t) { set_error("host allocation failed"); return OCTMG_E_OOM; }
  octmg_status st;
  if (desc->grade_repair == 1) {  // refine the coarser side to fixpoint first (host)
    std::vector<octmg_tile> rep;
    st = n < 0 ? OCTMG_E_INVALID : grade_repair(leaf_tiles_host, n, desc->ext, rep);
    if (st == OCTMG_OK) {
      octmg_tree_desc d2 = *desc;
      d2.grade_repair = 0;
      st = build_tree(&d2, rep.data(), (int64_t)rep.size(), (cudaStream_t)stream, &t->t);
    }
  } else {
    st = build_tree(desc, leaf_tiles_host, n, (cudaStream_t)stream, &t->t);
  }
  if (st != OCTMG_OK) { delete t; return st; }
  *out = t;
  return OCTMG_OK;
}

octmg_status octmg_tree_info_get(const octmg_tree* tree, octmg_tree_info* out) {
  if (!tree || !out) { set_error("null argument"); return OCTMG_E_INVALID; }
  const Tree& T = tree->t;
  std::memset(out, 0, sizeof(*out));
  out->levels = T.L + 1;
  out->n_leaf_tiles = T.NL;
  out->n_inner_tiles = T.NI;
  out->n_leaf_cells = (int64_t)T.NL * TB3;
  for (int l = 0; l <= T.L; ++l) {
    out->leaf_begin[l] = T.lb[l]; out->leaf_count[l] = T.lc[l];
    out->inner_begin[l] = T.ib[l]; out->inner_count[l] = T.ic[l];
  }
  out->n_ghost_layers = T.n_glayers;
  return OCTMG_OK;
}

octmg_status octmg_tree_export(const octmg_tree* tree, int32_t what, void* host_dst, size_t bytes) {
  if (!tree || !host_dst) { set_error("null argument"); return OCTMG_E_INVALID; }
  const Tree& T = tree->t;
  const void* src = nullptr;
  size_t need = 0;
  switch (what) {
    case OCTMG_EXPORT_TILES: src = T.tile; need = (size_t)T.T * 16; break;
    case OCTMG_EXPORT_NBR: src = T.nbr; need = (size_t)T.T * 24; break;
    case OCTMG_EXPORT_PARENT: src = T.parent; need = (size_t)T.T * 4; break;
    case OCTMG_EXPORT_CHILD: src = T.child; need = (size_t)T.NI * 32; break;
    default: set_error("unknown export id"); return OCTMG_E_INVALID;
  }
  if (bytes != need) { set_error("export buffer size mismatch"); return OCTMG_E_INVALID; }
  if (need) OCTMG_CUDA(cudaMemcpy(host_dst, src, need, cudaMemcpyDeviceToHost));
  return OCTMG_OK;
}

}  // extern "C"

namespace octmg {
namespace {

// allocate and assemble one part (every part holds the full replicated coefficient set)
octmg_status setup_part(Hier& h, Tree* tree, const uint8_t* kind, const float* fbeta, const float* ffrac,
                        const octmg_mg_params& prm, cudaStream_t s) {
  h.tree = tree;
  h.prm = prm;
  const Tree& T = *tree;
  size_t NLc = (size_t)T.NL * TB3, NIc = (size_t)T.NI * TB3;
  OCTMG_TRY(halloc(h.allocs, &h.coef, (size_t)T.T * TB3 * 4));
  OCTMG_TRY(halloc(h.allocs, &h.glayer_val, (size_t)T.n_glayers * 64));
  OCTMG_TRY(halloc(h.allocs, &h.act, NLc / 32));
  OCTMG_TRY(halloc(h.allocs, &h.z, NLc));
  OCTMG_TRY(halloc(h.allocs, &h.uinA, NIc));
  OCTMG_TRY(halloc(h.allocs, &h.binner, NIc));
  OCTMG_TRY(halloc(h.allocs, &h.ustar, NIc));
  OCTMG_TRY(halloc(h.allocs, &h.r, NLc));
  OCTMG_TRY(halloc(h.allocs, &h.xs, NLc));
  OCTMG_TRY(halloc(h.allocs, &h.p0, NLc));
  OCTMG_TRY(halloc(h.allocs, &h.p1, NLc));
  OCTMG_TRY(halloc(h.allocs, &h.q, NLc));
  // apply: 4 warp partials per leaf tile of p.q and of sum q + their chunk sums
  h.n_partial = std::max<size_t>(8 * (size_t)T.NL + 1024, 2 * (size_t)vec_grid()) + 16;
  OCTMG_TRY(halloc(h.allocs, &h.partial, h.n_partial));
  OCTMG_TRY(halloc(h.allocs, &h.counter, 16));
  OCTMG_TRY(halloc(h.allocs, &h.sc, 1));
  // mapped pinned memory: the solve reads its scalars through a kernel that writes them
  // there, not through a device-to-host copy, which would queue behind a caller's large
  // copies on the copy engine (a serving loop downloads the previous solution meanwhile)
  if (cudaHostAlloc(&h.sc_host, sizeof(Scalars), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void**)&h.sc_host_dev, h.sc_host, 0) != cudaSuccess) {
    cudaGetLastError();
    set_error("pinned allocation failed");
    return OCTMG_E_OOM;
  }
  OCTMG_CUDA(cudaMemsetAsync(h.counter, 0, 16 * sizeof(unsigned), s));
  OCTMG_CUDA(cudaMemsetAsync(h.uinA, 0, NIc * sizeof(float), s));
  OCTMG_CUDA(cudaMemsetAsync(h.z, 0, NLc * sizeof(float), s));
  OCTMG_CUDA(cudaMemsetAsync(h.p0, 0, NLc * sizeof(float), s));
  OCTMG_CUDA(cudaMemsetAsync(h.p1, 0, NLc * sizeof(float), s));
  OCTMG_CUDA(cudaMemsetAsync(h.sc, 0, sizeof(Scalars), s));
  OCTMG_TRY(assemble_leaf_coefs(h, kind, fbeta, ffrac, s));  // + Alg. 3 coarsening and leaf row sums
  launch_build_mask(h.coef, (int64_t)NLc, h.act, s);
  if (prm.coarsest == 1) OCTMG_TRY(build_coarse_direct(h, s));  // M0 of level 0 (Alg. 4 line 4)
  OCTMG_CUDA(cudaStreamSynchronize(s));
  Scalars init{};
  init.n_active = h.n_active;
  OCTMG_CUDA(cudaMemcpy(h.sc, &init, sizeof(Scalars), cudaMemcpyHostToDevice));
  return OCTMG_OK;
}

}  // namespace
uint64_t morton3h(uint32_t i, uint32_t j, uint32_t k) {
  uint64_t m = 0;
  for (int b = 0; b < 21; ++b)
    m |= ((uint64_t)((i >> b) & 1) << (3 * b)) | ((uint64_t)((j >> b) & 1) << (3 * b + 1)) |
         ((uint64_t)((k >> b) & 1) << (3 * b + 2));
  return m;
}
namespace {

octmg_status plan_input(const Tree& T, PartInput& in) {
  in.L = T.L; in.NL = T.NL; in.NI = T.NI;
  in.lb = T.lb; in.lc = T.lc; in.ib = T.ib; in.ic = T.ic;
  in.tiles4.resize((size_t)T.T * 4);
  in.nbr.resize((size_t)T.T * 6);
  in.parent.resize(T.T);
  in.child.resize((size_t)T.NI * 8);
  OCTMG_CUDA(cudaMemcpy(in.tiles4.data(), T.tile, sizeof(int4) * T.T, cudaMemcpyDeviceToHost));
  OCTMG_CUDA(cudaMemcpy(in.nbr.data(), T.nbr, sizeof(int) * 6 * T.T, cudaMemcpyDeviceToHost));
  OCTMG_CUDA(cudaMemcpy(in.parent.data(), T.parent, sizeof(int) * T.T, cudaMemcpyDeviceToHost));
  if (T.NI) OCTMG_CUDA(cudaMemcpy(in.child.data(), T.child, sizeof(int) * 8 * T.NI, cudaMemcpyDeviceToHost));
  in.morton.resize(T.T);
  for (int t = 0; t < T.T; ++t) in.morton[t] = morton3h(in.tiles4[4 * t + 1], in.tiles4[4 * t + 2], in.tiles4[4 * t + 3]);
  return OCTMG_OK;
}

// owned tile ranges of part h (contiguous per level by construction of the partition)
octmg_status set_ownership(Hier& h, const PartPlan* P) {
  const Tree& T = *h.tree;
  std::vector<int> tiles;
  for (int l = 0; l <= T.L; ++l) {
    auto range = [&](int b, int c, int* ob, int* oc) -> bool {
      if (!P || l < P->lg) { *ob = b; *oc = c; return true; }
      int first = -1, cnt = 0;
      for (int t = b; t < b + c; ++t)
        if (P->owner[t] == h.rank) {
          if (first < 0) first = t;
          else if (t != first + cnt) return false;
          cnt++;
        }
      *ob = first < 0 ? b : first;
      *oc = cnt;
      return true;
    };
    if (!range(T.lb[l], T.lc[l], &h.own_lb[l], &h.own_lc[l]) || !range(T.ib[l], T.ic[l], &h.own_ib[l], &h.own_ic[l])) {
      set_error("partition ownership is not contiguous per level");
      return OCTMG_E_INVALID;
    }
  }
  h.own_cells = Ranges{};
  for (int l = T.L; l >= 0; --l) {
    if (!h.own_lc[l]) continue;
    h.own_cells.begin[h.own_cells.n] = (int64_t)h.own_lb[l] * TB3 / 4;
    h.own_cells.len[h.own_cells.n] = (int64_t)h.own_lc[l] * TB3 / 4;
    h.own_cells.n++;
    for (int t = h.own_lb[l]; t < h.own_lb[l] + h.own_lc[l]; ++t) tiles.push_back(t);
  }
  h.n_apply_tiles = (int)tiles.size();
  OCTMG_TRY(halloc(h.allocs, &h.apply_tiles, tiles.size()));
  OCTMG_CUDA(cudaMemcpy(h.apply_tiles, tiles.data(), sizeof(int) * tiles.size(), cudaMemcpyHostToDevice));
  return OCTMG_OK;
}

bool valid_params(const octmg_mg_params& prm) {
  return prm.alpha > 0.0f && prm.mu >= 1 && prm.mu <= 4 && prm.nu_pre >= 1 && prm.nu_post >= 1 &&
         prm.nu_coarsest >= 1 && (prm.form == 0 || prm.form == 1) && (prm.coarsen_literal == 0 || prm.coarsen_literal == 1) &&
         (prm.coarsest == 0 || prm.coarsest == 1) && prm.gather_below_cells >= 0;
}

// a Group of `nparts` parts (1 = single GPU / one NCCL rank; >1 = loopback partition)
octmg_status make_group(octmg_tree* tree, int nparts, int rank, int nranks, void* nccl_comm, const uint8_t* kind,
                        const float* fbeta, const float* ffrac, const octmg_mg_params* params, cudaStream_t s,
                        octmg_hier** out, const uint8_t* gmg_kind = nullptr, const float* gmg_beta = nullptr,
                        const float* gmg_frac = nullptr) {
  octmg_mg_params prm{2.0f, 2.0f, 1, 2, 2, 10, 0, 0, 0, 0, 0};
  if (params) prm = *params;
  if (!valid_params(prm)) {
    set_error("invalid multigrid parameters (need alpha > 0, 1 <= mu <= 4, nu_* >= 1, form and coarsen_literal 0/1)");
    return OCTMG_E_INVALID;
  }
  if (prm.form == 1 && tree->t.NL != tree->t.lc[tree->t.L]) {
    set_error("the standard mu-cycle (Alg. 2, form = 1) needs a uniform tree (every leaf at the finest level)");
    return OCTMG_E_INVALID;
  }
  auto* hh = new (std::nothrow) octmg_hier();
  if (!hh) { set_error("host allocation failed"); return OCTMG_E_OOM; }
  Group& g = hh->g;
  auto fail = [&](octmg_status e) { delete hh; return e; };
  for (int p = 0; p < nparts; ++p) {
    Hier* h = new (std::nothrow) Hier();
    if (!h) return fail(OCTMG_E_OOM);
    g.parts.push_back(h);
    h->rank = nparts > 1 ? p : rank;
    h->nranks = nranks;
    h->gmg_kind = gmg_kind;
    h->gmg_beta = gmg_beta;
    h->gmg_frac = gmg_frac;
    octmg_status st = setup_part(*h, &tree->t, kind, fbeta, ffrac, prm, s);
    h->gmg_kind = nullptr;
    h->gmg_beta = h->gmg_frac = nullptr;
    if (st) return fail(st);
  }
  const PartPlan* P = nullptr;
  if (nranks > 1) {
    g.plan = new PartPlanHolder();
    PartInput in;
    octmg_status st = plan_input(tree->t, in);
    if (st) return fail(st);
    const int lg = choose_partition_level(in, nranks, prm.gather_below_cells);
    if (lg == 0 && prm.coarsest == 1) {
      set_error("direct coarsest solve needs a replicated level 0 (partition level >= 1)");
      return fail(OCTMG_E_INVALID);
    }
    build_partition(in, nranks, lg, g.plan->plan);
    P = &g.plan->plan;
    for (Hier* h : g.parts) h->lg = lg;
    g.comm = nparts > 1 ? make_loopback_comm() : make_nccl_comm(nccl_comm, rank, nranks);
  }
  for (Hier* h : g.parts) {
    octmg_status st = set_ownership(*h, P);
    if (st) return fail(st);
  }
  if (P) {
    octmg_status st = build_links(g, *P, s);
    if (st) return fail(st);
  }
  octmg_status st = build_schedule(g);
  if (st) return fail(st);
  *out = hh;
  return OCTMG_OK;
}

ApplyArgs apply_args(const Hier& h) {
  const Tree& T = *h.tree;
  ApplyArgs a;
  a.tiles = h.apply_tiles; a.ntiles = h.n_apply_tiles;
  if (h.nranks == 1 && h.n_apply_tiles == h.tree->NL) a.tiles = nullptr;  // identity: skip the indirection
  a.tile = T.tile; a.nbr = T.nbr; a.child = T.child; a.coef = h.coef; a.glayer_val = h.glayer_val;
  a.glayer = T.glayer; a.dtile = h.dtile; a.dval = h.dval; a.z = nullptr; a.q = nullptr;
  a.pbar = h.pbar; a.ifaces = h.ifaces; a.n_ifaces = h.n_ifaces;
  a.partial = nullptr; a.counter = nullptr; a.sc = h.sc; a.NL = T.NL;
  a.irr_inline = 0;
  for (int l = 0; l <= T.L; ++l) a.irr_inline |= h.lvl_ghost[l] ? 1 : 0;
  a.lean = h.n_dtiles == 0 ? 1 : 0;
  a.sumq = 0;
  return a;
}

}  // namespace
}  // namespace octmg

extern "C" {

octmg_status octmg_setup_hierarchy(octmg_tree* tree, const uint8_t* kind, const float* face_beta,
                                   const float* face_frac, const octmg_mg_params* params, octmg_stream stream,
                                   octmg_hier** out) {
  if (!tree || !kind || !out) { set_error("null argument"); return OCTMG_E_INVALID; }
  *out = nullptr;
  const Tree& T = tree->t;
  return make_group(tree, 1, T.rank, T.nranks, T.nccl_comm, kind, face_beta, face_frac, params, (cudaStream_t)stream,
                    out);
}

octmg_status octmg_setup_hierarchy_gmg(octmg_tree* tree, const uint8_t* kind, const float* face_beta,
                                       const float* face_frac, const uint8_t* kind_inner,
                                       const float* face_beta_inner, const float* face_frac_inner,
                                       const octmg_mg_params* params, octmg_stream stream, octmg_hier** out) {
  if (!tree || !kind || !kind_inner || !out) { set_error("null argument"); return OCTMG_E_INVALID; }
  *out = nullptr;
  const Tree& T = tree->t;
  if (T.nranks > 1) { set_error("the GMG comparison mode is single-part only"); return OCTMG_E_INVALID; }
  return make_group(tree, 1, 0, 1, nullptr, kind, face_beta, face_frac, params, (cudaStream_t)stream, out,
                    kind_inner, face_beta_inner, face_frac_inner);
}

octmg_status octmg_setup_hierarchy_loopback(octmg_tree* tree, int32_t nparts, const uint8_t* kind,
                                            const float* face_beta, const float* face_frac,
                                            const octmg_mg_params* params, octmg_stream stream, octmg_hier** out) {
  if (!tree || !kind || !out || nparts < 1 || nparts > 64) { set_error("bad argument"); return OCTMG_E_INVALID; }
  *out = nullptr;
  return make_group(tree, nparts, 0, nparts, nullptr, kind, face_beta, face_frac, params, (cudaStream_t)stream, out);
}

octmg_status octmg_partition_info(const octmg_hier* hh, int32_t part, int32_t* lg, int32_t* rank, int32_t* nranks,
                                  int32_t* own_leaf_begin, int32_t* own_leaf_count) {
  if (!hh || part < 0 || part >= (int)hh->g.parts.size()) { set_error("bad argument"); return OCTMG_E_INVALID; }
  const Hier& h = *hh->g.parts[part];
  if (lg) *lg = h.lg;
  if (rank) *rank = h.rank;
  if (nranks) *nranks = h.nranks;
  for (int l = 0; l <= h.tree->L; ++l) {
    if (own_leaf_begin) own_leaf_begin[l] = h.own_lb[l];
    if (own_leaf_count) own_leaf_count[l] = h.own_lc[l];
  }
  return OCTMG_OK;
}

octmg_status octmg_nccl_unique_id(void* out128) {
  if (!out128) { set_error("null argument"); return OCTMG_E_INVALID; }
  return nccl_unique_id(out128);
}

octmg_status octmg_nccl_comm_init(int32_t rank, int32_t nranks, const void* id128, void** comm) {
  if (!id128 || !comm) { set_error("null argument"); return OCTMG_E_INVALID; }
  return nccl_comm_init(rank, nranks, id128, comm);
}

void octmg_nccl_comm_destroy(void* comm) { nccl_comm_destroy(comm); }

octmg_status octmg_partition_plan_host(const int32_t* tiles4, const int32_t* nbr, const int32_t* parent,
                                       const int32_t* child, int32_t NL, int32_t NI, int32_t L,
                                       const int32_t* level_counts, int32_t nranks, int32_t* lg_out,
                                       int32_t* owner_out, int32_t* n_items_out, int32_t* items_out,
                                       int64_t items_cap, int64_t gather_below_cells) {
  if (!tiles4 || !nbr || !parent || !level_counts || !lg_out || !owner_out || !n_items_out || nranks < 1 ||
      L < 0 || L > MAXL) {
    set_error("bad argument");
    return OCTMG_E_INVALID;
  }
  static thread_local int lb[MAXL + 1], lc[MAXL + 1], ib[MAXL + 1], ic[MAXL + 1];
  int accl = 0, acci = NL;
  for (int l = L; l >= 0; --l) {
    lb[l] = accl; lc[l] = level_counts[4 * l + 1]; accl += lc[l];
    ib[l] = acci; ic[l] = level_counts[4 * l + 3]; acci += ic[l];
  }
  PartInput in;
  in.L = L; in.NL = NL; in.NI = NI;
  in.lb = lb; in.lc = lc; in.ib = ib; in.ic = ic;
  const int T = NL + NI;
  in.tiles4.assign(tiles4, tiles4 + (size_t)T * 4);
  in.nbr.assign(nbr, nbr + (size_t)T * 6);
  in.parent.assign(parent, parent + T);
  if (NI) in.child.assign(child, child + (size_t)NI * 8);
  in.morton.resize(T);
  for (int t = 0; t < T; ++t) in.morton[t] = morton3h(in.tiles4[4 * t + 1], in.tiles4[4 * t + 2], in.tiles4[4 * t + 3]);
  PartPlan P;
  if (gather_below_cells < 0) { set_error("gather_below_cells < 0"); return OCTMG_E_INVALID; }
  const int lg = choose_partition_level(in, nranks, gather_below_cells);
  build_partition(in, nranks, lg, P);
  *lg_out = lg;
  std::memcpy(owner_out, P.owner.data(), sizeof(int32_t) * T);
  int64_t k = 0;
  for (size_t q = 0; q < P.items.size(); ++q) {
    n_items_out[q] = (int32_t)P.items[q].size();
    for (const HaloItem& it : P.items[q]) {
      if (items_out && k + 2 <= 2 * items_cap) { items_out[k] = it.tile; items_out[k + 1] = it.kind; }
      k += 2;
    }
  }
  if (k > 2 * items_cap) { set_error("items buffer too small"); return OCTMG_E_INVALID; }
  return OCTMG_OK;
}

octmg_status octmg_divergence(const octmg_hier* hh, const float* face_frac, const float* u6, float* b,
                              octmg_stream stream) {
  if (!hh || !u6 || !b) { set_error("null argument"); return OCTMG_E_INVALID; }
  if (hh->g.parts.size() != 1 || hh->g.parts[0]->nranks != 1) {
    set_error("octmg_divergence: single-part hierarchies only");
    return OCTMG_E_INVALID;
  }
  return divergence(*hh->g.parts[0], face_frac, u6, b, (cudaStream_t)stream);
}

octmg_status octmg_subtract_gradient(const octmg_hier* hh, const uint8_t* kind, const float* face_beta,
                                     const float* face_frac, const float* p, float* u6, octmg_stream stream) {
  if (!hh || !kind || !p || !u6) { set_error("null argument"); return OCTMG_E_INVALID; }
  if (hh->g.parts.size() != 1 || hh->g.parts[0]->nranks != 1) {
    set_error("octmg_subtract_gradient: single-part hierarchies only");
    return OCTMG_E_INVALID;
  }
  return subtract_gradient(*hh->g.parts[0], kind, face_beta, face_frac, p, u6, (cudaStream_t)stream);
}

octmg_status octmg_band_tiles(const int32_t* ext3, int32_t l0, int32_t extra, const double* centre3, double radius,
                             int32_t grade_repair, octmg_tile* out_host, int64_t cap, int64_t* n_out,
                             octmg_stream stream) {
  return band_tiles(ext3, l0, extra, centre3, radius, grade_repair, out_host, cap, n_out, (cudaStream_t)stream);
}

octmg_status octmg_tank_fields(const octmg_tree* tree, const double* centre3, double radius, uint8_t* kind,
                               float* face_frac, float* b, octmg_stream stream) {
  if (!tree || !centre3 || !kind || !face_frac || !b) { set_error("null argument"); return OCTMG_E_INVALID; }
  return tank_fields(tree->t, centre3, radius, kind, face_frac, b, (cudaStream_t)stream);
}

octmg_status octmg_tank_fields_inner(const octmg_tree* tree, const double* centre3, double radius, uint8_t* kind_inner,
                                     float* face_frac_inner, octmg_stream stream) {
  if (!tree || !centre3 || !kind_inner || !face_frac_inner) { set_error("null argument"); return OCTMG_E_INVALID; }
  return tank_fields_inner(tree->t, centre3, radius, kind_inner, face_frac_inner, (cudaStream_t)stream);
}

static octmg_status export_store(const octmg_hier* hh, float* host_dst, size_t bytes, bool cycle) {
  if (!hh || !host_dst) { set_error("null argument"); return OCTMG_E_INVALID; }
  const Hier& h = *hh->g.parts[0];
  const float* src = cycle ? h.ccoef : h.coef;
  size_t need = (size_t)h.tree->T * TB3 * sizeof(float4);
  if (bytes != need) { set_error("export buffer size mismatch"); return OCTMG_E_INVALID; }
  OCTMG_CUDA(cudaDeviceSynchronize());
  std::vector<float> soa((size_t)h.tree->T * TB3 * 4);
  OCTMG_CUDA(cudaMemcpy(soa.data(), src, need, cudaMemcpyDeviceToHost));
  // SoA planes per tile in slot order -> the ABI's record order (c, c_x-, c_y-, c_z-) per
  // cell in natural order
  for (size_t t = 0; t < (size_t)h.tree->T; ++t)
    for (int sl = 0; sl < TB3; ++sl) {
      const size_t i = t * TB3 + sl, o = t * TB3 + slot_nat(sl);
      for (int k = 0; k < 4; ++k) host_dst[4 * o + k] = soa[cidx(i, k)];
    }
  return OCTMG_OK;
}

octmg_status octmg_hier_export_coefs(const octmg_hier* hh, float* host_dst, size_t bytes) {
  return export_store(hh, host_dst, bytes, false);
}

octmg_status octmg_hier_export_cycle_coefs(const octmg_hier* hh, float* host_dst, size_t bytes) {
  return export_store(hh, host_dst, bytes, true);
}

octmg_status octmg_apply(octmg_hier* hh, const float* x, float* y, octmg_stream stream) {
  if (!hh || !x || !y) { set_error("null argument"); return OCTMG_E_INVALID; }
  Group& g = hh->g;
  cudaStream_t s = (cudaStream_t)stream;
  for (Hier* hp : g.parts) {
    Hier& h = *hp;
    // mask the caller's (replicated) x to the active cells: the operator relies on zeros
    launch_mask_copy(x, h.act, h.p1, (int64_t)h.tree->NL * TB3, s);  // caller's order -> slots
    ApplyArgs a = apply_args(h);
    a.z = h.p1;
    a.q = h.q;
    {
      ProfScope ps(h, KC_APPLY, s, (double)h.n_apply_tiles * TB3 * 24.0);  // read x, record; write y
      launch_apply(a, s);
    }
    launch_copy_to_nat(h.q, y, h.own_cells, s);  // each part writes its owned leaf tiles
  }
  g.launches += 3 * (int64_t)g.parts.size();
  OCTMG_CUDA(cudaGetLastError());
  return OCTMG_OK;
}

octmg_status octmg_vcycle(octmg_hier* hh, const float* b, float* u, octmg_stream stream) {
  if (!hh || !b || !u) { set_error("null argument"); return OCTMG_E_INVALID; }
  Group& g = hh->g;
  cudaStream_t s = (cudaStream_t)stream;
  for (Hier* h : g.parts) launch_mask_copy(b, h->act, h->r, (int64_t)h->tree->NL * TB3, s);
  OCTMG_TRY(run_M(g, s));
  for (Hier* h : g.parts) launch_copy_to_nat(h->z, u, h->own_cells, s);  // owned cells of each part
  g.launches += 2 * (int64_t)g.parts.size();
  OCTMG_CUDA(cudaGetLastError());
  return OCTMG_OK;
}

}  // extern "C"

namespace octmg {
namespace {

// The whole PCG loop (Alg. 1 lines 8-13) as ONE CUDA graph with a conditional while node
// (SURVEY 8(a) S12): each body iteration is z = M r, (r, z) and beta, p = z + beta p,
// q = A p and p.q, the x / r update, the null-space projection, and the stopping test,
// which sets the while condition on the device — no host round trip per iteration.  A
// partitioned group (loopback parts, or one NCCL rank) captures the same sequence with its
// transport's halo exchanges and scalar allreduces in the body (every rank runs the same
// number of iterations: the test reads the allreduced sums).
octmg_status build_loop_graph(Group& g, bool ns) {
  Hier& h = *g.parts[0];
  if (!g.graph_stream) OCTMG_CUDA(cudaStreamCreateWithFlags(&g.graph_stream, cudaStreamNonBlocking));
  if (!g.loop) {
    g.loop = (LoopState*)dev_malloc(sizeof(LoopState));
    if (!g.loop) { set_error("device allocation failed (PCG loop state)"); return OCTMG_E_OOM; }
    OCTMG_CUDA(cudaHostAlloc(&g.loop_host, sizeof(LoopState), cudaHostAllocMapped));
    OCTMG_CUDA(cudaHostGetDevicePointer((void**)&g.loop_host_dev, g.loop_host, 0));
  }
  if (g.loop_graph) {
    cudaGraphExecDestroy(g.loop_graph);
    g.loop_graph = nullptr;
  }
  cudaGraph_t graph;
  OCTMG_CUDA(cudaGraphCreate(&graph, 0));
  cudaGraphConditionalHandle hd;
  OCTMG_CUDA(cudaGraphConditionalHandleCreate(&hd, graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hd;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  OCTMG_CUDA(cudaGraphAddNode(&node, graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaStream_t cs = g.graph_stream;
  const int G = vec_grid();
  OCTMG_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  auto seq = [&]() -> octmg_status {
    OCTMG_TRY(launch_ops(g, cs));  // z = M r (with (r, z) when fused into its last pass)
    if (!g.rz_fused)
      for (Hier* p : g.parts) launch_dot_rz(p->r, p->z, p->own_cells, p->partial, p->counter + 2, p->sc, cs, G);
    OCTMG_TRY(allreduce(g, SF_RZ, 1, cs));  // (r, z)
    if (g.comm)
      for (Hier* p : g.parts) launch_set_beta(p->sc, cs);  // beta from the summed (r, z)
    std::vector<Fld> pf;
    for (Hier* p : g.parts) {
      launch_pupdate(p->z, p->p0, p->own_cells, p->sc, true, cs, G);  // p = z + beta p
      pf.push_back(Fld{p->p0, nullptr});
    }
    if (g.comm) OCTMG_TRY(g.comm->exchange(g, 0, 1, pf, cs));  // p of the boundary tiles
    for (Hier* p : g.parts) {
      ApplyArgs a = apply_args(*p);
      a.z = p->p0;
      a.q = p->q;
      a.partial = p->partial;
      a.counter = p->counter + 3;
      a.sumq = ns ? 1 : 0;
      launch_apply(a, cs);  // q = A p, p.q
    }
    OCTMG_TRY(allreduce(g, SF_PQ, 2, cs));  // p.q and sum q
    // x, r update with the null-space projection of r fused in (k_update)
    for (Hier* p : g.parts)
      launch_update(p->xs, p->r, p->p0, p->q, p->own_cells, p->partial, p->counter + 4, p->sc, cs, G, 0.0f,
                    ns ? p->act : nullptr);
    OCTMG_TRY(allreduce(g, SF_RR, 2, cs));
    launch_pcg_check(h.sc, g.loop, (unsigned long long)hd, cs);  // the allreduced sums of part 0
    return OCTMG_OK;
  };
  octmg_status st = seq();
  cudaError_t e = cudaStreamEndCapture(cs, &body);
  if (st != OCTMG_OK) { cudaGraphDestroy(graph); return st; }
  if (e != cudaSuccess) { cudaGraphDestroy(graph); return cuda_status(e, "cudaStreamEndCapture (PCG loop)"); }
  e = cudaGraphInstantiate(&g.loop_graph, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) return cuda_status(e, "cudaGraphInstantiate (PCG loop)");
  g.loop_ns = ns ? 1 : 0;
  return OCTMG_OK;
}

}  // namespace
}  // namespace octmg

extern "C" {

octmg_status octmg_pcg_solve(octmg_hier* hh, const float* b, float* x, const octmg_solve_params* params,
                             octmg_solve_report* report, octmg_stream stream) {
  if (!hh || !b || !x) { set_error("null argument"); return OCTMG_E_INVALID; }
  Group& g = hh->g;
  Hier& h0 = *g.parts[0];
  cudaStream_t s = (cudaStream_t)stream;
  octmg_solve_params prm{1e-6, 200, -1};
  if (params) prm = *params;
  if (!(prm.rtol > 0.0) || prm.max_iters < 1) { set_error("invalid solve parameters"); return OCTMG_E_INVALID; }
  const bool ns = prm.nullspace < 0 ? !h0.any_dirichlet : prm.nullspace == 1;
  const int G = vec_grid();
  const int64_t launches0 = g.launches;
  const int np = (int)g.parts.size();
  Scalars* hs = h0.sc_host;
  int hist_lim = 1 << 30;  // the device-side loop records LOOP_HCAP entries at most
  bool x_copied = false;  // the device loop issues the copy-out with its state read-back
  auto fill = [&](octmg_status st, int iters, bool conv, double rel, double bn) {
    // the iterate (slot order) -> the caller's x (natural order), owned cells of each part
    if (!x_copied) {
      for (Hier* h : g.parts) launch_copy_to_nat(h->xs, x, h->own_cells, s);
      cudaStreamSynchronize(s);
    }
    if (report) {
      report->iters = iters;
      report->converged = conv ? 1 : 0;
      report->rel_residual = rel;
      report->bnorm = bn;
      report->status = st;
      report->kernel_launches = g.launches - launches0;
      report->history_len = report->history ? std::min(std::min(iters, (int)report->history_cap), hist_lim) : 0;
      report->device_loop = hist_lim == LOOP_HCAP ? 1 : 0;
    }
    return st;
  };
  auto fetch = [&]() -> octmg_status {  // the scalars into mapped host memory by a kernel
    launch_copy_words(h0.sc, h0.sc_host_dev, sizeof(Scalars), s);
    OCTMG_CUDA(cudaStreamSynchronize(s));
    return OCTMG_OK;
  };
  auto project = [&]() -> octmg_status {  // r -= mean(r) over all parts, then ||r||^2
    for (Hier* h : g.parts) {
      ProfScope ps(*h, KC_PROJECT, s, (double)h->n_apply_tiles * TB3 * 8.125);  // read r, mask; write r
      launch_project(h->r, h->act, h->own_cells, h->partial, h->counter + 1, h->sc, s, G);
    }
    g.launches += np;
    return allreduce(g, SF_RR, 2, s);  // ||r||^2 and sum r of the projected r
  };
  auto dot_rz = [&]() -> octmg_status {
    if (!g.rz_fused) {  // (else summed by the last pass of M)
      for (Hier* h : g.parts) {
        ProfScope ps(*h, KC_DOT, s, (double)h->n_apply_tiles * TB3 * 8.0);
        launch_dot_rz(h->r, h->z, h->own_cells, h->partial, h->counter + 2, h->sc, s, G);
      }
      g.launches += np;
    }
    OCTMG_TRY(allreduce(g, SF_RZ, 1, s));
    if (g.comm) {  // beta from the summed (r, z)
      for (Hier* h : g.parts) launch_set_beta(h->sc, s);
      g.launches += np;
    }
    return OCTMG_OK;
  };
  for (Hier* h : g.parts) {
    ProfScope ps(*h, KC_INIT, s, (double)h->n_apply_tiles * TB3 * 12.125);  // read b, mask; write r, x
    launch_init(b, h->act, h->r, h->xs, h->own_cells, h->partial, h->counter, h->sc, s, G);
  }
  g.launches += np;
  OCTMG_TRY(allreduce(g, SF_RR, 2, s));
  if (ns) OCTMG_TRY(project());
  OCTMG_TRY(fetch());
  if (!std::isfinite(hs->sum_rr)) { set_error("non-finite right-hand side"); return fill(OCTMG_E_NONFINITE, 0, false, 0, 0); }
  const double bn = std::sqrt(hs->sum_rr);
  if (bn == 0.0) return fill(OCTMG_OK, 0, true, 0.0, 0.0);
  const char* gl = getenv("OCTMG_GRAPH_LOOP");  // default on for single-part hierarchies; 0: host loop
  bool device_loop = !(gl && atoi(gl) == 0) && !profiling(g) && !g.loop_unavailable;
  if (device_loop && (!g.loop_graph || g.loop_ns != (ns ? 1 : 0))) {
    // a driver without conditional nodes, or a schedule variant whose launches a
    // conditional body cannot hold (cooperative / cluster launches): fall back to the
    // host-driven loop for this hierarchy from now on
    if (build_loop_graph(g, ns) != OCTMG_OK) {
      cudaGetLastError();
      g.loop_unavailable = true;
      device_loop = false;
    }
  }
  if (device_loop) {
    // the device-side loop: one graph launch, one synchronisation per solve
    LoopState* L = g.loop_host;
    L->bn = bn;
    L->rtol = prm.rtol;
    L->rel = 1.0;
    L->k = 0;
    L->max_iters = prm.max_iters;
    L->status = 0;
    L->converged = 0;
    launch_copy_words(g.loop_host_dev, g.loop, offsetof(LoopState, hist), s);  // read over PCIe by a kernel
    // beta = 0 on the first iteration: rho = inf, p = 0
    for (Hier* h : g.parts) {
      launch_set_rho_inf(h->sc, s);
      OCTMG_CUDA(cudaMemsetAsync(h->p0, 0, sizeof(float) * (size_t)h->tree->NL * TB3, s));
    }
    OCTMG_CUDA(cudaGraphLaunch(g.loop_graph, s));
    launch_copy_words(g.loop, g.loop_host_dev, sizeof(LoopState), s);
    for (Hier* h : g.parts) launch_copy_to_nat(h->xs, x, h->own_cells, s);  // the result, same sync
    x_copied = true;
    OCTMG_CUDA(cudaStreamSynchronize(s));
    const int kk = L->k;
    // per iteration: the cycle, dot_rz, p update, apply + finish, x/r update, projection, check
    g.launches += (int64_t)kk * (schedule_kernels(g) + np * (6 - (g.rz_fused ? 1 : 0) + (g.comm ? 1 : 0)) + 1 +
                                 inner_mean_kernels(g));
    hist_lim = LOOP_HCAP;
    if (report && report->history) {
      const int nh = std::min(kk, std::min((int)report->history_cap, LOOP_HCAP));
      for (int i = 0; i < nh; ++i) report->history[i] = L->hist[i];
    }
    if (L->status == 9) { set_error("PCG breakdown: p.Ap <= 0"); return fill(OCTMG_E_BREAKDOWN, kk - 1, false, L->rel, bn); }
    if (L->status == 8) { set_error("non-finite PCG scalar"); return fill(OCTMG_E_NONFINITE, kk - 1, false, L->rel, bn); }
    if (L->converged) return fill(OCTMG_OK, kk, true, L->rel, bn);
    set_error("PCG did not converge within max_iters");
    return fill(OCTMG_E_MAXITER, kk, false, L->rel, bn);
  }
  OCTMG_TRY(run_M(g, s));
  OCTMG_TRY(dot_rz());
  int k = 0;
  double rel = 1.0;
  // direction update p = z + beta p (own cells, in place), halo of p, then q = A p with
  // the fp64 p.q
  while (true) {
    std::vector<Fld> pf;
    for (Hier* h : g.parts) {
      ProfScope ps(*h, KC_PUPDATE, s, (double)h->n_apply_tiles * TB3 * (k > 0 ? 12.0 : 8.0));  // read z, p; write p
      launch_pupdate(h->z, h->p0, h->own_cells, h->sc, k > 0, s, G);
      pf.push_back(Fld{h->p0, nullptr});
    }
    g.launches += np;
    if (g.comm) OCTMG_TRY(g.comm->exchange(g, 0, 1, pf, s));  // p of the boundary tiles
    for (Hier* h : g.parts) {
      ApplyArgs a = apply_args(*h);
      a.z = h->p0;
      a.q = h->q;
      a.partial = h->partial;
      a.counter = h->counter + 3;
      a.sumq = ns ? 1 : 0;
      {
        // read p, record; write q
        ProfScope ps(*h, KC_APPLY, s, (double)h->n_apply_tiles * TB3 * 24.0);
        launch_apply(a, s);
      }
    }
    g.launches += 3 * np + inner_mean_kernels(g);  // (inner-face means,) apply, chunk sums, finish
    OCTMG_TRY(allreduce(g, SF_PQ, 2, s));  // p.q and sum q
    for (Hier* h : g.parts) {
      // read x, r, p, q (+ the activity bits with the fused projection); write x, r
      ProfScope ps(*h, KC_UPDATE, s, (double)h->n_apply_tiles * TB3 * (ns ? 24.125 : 24.0));
      launch_update(h->xs, h->r, h->p0, h->q, h->own_cells, h->partial, h->counter + 4, h->sc, s, G, 0.0f,
                    ns ? h->act : nullptr);
    }
    g.launches += np;
    OCTMG_TRY(allreduce(g, SF_RR, 2, s));
    OCTMG_CUDA(cudaGetLastError());
    OCTMG_TRY(fetch());
    if (hs->flags & 1) {
      set_error("PCG breakdown: p.Ap <= 0");
      return fill(OCTMG_E_BREAKDOWN, k, false, rel, bn);
    }
    if (!std::isfinite(hs->sum_rr)) { set_error("non-finite PCG scalar"); return fill(OCTMG_E_NONFINITE, k, false, rel, bn); }
    k++;
    rel = std::sqrt(hs->sum_rr) / bn;
    if (report && report->history && k - 1 < report->history_cap) report->history[k - 1] = rel;
    if (rel <= prm.rtol) return fill(OCTMG_OK, k, true, rel, bn);
    if (k >= prm.max_iters) { set_error("PCG did not converge within max_iters"); return fill(OCTMG_E_MAXITER, k, false, rel, bn); }
    OCTMG_TRY(run_M(g, s));
    OCTMG_TRY(dot_rz());
  }
}

// Multigrid as a standalone solver: x += M r, r -= A (M r).
octmg_status octmg_mg_solve(octmg_hier* hh, const float* b, float* x, const octmg_solve_params* params,
                            octmg_solve_report* report, octmg_stream stream) {
  if (!hh || !b || !x) { set_error("null argument"); return OCTMG_E_INVALID; }
  Group& g = hh->g;
  Hier& h0 = *g.parts[0];
  cudaStream_t s = (cudaStream_t)stream;
  octmg_solve_params prm{1e-6, 200, -1};
  if (params) prm = *params;
  if (!(prm.rtol > 0.0) || prm.max_iters < 1) { set_error("invalid solve parameters"); return OCTMG_E_INVALID; }
  const bool ns = prm.nullspace < 0 ? !h0.any_dirichlet : prm.nullspace == 1;
  const int G = vec_grid();
  const int64_t launches0 = g.launches;
  const int np = (int)g.parts.size();
  Scalars* hs = h0.sc_host;
  bool x_copied = false;  // the device loop issues the copy-out with its state read-back
  auto fill = [&](octmg_status st, int iters, bool conv, double rel, double bn) {
    // the iterate (slot order) -> the caller's x (natural order), owned cells of each part
    if (!x_copied) {
      for (Hier* h : g.parts) launch_copy_to_nat(h->xs, x, h->own_cells, s);
      cudaStreamSynchronize(s);
    }
    if (report) {
      report->iters = iters;
      report->converged = conv ? 1 : 0;
      report->rel_residual = rel;
      report->bnorm = bn;
      report->status = st;
      report->kernel_launches = g.launches - launches0;
      report->history_len = report->history ? std::min(iters, (int)report->history_cap) : 0;
      report->device_loop = 0;
    }
    return st;
  };
  auto fetch = [&]() -> octmg_status {  // the scalars into mapped host memory by a kernel
    launch_copy_words(h0.sc, h0.sc_host_dev, sizeof(Scalars), s);
    OCTMG_CUDA(cudaStreamSynchronize(s));
    return OCTMG_OK;
  };
  auto project = [&]() -> octmg_status {
    for (Hier* h : g.parts) {
      ProfScope ps(*h, KC_PROJECT, s, (double)h->n_apply_tiles * TB3 * 8.125);
      launch_project(h->r, h->act, h->own_cells, h->partial, h->counter + 1, h->sc, s, G);
    }
    g.launches += np;
    return allreduce(g, SF_RR, 2, s);  // ||r||^2 and sum r
  };
  for (Hier* h : g.parts) {
    ProfScope ps(*h, KC_INIT, s, (double)h->n_apply_tiles * TB3 * 12.125);
    launch_init(b, h->act, h->r, h->xs, h->own_cells, h->partial, h->counter, h->sc, s, G);
  }
  g.launches += np;
  OCTMG_TRY(allreduce(g, SF_RR, 2, s));
  if (ns) OCTMG_TRY(project());
  OCTMG_TRY(fetch());
  if (!std::isfinite(hs->sum_rr)) { set_error("non-finite right-hand side"); return fill(OCTMG_E_NONFINITE, 0, false, 0, 0); }
  const double bn = std::sqrt(hs->sum_rr);
  if (bn == 0.0) return fill(OCTMG_OK, 0, true, 0.0, 0.0);
  int k = 0;
  double rel = 1.0;
  while (true) {
    OCTMG_TRY(run_M(g, s));  // z = M r (z = leaf part of the cycle's u)
    for (Hier* h : g.parts) {
      ApplyArgs a = apply_args(*h);
      a.z = h->z;      // zero on inactive cells (the cycle writes active cells only, zeros the rest)
      a.q = h->q;      // A z
      a.partial = nullptr;
      ProfScope ps(*h, KC_APPLY, s, (double)h->n_apply_tiles * TB3 * 24.0);  // read z, record; write q
      launch_apply(a, s);
    }
    g.launches += np;
    for (Hier* h : g.parts) {
      ProfScope ps(*h, KC_UPDATE, s, (double)h->n_apply_tiles * TB3 * 24.0);
      launch_update(h->xs, h->r, h->z, h->q, h->own_cells, h->partial, h->counter + 4, h->sc, s, G, 1.0f);
    }
    g.launches += np;
    OCTMG_TRY(allreduce(g, SF_RR, 2, s));
    if (ns) OCTMG_TRY(project());
    OCTMG_CUDA(cudaGetLastError());
    OCTMG_TRY(fetch());
    if (!std::isfinite(hs->sum_rr)) { set_error("non-finite residual"); return fill(OCTMG_E_NONFINITE, k, false, rel, bn); }
    k++;
    rel = std::sqrt(hs->sum_rr) / bn;
    if (report && report->history && k - 1 < report->history_cap) report->history[k - 1] = rel;
    if (rel <= prm.rtol) return fill(OCTMG_OK, k, true, rel, bn);
    if (k >= prm.max_iters) { set_error("multigrid did not converge within max_iters"); return fill(OCTMG_E_MAXITER, k, false, rel, bn); }
  }
}

octmg_status octmg_profile_enable(octmg_hier* hh, int32_t on) {
  if (!hh) { set_error("null argument"); return OCTMG_E_INVALID; }
  for (Hier* hp : hh->g.parts) {
    Hier& h = *hp;
    h.profiling = on != 0;
    h.events.clear();
    h.event_next = 0;
    for (int c = 0; c < KC_COUNT; ++c) { h.prof_ms[c] = 0.0; h.prof_cnt[c] = 0; h.prof_bytes[c] = 0.0; }
    for (int l = 0; l <= MAXL; ++l)
      for (int c = 0; c < KC_COUNT; ++c) { h.prof_lvl_ms[l][c] = 0.0; h.prof_lvl_cnt[l][c] = 0; h.prof_lvl_bytes[l][c] = 0.0; }
  }
  return OCTMG_OK;
}

namespace {
octmg_status prof_collect(octmg::Hier& h) {
  OCTMG_CUDA(cudaDeviceSynchronize());
  for (auto& ev : h.events) {
    float t = 0.0f;
    OCTMG_CUDA(cudaEventElapsedTime(&t, ev.a, ev.b));
    h.prof_ms[ev.cls] += t;
    h.prof_cnt[ev.cls] += 1;
    h.prof_bytes[ev.cls] += ev.bytes;
    if (ev.level >= 0 && ev.level <= octmg::MAXL) {
      h.prof_lvl_ms[ev.level][ev.cls] += t;
      h.prof_lvl_cnt[ev.level][ev.cls] += 1;
      h.prof_lvl_bytes[ev.level][ev.cls] += ev.bytes;
    }
  }
  h.events.clear();
  h.event_next = 0;
  return OCTMG_OK;
}
}  // namespace

octmg_status octmg_profile_read_level(octmg_hier* hh, int32_t level, double* ms, int64_t* counts, double* bytes,
                                      int32_t cap, int32_t* n) {
  if (!hh || !n || level < 0 || level > octmg::MAXL) { set_error("null argument or level out of range"); return OCTMG_E_INVALID; }
  Hier& h = *hh->g.parts[0];
  OCTMG_TRY(prof_collect(h));
  int k = 0;
  for (int c = 0; c < KC_COUNT && k < cap; ++c, ++k) {
    if (ms) ms[k] = h.prof_lvl_ms[level][c];
    if (counts) counts[k] = h.prof_lvl_cnt[level][c];
    if (bytes) bytes[k] = h.prof_lvl_bytes[level][c];
  }
  *n = k;
  return OCTMG_OK;
}

octmg_status octmg_profile_read(octmg_hier* hh, const char** names, double* ms, int64_t* counts, double* bytes,
                                int32_t cap, int32_t* n) {
  if (!hh || !n) { set_error("null argument"); return OCTMG_E_INVALID; }
  Hier& h = *hh->g.parts[0];
  OCTMG_TRY(prof_collect(h));
  int k = 0;
  for (int c = 0; c < KC_COUNT && k < cap; ++c, ++k) {
    if (names) names[k] = kclass_name[c];
    if (ms) ms[k] = h.prof_ms[c];
    if (counts) counts[k] = h.prof_cnt[c];
    if (bytes) bytes[k] = h.prof_bytes[c];
  }
  *n = k;
  return OCTMG_OK;
}

void octmg_hier_destroy(octmg_hier* h) { delete h; }
void octmg_tree_destroy(octmg_tree* t) { delete t; }

}  // extern "C"
