// C-ABI entry points (include/octmg.h), hierarchy management, the unrolled mu-cycle
// schedule (captured once into a CUDA graph) and the PCG driver (Alg. 1).
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "octmg_internal.cuh"

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
                                     "copy_level"};

template <class T>
static octmg_status halloc(std::vector<void*>& list, T** p, size_t count) {
  void* q = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(&q, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    set_error("device allocation failed (" + std::to_string(count * sizeof(T)) + " bytes)");
    return OCTMG_E_OOM;
  }
  list.push_back(q);
  *p = (T*)q;
  return OCTMG_OK;
}

Hier::~Hier() {
  if (graph) cudaGraphExecDestroy(graph);
  if (graph_stream) cudaStreamDestroy(graph_stream);
  for (auto e : event_pool) cudaEventDestroy(e);
  for (void* p : allocs) cudaFree(p);
  if (sc_host) cudaFreeHost(sc_host);
}

// ------------------------------------------------------------------------------------
// schedule of one preconditioner application M (Alg. 4; SURVEY c-6)
// ------------------------------------------------------------------------------------
namespace {

enum { SM_PLAIN = 0, SM_ZERO1 = 1, SM_ZERO2 = 2, SM_PRO1 = 3, SM_PRO2 = 4, SM_RESTRICT = 5 };

inline int stage_desc(int colour, int mode) { return colour | (mode << 1); }

// Tiles of each level in rank order (slab-major: z, then Morton of (x, y)), so that the
// consecutive tiles of a CTA's run share faces (host, once per hierarchy).
octmg_status build_orders(Hier& h) {
  const Tree& T = *h.tree;
  std::vector<int4> tile(T.T);
  OCTMG_CUDA(cudaMemcpy(tile.data(), T.tile, sizeof(int4) * T.T, cudaMemcpyDeviceToHost));
  auto m2 = [](uint32_t x, uint32_t y) {
    uint64_t m = 0;
    for (int b = 0; b < 21; ++b) m |= ((uint64_t)((x >> b) & 1) << (2 * b)) | ((uint64_t)((y >> b) & 1) << (2 * b + 1));
    return m;
  };
  std::vector<int> order;
  order.reserve(T.T);
  for (int l = 0; l <= T.L; ++l) {
    std::vector<int> ts;
    for (int t = T.lb[l]; t < T.lb[l] + T.lc[l]; ++t) ts.push_back(t);
    for (int t = T.ib[l]; t < T.ib[l] + T.ic[l]; ++t) ts.push_back(t);
    std::sort(ts.begin(), ts.end(), [&](int a, int b) {
      if (tile[a].w != tile[b].w) return tile[a].w < tile[b].w;
      return m2(tile[a].y, tile[a].z) < m2(tile[b].y, tile[b].z);
    });
    h.lvl_order_off[l] = (int)order.size();
    h.lvl_n[l] = (int)ts.size();
    order.insert(order.end(), ts.begin(), ts.end());
  }
  int* d;
  OCTMG_CUDA(cudaMalloc(&d, sizeof(int) * std::max<size_t>(order.size(), 1)));
  h.allocs.push_back(d);
  OCTMG_CUDA(cudaMemcpy(d, order.data(), sizeof(int) * order.size(), cudaMemcpyHostToDevice));
  h.order = d;
  return OCTMG_OK;
}

struct Builder {
  Hier& h;
  void stage(int l, int desc) { h.ops.push_back(Op{0, l, desc}); }
  void passes(int l, int iters, bool red_first, int m1, int m2) {
    if (h.rb_fused) {  // one launch per RB iteration, ping-pong A -> B -> A ...
      int cur = 0;
      for (int k = 0; k < iters; ++k) {
        const int zero = (k == 0 && m1 == SM_ZERO1) ? 2 : 0;
        h.ops.push_back(Op{5, l, (red_first ? 0 : 1) | zero, cur, 1 - cur});
        cur = 1 - cur;
      }
      if (cur == 1) h.ops.push_back(Op{6, l, 0, 1, 0});  // odd count: back to the rest buffer
      return;
    }
    for (int k = 0; k < iters; ++k) {
      stage(l, stage_desc(red_first ? 0 : 1, k == 0 ? m1 : SM_PLAIN));
      stage(l, stage_desc(red_first ? 1 : 0, k == 0 ? m2 : SM_PLAIN));
    }
  }
  // Alg. 4 at level l; fas_first: first of the mu calls from level l+1 (forms the FAS rhs)
  void fas(int l, bool fas_first) {
    const Tree& T = *h.tree;
    if (l <= h.sub_K) {  // the rest of the cycle runs on chip in one CTA
      h.ops.push_back(Op{4, l, fas_first ? 1 : 0});
      return;
    }
    if (l < T.L && fas_first && T.ic[l] > 0) h.ops.push_back(Op{1, l, 0});
    const bool finest = l == T.L;
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
    h.ops.push_back(Op{3, l, 0});  // prolongation u += P(u^{l-1} - u*), in place
    passes(l, h.prm.nu_post, false, SM_PLAIN, SM_PLAIN);
  }
};

octmg_status build_schedule(Hier& h) {
  h.ops.clear();
  OCTMG_TRY(build_orders(h));
  const char* rbv = getenv("OCTMG_RB");
  // default: one launch per colour pass; OCTMG_RB=fused selects the fused RB iteration
  // (parity-tested, currently slower: see DESIGN.md "Fused red-black")
  h.rb_fused = (rbv && std::string(rbv) == "fused") ? 1 : ((rbv && std::string(rbv) == "fused_noshell") ? 2 : 0);
  const char* pc = getenv("OCTMG_PASS_CPT");
  h.pass_cpt = pc ? std::max(1, std::min(2, atoi(pc))) : 2;
  const Tree& T = *h.tree;
  const char* sc = getenv("OCTMG_SUBCYCLE");
  h.sub_K = -1;
  if (!(sc && std::string(sc) == "0"))
    for (int l = 0; l <= std::min(T.L, subcycle_max_level()); ++l) {
      if (h.lvl_n[l] > subcycle_max_tiles()) break;
      h.sub_K = l;
    }
  if (T.NL > T.lc[T.L]) h.ops.push_back(Op{2, 0, 0});  // coarse leaves start the cycle at 0
  Builder b{h};
  b.fas(T.L, false);
  return OCTMG_OK;
}

int64_t schedule_kernels(const Hier& h) {
  int64_t n = 0;
  for (const Op& op : h.ops) n += op.kind != 2;
  return n;
}

Fld ubuf(const Hier& h, int which = 0) { return which == 0 ? Fld{h.z, h.uinA} : Fld{h.zB, h.uinB}; }

cudaEvent_t next_event(Hier& h) {
  if (h.event_next == h.event_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    h.event_pool.push_back(e);
  }
  return h.event_pool[h.event_next++];
}

struct ProfScope {
  Hier& h;
  int cls;
  cudaStream_t s;
  cudaEvent_t b = nullptr;
  ProfScope(Hier& hh, int c, cudaStream_t ss, double bytes) : h(hh), cls(c), s(ss) {
    if (h.profiling) {
      cudaEvent_t a = next_event(h);
      b = next_event(h);
      cudaEventRecord(a, s);
      h.events.push_back({cls, bytes, a, b});
    }
  }
  ~ProfScope() {
    if (h.profiling) cudaEventRecord(b, s);
  }
};

void launch_op(Hier& h, const Op& op, cudaStream_t s) {
  const Tree& T = *h.tree;
  if (op.kind == 2) {
    size_t first = (size_t)T.lc[T.L] * TB3;
    ProfScope ps(h, KC_MEMSET, s, 4.0 * ((double)T.NL * TB3 - first));
    cudaMemsetAsync(h.z + first, 0, ((size_t)T.NL * TB3 - first) * sizeof(float), s);
    return;
  }
  const int l = op.level;
  SmoothArgs a;
  a.tile = T.tile; a.nbr = T.nbr; a.parent = T.parent; a.coef = h.coef; a.glayer_val = h.glayer_val;
  a.glayer = T.glayer; a.u = ubuf(h); a.u2 = ubuf(h, 1); a.uc = ubuf(h); a.ustar = h.ustar; a.ustar_w = h.ustar;
  a.b = Fld{h.r, h.binner};
  a.beta = h.prm.beta; a.alpha = h.prm.alpha; a.NL = T.NL;
  a.order = h.order + h.lvl_order_off[l];
  a.n = h.lvl_n[l];
  a.first_tile = T.ib[l];
  a.stage[0] = op.stage;
  if (op.kind == 5) {
    a.u = ubuf(h, op.in_buf);
    a.u2 = ubuf(h, op.out_buf);
    a.stage[0] = op.stage & 1;
    // one HBM pass per RB iteration: read u, b, 16-byte record, write u (28 B/cell)
    ProfScope ps(h, l < T.L ? KC_SMOOTH_COARSE : KC_RBFUSED, s, 28.0 * a.n * TB3);
    launch_rb_fused(a, (op.stage & 2) != 0, s, h.rb_fused != 2);
    return;
  }
  if (op.kind == 6) {
    a.u = ubuf(h, op.in_buf);
    a.u2 = ubuf(h, op.out_buf);
    ProfScope ps(h, KC_COPY, s, 8.0 * a.n * TB3);
    launch_copy_level(a, s);
    return;
  }
  if (op.kind == 4) {
    ProfScope ps(h, KC_SUBCYCLE, s, 0.0);
    launch_subcycle(a, T.L, l, op.stage, h.prm, h.order, h.lvl_order_off, h.lvl_n, T.ib, T.ic, s);
    return;
  }
  if (op.kind == 3) {
    // read u, record; write u (8 + 16 B/cell) + the parents' u, u* (1 B/cell)
    ProfScope ps(h, KC_PROLONG, s, 25.0 * a.n * TB3);
    launch_prolong(a, s);
    return;
  }
  if (op.kind == 1) {
    // read u, b, record; write b (inner cells of the level)
    ProfScope ps(h, KC_FASRHS, s, 28.0 * T.ic[l] * TB3);
    launch_fasrhs(a, T.ic[l], s);
    return;
  }
  const int mode = op.stage >> 1;
  // algorithmic bytes per cell of the level: colour pass = read u, b, 16-byte record, write
  // u (28 B; 24 B when u is known zero); restrict = read u, b, record (24 B) + the parents'
  // u, u*, b (1.5 B); prolongation-fused passes read the parents' u, u* (+1 B)
  const double cells = (double)a.n * TB3;
  double bytes = cells * (mode == SM_RESTRICT ? 25.5 : (mode == SM_ZERO1 ? 24.0 : 28.0));
  if (mode == SM_PRO1 || mode == SM_PRO2) bytes += cells;
  int cls = mode == SM_RESTRICT ? KC_RESTRICT
          : (l == 0 ? KC_COARSEST : (l < T.L ? KC_SMOOTH_COARSE : KC_PASS));
  ProfScope ps(h, cls, s, bytes);
  if (mode == SM_RESTRICT) {
    launch_restrict_direct(a, s);
  } else {
    launch_pass_direct(a, s, a.n >= 1024 ? h.pass_cpt : 1);
  }
}

octmg_status run_M(Hier& h, cudaStream_t s) {
  if (h.profiling) {
    for (const Op& op : h.ops) launch_op(h, op, s);
    OCTMG_CUDA(cudaGetLastError());
    h.launches += schedule_kernels(h);
    return OCTMG_OK;
  }
  if (!h.graph) {
    if (!h.graph_stream) OCTMG_CUDA(cudaStreamCreateWithFlags(&h.graph_stream, cudaStreamNonBlocking));
    cudaGraph_t g;
    OCTMG_CUDA(cudaStreamBeginCapture(h.graph_stream, cudaStreamCaptureModeThreadLocal));
    for (const Op& op : h.ops) launch_op(h, op, h.graph_stream);
    cudaError_t e = cudaStreamEndCapture(h.graph_stream, &g);
    if (e != cudaSuccess) return cuda_status(e, "cudaStreamEndCapture");
    e = cudaGraphInstantiate(&h.graph, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_status(e, "cudaGraphInstantiate");
  }
  OCTMG_CUDA(cudaGraphLaunch(h.graph, s));
  h.launches += schedule_kernels(h);
  return OCTMG_OK;
}

int vec_grid() { return 148 * 4; }

}  // namespace

}  // namespace octmg

using namespace octmg;

extern "C" {

const char* octmg_last_error(void) { return g_err.c_str(); }

const char* octmg_version(void) { return "octmg 0.1.0 (sm_100a, fp32 fields / fp64 dots)"; }

octmg_status octmg_build_tree(const octmg_tree_desc* desc, const octmg_tile* leaf_tiles_host, int64_t n,
                              octmg_stream stream, octmg_tree** out) {
  if (!desc || !leaf_tiles_host || !out) { set_error("null argument"); return OCTMG_E_INVALID; }
  *out = nullptr;
  auto* t = new (std::nothrow) octmg_tree();
  if (!t) { set_error("host allocation failed"); return OCTMG_E_OOM; }
  octmg_status st = build_tree(desc, leaf_tiles_host, n, (cudaStream_t)stream, &t->t);
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

octmg_status octmg_setup_hierarchy(octmg_tree* tree, const uint8_t* kind, const float* face_beta,
                                   const float* face_frac, const octmg_mg_params* params, octmg_stream stream,
                                   octmg_hier** out) {
  if (!tree || !kind || !out) { set_error("null argument"); return OCTMG_E_INVALID; }
  *out = nullptr;
  octmg_mg_params prm{2.0f, 2.0f, 1, 2, 2, 10};
  if (params) prm = *params;
  if (!(prm.alpha > 0.0f) || prm.mu < 1 || prm.mu > 4 || prm.nu_pre < 1 || prm.nu_post < 1 || prm.nu_coarsest < 1) {
    set_error("invalid multigrid parameters (need alpha > 0, 1 <= mu <= 4, nu_* >= 1)");
    return OCTMG_E_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  auto* hh = new (std::nothrow) octmg_hier();
  if (!hh) { set_error("host allocation failed"); return OCTMG_E_OOM; }
  Hier& h = hh->h;
  h.tree = &tree->t;
  h.prm = prm;
  const Tree& T = tree->t;
  size_t NLc = (size_t)T.NL * TB3, NIc = (size_t)T.NI * TB3;
  octmg_status st = OCTMG_OK;
  auto fail = [&](octmg_status e) { delete hh; return e; };
  if ((st = halloc(h.allocs, &h.coef, (size_t)T.T * TB3))) return fail(st);
  if ((st = halloc(h.allocs, &h.glayer_val, (size_t)T.n_glayers * 64))) return fail(st);
  if ((st = halloc(h.allocs, &h.act, NLc / 32))) return fail(st);
  if ((st = halloc(h.allocs, &h.z, NLc))) return fail(st);
  if ((st = halloc(h.allocs, &h.uinA, NIc))) return fail(st);
  if ((st = halloc(h.allocs, &h.zB, NLc))) return fail(st);
  if ((st = halloc(h.allocs, &h.uinB, NIc))) return fail(st);
  if ((st = halloc(h.allocs, &h.binner, NIc))) return fail(st);
  if ((st = halloc(h.allocs, &h.ustar, NIc))) return fail(st);
  if ((st = halloc(h.allocs, &h.r, NLc))) return fail(st);
  if ((st = halloc(h.allocs, &h.p0, NLc))) return fail(st);
  if ((st = halloc(h.allocs, &h.p1, NLc))) return fail(st);
  if ((st = halloc(h.allocs, &h.q, NLc))) return fail(st);
  h.n_partial = std::max<size_t>((size_t)T.NL, 2 * (size_t)vec_grid()) + 16;
  if ((st = halloc(h.allocs, &h.partial, h.n_partial))) return fail(st);
  if ((st = halloc(h.allocs, &h.counter, 16))) return fail(st);
  if ((st = halloc(h.allocs, &h.sc, 1))) return fail(st);
  if (cudaMallocHost(&h.sc_host, sizeof(Scalars)) != cudaSuccess) {
    cudaGetLastError();
    set_error("pinned allocation failed");
    return fail(OCTMG_E_OOM);
  }
  cudaError_t e = cudaMemsetAsync(h.counter, 0, 16 * sizeof(unsigned), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(h.uinA, 0, NIc * sizeof(float) + 0, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(h.z, 0, NLc * sizeof(float), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(h.sc, 0, sizeof(Scalars), s);
  if (e != cudaSuccess) return fail(cuda_status(e, "memset"));
  if ((st = assemble_leaf_coefs(h, kind, face_beta, face_frac, s))) return fail(st);
  if ((st = coarsen_all(h, s))) return fail(st);
  launch_build_mask(h.coef, (int64_t)NLc, h.act, s);
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(cuda_status(e, "setup"));
  if ((st = build_schedule(h))) return fail(st);
  if (e != cudaSuccess) return fail(cuda_status(e, "setup"));
  *out = hh;
  return OCTMG_OK;
}

octmg_status octmg_hier_export_coefs(const octmg_hier* hh, float* host_dst, size_t bytes) {
  if (!hh || !host_dst) { set_error("null argument"); return OCTMG_E_INVALID; }
  const Hier& h = hh->h;
  size_t need = (size_t)h.tree->T * TB3 * sizeof(float4);
  if (bytes != need) { set_error("export buffer size mismatch"); return OCTMG_E_INVALID; }
  OCTMG_CUDA(cudaDeviceSynchronize());
  OCTMG_CUDA(cudaMemcpy(host_dst, h.coef, need, cudaMemcpyDeviceToHost));
  return OCTMG_OK;
}

static ApplyArgs apply_args(const Hier& h) {
  const Tree& T = *h.tree;
  ApplyArgs a;
  a.tile = T.tile; a.nbr = T.nbr; a.child = T.child; a.coef = h.coef; a.glayer_val = h.glayer_val;
  a.glayer = T.glayer; a.z = nullptr; a.pold = nullptr; a.pnew = nullptr; a.q = nullptr;
  a.partial = nullptr; a.counter = nullptr; a.sc = h.sc; a.NL = T.NL; a.use_beta = 0;
  return a;
}

octmg_status octmg_apply(octmg_hier* hh, const float* x, float* y, octmg_stream stream) {
  if (!hh || !x || !y) { set_error("null argument"); return OCTMG_E_INVALID; }
  Hier& h = hh->h;
  cudaStream_t s = (cudaStream_t)stream;
  // mask the caller's x to the active cells (the operator kernel relies on zeros there)
  launch_mask_copy(x, h.act, h.p1, (int64_t)h.tree->NL * TB3, s);
  ApplyArgs a = apply_args(h);
  a.z = h.p1;
  a.q = y;
  {
    ProfScope ps(h, KC_APPLY, s, (double)h.tree->NL * TB3 * 24.0);  // read x, record; write y
    launch_apply(a, s);
  }
  h.launches += 1;
  OCTMG_CUDA(cudaGetLastError());
  return OCTMG_OK;
}

octmg_status octmg_vcycle(octmg_hier* hh, const float* b, float* u, octmg_stream stream) {
  if (!hh || !b || !u) { set_error("null argument"); return OCTMG_E_INVALID; }
  Hier& h = hh->h;
  cudaStream_t s = (cudaStream_t)stream;
  size_t N = (size_t)h.tree->NL * TB3;
  launch_mask_copy(b, h.act, h.r, (int64_t)N, s);
  OCTMG_TRY(run_M(h, s));
  OCTMG_CUDA(cudaMemcpyAsync(u, h.z, N * sizeof(float), cudaMemcpyDeviceToDevice, s));
  OCTMG_CUDA(cudaGetLastError());
  return OCTMG_OK;
}

octmg_status octmg_pcg_solve(octmg_hier* hh, const float* b, float* x, const octmg_solve_params* params,
                             octmg_solve_report* report, octmg_stream stream) {
  if (!hh || !b || !x) { set_error("null argument"); return OCTMG_E_INVALID; }
  Hier& h = hh->h;
  const Tree& T = *h.tree;
  cudaStream_t s = (cudaStream_t)stream;
  octmg_solve_params prm{1e-6, 200, -1};
  if (params) prm = *params;
  if (!(prm.rtol > 0.0) || prm.max_iters < 1) { set_error("invalid solve parameters"); return OCTMG_E_INVALID; }
  const bool ns = prm.nullspace < 0 ? !h.any_dirichlet : prm.nullspace == 1;
  const int64_t N = (int64_t)T.NL * TB3;
  const int G = vec_grid();
  const int64_t launches0 = h.launches;
  Scalars* hs = h.sc_host;
  auto fill = [&](octmg_status st, int iters, bool conv, double rel, double bn) {
    if (report) {
      report->iters = iters;
      report->converged = conv ? 1 : 0;
      report->rel_residual = rel;
      report->bnorm = bn;
      report->status = st;
      report->kernel_launches = h.launches - launches0;
    }
    return st;
  };
  auto fetch = [&]() -> octmg_status {
    OCTMG_CUDA(cudaMemcpyAsync(hs, h.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, s));
    OCTMG_CUDA(cudaStreamSynchronize(s));
    return OCTMG_OK;
  };
  // n_active for the projection mean
  hs->n_active = h.n_active;
  OCTMG_CUDA(cudaMemcpyAsync(&h.sc->n_active, &hs->n_active, sizeof(double), cudaMemcpyHostToDevice, s));
  {
    ProfScope ps(h, KC_INIT, s, (double)N * 12.125);  // read b, mask; write r, x
    launch_init(b, h.act, h.r, x, N, h.partial, h.counter, h.sc, s, G);
  }
  h.launches++;
  if (ns) {
    ProfScope ps(h, KC_PROJECT, s, (double)N * 8.125);  // read r, mask; write r
    launch_project(h.r, h.act, N, h.partial, h.counter + 1, h.sc, s, G);
    h.launches++;
  }
  OCTMG_TRY(fetch());
  if (hs->flags & 2) { set_error("non-finite right-hand side"); return fill(OCTMG_E_NONFINITE, 0, false, 0, 0); }
  const double bn = std::sqrt(hs->rr);
  if (bn == 0.0) return fill(OCTMG_OK, 0, true, 0.0, 0.0);
  OCTMG_TRY(run_M(h, s));
  {
    ProfScope ps(h, KC_DOT, s, (double)N * 8.0);
    launch_dot_rz(h.r, h.z, N, h.partial, h.counter + 2, h.sc, 1, s, G);
  }
  h.launches++;
  float* pcur = h.p0;
  float* pprev = h.p1;
  int k = 0;
  double rel = 1.0;
  while (true) {
    ApplyArgs a = apply_args(h);
    a.z = h.z;
    a.pold = k == 0 ? nullptr : pprev;
    a.pnew = pcur;
    a.q = h.q;
    a.partial = h.partial;
    a.counter = h.counter + 3;
    a.use_beta = k > 0;
    {
      // read z, p_old, record (24 B/leaf); write p, q (8 B/leaf)
      ProfScope ps(h, KC_APPLY, s, (double)N * 32.0);
      launch_apply(a, s);
    }
    {
      ProfScope ps(h, KC_UPDATE, s, (double)N * 24.0);  // read x, r, p, q; write x, r
      launch_update(x, h.r, pcur, h.q, N, h.partial, h.counter + 4, h.sc, s, G);
    }
    h.launches += 3;  // apply, finish_sigma, update
    if (ns) {
      ProfScope ps(h, KC_PROJECT, s, (double)N * 8.125);
      launch_project(h.r, h.act, N, h.partial, h.counter + 1, h.sc, s, G);
      h.launches++;
    }
    OCTMG_CUDA(cudaGetLastError());
    OCTMG_TRY(fetch());
    if (hs->flags & 1) {
      set_error("PCG breakdown: p.Ap <= 0");
      return fill(OCTMG_E_BREAKDOWN, k, false, rel, bn);
    }
    if (hs->flags & 2) { set_error("non-finite PCG scalar"); return fill(OCTMG_E_NONFINITE, k, false, rel, bn); }
    k++;
    rel = std::sqrt(hs->rr) / bn;
    if (report && report->history && k - 1 < report->history_cap) report->history[k - 1] = rel;
    if (rel <= prm.rtol) return fill(OCTMG_OK, k, true, rel, bn);
    if (k >= prm.max_iters) { set_error("PCG did not converge within max_iters"); return fill(OCTMG_E_MAXITER, k, false, rel, bn); }
    OCTMG_TRY(run_M(h, s));
    {
      ProfScope ps(h, KC_DOT, s, (double)N * 8.0);
      launch_dot_rz(h.r, h.z, N, h.partial, h.counter + 2, h.sc, 0, s, G);
    }
    h.launches++;
    std::swap(pcur, pprev);
  }
}

octmg_status octmg_profile_enable(octmg_hier* hh, int32_t on) {
  if (!hh) { set_error("null argument"); return OCTMG_E_INVALID; }
  Hier& h = hh->h;
  h.profiling = on != 0;
  h.events.clear();
  h.event_next = 0;
  for (int c = 0; c < KC_COUNT; ++c) { h.prof_ms[c] = 0.0; h.prof_cnt[c] = 0; h.prof_bytes[c] = 0.0; }
  return OCTMG_OK;
}

octmg_status octmg_profile_read(octmg_hier* hh, const char** names, double* ms, int64_t* counts, double* bytes,
                                int32_t cap, int32_t* n) {
  if (!hh || !n) { set_error("null argument"); return OCTMG_E_INVALID; }
  Hier& h = hh->h;
  OCTMG_CUDA(cudaDeviceSynchronize());
  for (auto& ev : h.events) {
    float t = 0.0f;
    OCTMG_CUDA(cudaEventElapsedTime(&t, ev.a, ev.b));
    h.prof_ms[ev.cls] += t;
    h.prof_cnt[ev.cls] += 1;
    h.prof_bytes[ev.cls] += ev.bytes;
  }
  h.events.clear();
  h.event_next = 0;
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
