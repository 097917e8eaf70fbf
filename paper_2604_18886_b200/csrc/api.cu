// C-ABI entry points (include/octmg.h), hierarchy management, the unrolled mu-cycle
// schedule (captured once into a CUDA graph) and the PCG driver (Alg. 1).
#include <algorithm>
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

const char* kclass_name[KC_COUNT] = {"smooth_pre_restrict", "smooth_post_prolong", "coarsest", "fas_rhs",
                                     "smooth_coarse_levels", "apply", "pcg_update", "dot_rz", "project",
                                     "init", "setup", "memset"};

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

// Tiles of each level in rank order (slab-major: z, then Morton of (x, y)) and the lag D =
// 1 + the largest rank gap between same-level face neighbours (host, once per hierarchy).
octmg_status build_orders(Hier& h) {
  const Tree& T = *h.tree;
  std::vector<int4> tile(T.T);
  std::vector<int> nbr((size_t)T.T * 6);
  OCTMG_CUDA(cudaMemcpy(tile.data(), T.tile, sizeof(int4) * T.T, cudaMemcpyDeviceToHost));
  OCTMG_CUDA(cudaMemcpy(nbr.data(), T.nbr, sizeof(int) * 6 * T.T, cudaMemcpyDeviceToHost));
  auto m2 = [](uint32_t x, uint32_t y) {
    uint64_t m = 0;
    for (int b = 0; b < 21; ++b) m |= ((uint64_t)((x >> b) & 1) << (2 * b)) | ((uint64_t)((y >> b) & 1) << (2 * b + 1));
    return m;
  };
  std::vector<int> order;
  order.reserve(T.T);
  std::vector<int> rank(T.T, -1);
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
    for (size_t r = 0; r < ts.size(); ++r) rank[ts[r]] = (int)r;
    order.insert(order.end(), ts.begin(), ts.end());
    int D = 1;
    for (int t : ts)
      for (int f = 0; f < 6; ++f) {
        int n = nbr[6 * (size_t)t + f];
        if (n >= 0) D = std::max(D, rank[n] - rank[t] + 1);
      }
    h.lvl_D[l] = D;
  }
  int* d;
  OCTMG_CUDA(cudaMalloc(&d, sizeof(int) * std::max<size_t>(order.size(), 1)));
  h.allocs.push_back(d);
  OCTMG_CUDA(cudaMemcpy(d, order.data(), sizeof(int) * order.size(), cudaMemcpyHostToDevice));
  h.order = d;
  return OCTMG_OK;
}

// issue order of the (stage, rank) items of a level: by key = rank + stage * D
int get_list(Hier& h, int level, int S) {
  for (size_t k = 0; k < h.lists.size(); ++k)
    if (h.lists[k].level == level && h.lists[k].nstages == S) return (int)k;
  const int n = h.lvl_n[level], D = h.lvl_D[level];
  std::vector<int> items;
  items.reserve((size_t)n * S);
  for (int64_t key = 0; key < n + (int64_t)(S - 1) * D; ++key)
    for (int s = S - 1; s >= 0; --s) {
      int64_t r = key - (int64_t)s * D;
      if (r >= 0 && r < n) items.push_back((s << 24) | (int)r);
    }
  ItemList L{level, S, nullptr, (int)items.size()};
  if (cudaMalloc(&L.items, sizeof(int) * std::max<size_t>(items.size(), 1)) != cudaSuccess) return -1;
  h.allocs.push_back(L.items);
  cudaMemcpy(L.items, items.data(), sizeof(int) * items.size(), cudaMemcpyHostToDevice);
  h.lists.push_back(L);
  return (int)h.lists.size() - 1;
}

struct Builder {
  Hier& h;
  int epoch = 1;
  int counters = 0;
  bool ok = true;
  void smooth(int l, const std::vector<int>& st) {
    Op op{};
    op.kind = 0;
    op.level = l;
    op.list = get_list(h, l, (int)st.size());
    if (op.list < 0) ok = false;
    op.epoch = epoch;
    epoch += (int)st.size() + 1;
    op.counter = counters++;
    op.nstages = (int)st.size();
    for (size_t k = 0; k < st.size(); ++k) op.stage[k] = st[k];
    h.ops.push_back(op);
  }
  // colour passes of `iters` RBGS iterations, red first or black first
  static void passes(std::vector<int>& st, int iters, bool red_first) {
    for (int k = 0; k < iters; ++k) {
      st.push_back(stage_desc(red_first ? 0 : 1, SM_PLAIN));
      st.push_back(stage_desc(red_first ? 1 : 0, SM_PLAIN));
    }
  }
  static void first_two(std::vector<int>& st, int m1, int m2) {
    st[0] = (st[0] & 1) | (m1 << 1);
    st[1] = (st[1] & 1) | (m2 << 1);
  }
  // Alg. 4 at level l; fas_first: first of the mu calls from level l+1 (forms the FAS rhs)
  void fas(int l, bool fas_first) {
    const Tree& T = *h.tree;
    if (l < T.L && fas_first && T.ic[l] > 0) {
      Op op{};
      op.kind = 1;
      op.level = l;
      h.ops.push_back(op);
    }
    std::vector<int> st;
    if (l == 0) {
      int nb = h.prm.nu_coarsest;
      passes(st, nb / 2, true);
      passes(st, nb - nb / 2, false);
      if (l == T.L) first_two(st, SM_ZERO1, SM_ZERO2);
      smooth(0, st);
      return;
    }
    passes(st, h.prm.nu_pre, true);
    if (l == T.L) first_two(st, SM_ZERO1, SM_ZERO2);
    st.push_back(stage_desc(0, SM_RESTRICT));
    smooth(l, st);
    for (int k = 0; k < h.prm.mu; ++k) fas(l - 1, k == 0);
    std::vector<int> post;
    passes(post, h.prm.nu_post, false);
    first_two(post, SM_PRO1, SM_PRO2);
    smooth(l, post);
  }
};

octmg_status build_schedule(Hier& h) {
  h.ops.clear();
  OCTMG_TRY(build_orders(h));
  Builder b{h};
  const Tree& T = *h.tree;
  Op reset{};
  reset.kind = 3;
  h.ops.push_back(reset);
  if (T.NL > T.lc[T.L]) {
    Op z{};
    z.kind = 2;
    h.ops.push_back(z);  // coarse leaves start the cycle at 0
  }
  b.fas(T.L, false);
  if (!b.ok) { set_error("item list allocation failed"); return OCTMG_E_OOM; }
  h.n_counters = b.counters;
  int* d;
  OCTMG_CUDA(cudaMalloc(&d, sizeof(int) * ((size_t)T.T + h.n_counters + 1)));
  h.allocs.push_back(d);
  h.flags = d;
  h.counters = d + T.T;
  OCTMG_CUDA(cudaMemset(d, 0, sizeof(int) * ((size_t)T.T + h.n_counters + 1)));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, smooth_kernel_ptr(), 256, 0);
  h.smooth_grid = sms * std::max(per, 1);
  return OCTMG_OK;
}

int64_t schedule_kernels(const Hier& h) {
  int64_t n = 0;
  for (const Op& op : h.ops) n += op.kind <= 1;
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
  if (op.kind == 3) {
    ProfScope ps(h, KC_MEMSET, s, 4.0 * ((double)T.T + h.n_counters));
    cudaMemsetAsync(h.flags, 0, sizeof(int) * ((size_t)T.T + h.n_counters), s);
    return;
  }
  if (op.kind == 2) {
    size_t first = (size_t)T.lc[T.L] * TB3;
    ProfScope ps(h, KC_MEMSET, s, 4.0 * ((double)T.NL * TB3 - first));
    cudaMemsetAsync(h.z + first, 0, ((size_t)T.NL * TB3 - first) * sizeof(float), s);
    return;
  }
  const int l = op.level;
  SmoothArgs a;
  a.tile = T.tile; a.nbr = T.nbr; a.parent = T.parent; a.coef = h.coef; a.glayer_val = h.glayer_val;
  a.glayer = T.glayer; a.u = ubuf(h); a.ustar = h.ustar; a.ustar_w = h.ustar; a.b = Fld{h.r, h.binner};
  a.beta = h.prm.beta; a.alpha = h.prm.alpha; a.NL = T.NL;
  a.order = h.order + h.lvl_order_off[l];
  a.n = h.lvl_n[l];
  a.first_tile = T.ib[l];
  a.flags = h.flags;
  a.epoch = op.epoch;
  a.has_prolong = 0;
  if (op.kind == 1) {
    a.items = nullptr; a.nstages = 0; a.counter = nullptr;
    // read u, b, record; write b (inner cells of the level)
    ProfScope ps(h, KC_FASRHS, s, 28.0 * T.ic[l] * TB3);
    launch_fasrhs(a, T.ic[l], s);
    return;
  }
  const ItemList& L = h.lists[op.list];
  a.items = L.items;
  a.nstages = op.nstages;
  a.counter = h.counters + op.counter;
  bool restrict_ = false;
  for (int k = 0; k < op.nstages; ++k) {
    a.stage[k] = op.stage[k];
    if ((op.stage[k] >> 1) == SM_PRO1) a.has_prolong = 1;
    if ((op.stage[k] >> 1) == SM_RESTRICT) restrict_ = true;
  }
  // algorithmic bytes of the launch: every cell's u, b and 16-byte record read once and u
  // written once (28 B/cell); restriction adds the parents' u, u*, b (1.5 B/cell),
  // prolongation the parents' u, u* (1 B/cell)
  double cells = (double)a.n * TB3;
  double bytes = cells * 28.0 + (restrict_ ? 1.5 * cells : 0.0) + (a.has_prolong ? 1.0 * cells : 0.0);
  int cls = l == 0 ? KC_COARSEST : (l < T.L ? KC_SMOOTH_COARSE : (a.has_prolong ? KC_SMOOTH_POST : KC_SMOOTH_PRE));
  int grid = (int)std::min<int64_t>(h.smooth_grid, (int64_t)L.n_items);
  ProfScope ps(h, cls, s, bytes);
  launch_smooth(a, grid, s);
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
  if ((st = halloc(h.allocs, &h.z, NLc))) return fail(st);
  if ((st = halloc(h.allocs, &h.uinA, NIc))) return fail(st);
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
  ApplyArgs a = apply_args(h);
  a.z = x;
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
  launch_mask_copy(b, h.coef, h.r, (int64_t)N, s);
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
    ProfScope ps(h, KC_INIT, s, (double)N * 28.0);  // read b, record; write r, x
    launch_init(b, h.coef, h.r, x, N, h.partial, h.counter, h.sc, s, G);
  }
  h.launches++;
  if (ns) {
    ProfScope ps(h, KC_PROJECT, s, (double)N * 24.0);  // read r, record; write r
    launch_project(h.r, h.coef, N, h.partial, h.counter + 1, h.sc, s, G);
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
    h.launches += 2;
    if (ns) {
      ProfScope ps(h, KC_PROJECT, s, (double)N * 24.0);
      launch_project(h.r, h.coef, N, h.partial, h.counter + 1, h.sc, s, G);
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
