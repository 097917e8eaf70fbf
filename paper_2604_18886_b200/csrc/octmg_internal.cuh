// Internal declarations of the octmg CUDA library (sm_100a).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/octmg.h"

namespace octmg {

constexpr int TB = 8;          // tile edge
constexpr int TB3 = 512;       // cells per tile
constexpr int MAXL = OCTMG_MAX_LEVELS - 1;
constexpr int KEY_LEVEL_SHIFT = 58;  // key = (MAXL - level) << 58 | morton(i,j,k) (19 bits/axis)

// ------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------
void set_error(const std::string& msg);
octmg_status cuda_status(cudaError_t e, const char* what);

#define OCTMG_CUDA(call)                                                   \
  do {                                                                     \
    cudaError_t e_ = (call);                                               \
    if (e_ != cudaSuccess) return ::octmg::cuda_status(e_, #call);         \
  } while (0)

#define OCTMG_TRY(call)                                                    \
  do {                                                                     \
    octmg_status s_ = (call);                                              \
    if (s_ != OCTMG_OK) return s_;                                         \
  } while (0)

// Device memory of the handles (octmg_set_allocator): allocations go through the allocator
// current at allocation time, and each pointer is released through the one that made it.
void* dev_malloc(size_t bytes);  // nullptr on failure
void dev_free(void* p);

// ------------------------------------------------------------------------------------
// Tree (device tables + host metadata)
// ------------------------------------------------------------------------------------
struct Tree {
  int ext[3] = {1, 1, 1};
  uint8_t wall[6] = {1, 1, 1, 1, 1, 1};
  int L = 0;
  int NL = 0, NI = 0, T = 0;
  int lb[MAXL + 1] = {}, lc[MAXL + 1] = {}, ib[MAXL + 1] = {}, ic[MAXL + 1] = {};
  int n_glayers = 0;
  int rank = 0, nranks = 1;        // multi-GPU job (octmg_tree_desc)
  void* nccl_comm = nullptr;
  // device
  uint64_t* leaf_keys = nullptr;   // [NL] sorted
  uint64_t* inner_keys = nullptr;  // [NI] sorted
  int4* tile = nullptr;            // [T] (level, i, j, k)
  int* nbr = nullptr;              // [T*6]
  int* parent = nullptr;           // [T]
  int* child = nullptr;            // [NI*8]
  int* glayer = nullptr;           // [NL*3] layer index of the +x/+y/+z ghost face, or -1
  std::vector<void*> allocs;
  ~Tree();
};

// Cell order inside a tile ("slot"): colour-split, red (x+y+z even) cells first,
//   slot = ((x+y+z) & 1) * 256 + (x >> 1) + 4 y + 32 z,
// so a red-black colour pass reads and writes contiguous halves of every field (its own
// colour's values and coefficients, the other colour's neighbour values).  User vectors
// keep the natural order x + 8y + 64z (the ABI's leaf-slot order); the library permutes at
// its boundary.
__host__ __device__ __forceinline__ int cslot(int x, int y, int z) {
  return (((x + y + z) & 1) << 8) | ((x >> 1) + 4 * y + 32 * z);
}
__host__ __device__ __forceinline__ void slot_xyz(int s, int& x, int& y, int& z) {
  const int q = s & 255;
  y = (q >> 2) & 7;
  z = q >> 5;
  x = 2 * (q & 3) + (((s >> 8) + y + z) & 1);
}
__host__ __device__ __forceinline__ int slot_nat(int s) {  // natural offset x + 8y + 64z of a slot
  int x, y, z;
  slot_xyz(s, x, y, z);
  return x + 8 * y + 64 * z;
}

// A field over all tiles, stored as a leaf part and an inner part (either may alias a
// caller / PCG vector).  Tile t's 512 cells start at leaf + t*512 (t < NL) or
// inner + (t-NL)*512.
struct Fld {
  float* leaf;
  float* inner;
};

struct SmoothArgs;
__device__ __forceinline__ float* tptr(const Fld& f, int t, int NL) {
  return t < NL ? f.leaf + (size_t)t * TB3 : f.inner + (size_t)(t - NL) * TB3;
}

// Coefficient store (Eq. 3 compact record (c, c_x-, c_y-, c_z-)), SoA per tile:
// tile t holds 4 planes of 512 floats (c, c_x-, c_y-, c_z-) at coef + t*2048, so a row of
// cells loads each component as a 128-bit vector.  Cell index i = t*512 + cell.
__host__ __device__ __forceinline__ size_t cidx(size_t i, int k) {
  return ((i >> 9) << 11) + ((size_t)k << 9) + (i & 511);
}
__device__ __forceinline__ float4 ldcoef(const float* c, size_t i) {
  const float* p = c + ((i >> 9) << 11) + (i & 511);
  return make_float4(__ldg(p), __ldg(p + 512), __ldg(p + 1024), __ldg(p + 1536));
}
__device__ __forceinline__ float4 rdcoef(const float* c, size_t i) {  // coherent (setup kernels)
  const float* p = c + ((i >> 9) << 11) + (i & 511);
  return make_float4(p[0], p[512], p[1024], p[1536]);
}
__device__ __forceinline__ void stcoef(float* c, size_t i, const float4& v) {
  float* p = c + ((i >> 9) << 11) + (i & 511);
  p[0] = v.x; p[512] = v.y; p[1024] = v.z; p[1536] = v.w;
}

// PCG scalars, device resident (fp64).  The sum_* fields are the reductions of
// the last kernel that produced them: local to this part first, then (multi-part) summed
// over all parts in place before any consumer reads them.
struct Scalars {
  double sum_rr;   // ||r||^2
  double sum_r;    // sum of r over active cells (null-space projection)
  double sum_rz;   // (r, z) of the current iteration
  double sum_pq;   // (p, A p)
  double sum_q;    // sum of A p over active cells (the projected update's mean)
  double rho;      // (r, z) of the previous iteration (beta = sum_rz / rho)
  double n_active; // number of active leaf cells (all parts)
  int flags;       // bit0: breakdown (sigma <= 0 or non-finite)
  float beta_f;    // beta = sum_rz / rho of Alg. 1 line 12 in fp32, set once per iteration
};
// offsets (in doubles) of the reduced fields, for the cross-part sums
enum { SF_RR = 0, SF_R = 1, SF_RZ = 2, SF_PQ = 3, SF_Q = 4 };

// owned leaf cells as float4 index ranges (one per level at most)
struct Ranges {
  int n = 0;
  int64_t begin[OCTMG_MAX_LEVELS + 1] = {};
  int64_t len[OCTMG_MAX_LEVELS + 1] = {};
};

// Kernel classes for profiling
enum KClass {
  KC_PASS = 0, KC_PROLONG, KC_RESTRICT, KC_COARSEST, KC_FASRHS, KC_SMOOTH_COARSE,
  KC_APPLY, KC_UPDATE, KC_DOT, KC_PROJECT, KC_INIT, KC_SETUP, KC_MEMSET, KC_SUBCYCLE, KC_RBFUSED, KC_COPY, KC_COARSE_GRID, KC_PUPDATE, KC_COUNT
};
extern const char* kclass_name[KC_COUNT];

struct Hier;

// launch helpers implemented in kernels.cu
struct ApplyArgs {
  const int* tiles;     // leaf tiles to compute (owned by this part); nullptr: tiles 0..ntiles-1
  int ntiles;
  const int4* tile;
  const int* nbr;
  const int* child;
  const float* coef;    // SoA per tile: planes c, c_x-, c_y-, c_z- (cidx)
  const float* glayer_val;
  const int* glayer;
  const int* dtile;     // leaf row sums (flux form): tile -> row of dval, -1 = all zero
  const float* dval;
  const float* z;       // p (user x for octmg_apply), zero on inactive cells
  float* pbar;          // inner-tile field: the active-children means of p on the listed face layers
  const int2* ifaces;   // (inner tile, face) layers neighbouring this part's leaf tiles
  int n_ifaces;
  float* q;             // A p
  double* partial;      // per-tile fp64 partial of p.q (nullptr: no dot)
  unsigned* counter;
  Scalars* sc;          // sum_pq written by the finish kernel
  int NL;
  int irr_inline;       // the irregular-tile body inlined (trees with T-junction tiles)
  int lean;             // no nonzero leaf row sums (the lean body skips the row-sum load)
  int sumq;             // also sum q into Scalars::sum_q (PCG with the null-space projection)
};
void launch_apply(const ApplyArgs& a, cudaStream_t s);

// vector kernels (PCG)
void launch_init(const float* b, const uint32_t* act, float* r, float* x, const Ranges& R, double* partial,
                 unsigned* counter, Scalars* sc, cudaStream_t s, int grid);
void launch_update(float* x, float* r, const float* p, const float* q, const Ranges& R, double* partial,
                   unsigned* counter, Scalars* sc, cudaStream_t s, int grid, float alpha_fixed = 0.0f,
                   const uint32_t* act_proj = nullptr);  // act_proj: also project r (null-space, fused)
void launch_project(float* r, const uint32_t* act, const Ranges& R, double* partial, unsigned* counter,
                    Scalars* sc, cudaStream_t s, int grid);
void launch_dot_rz(const float* r, const float* z, const Ranges& R, double* partial, unsigned* counter,
                   Scalars* sc, cudaStream_t s, int grid);
void launch_copy_ranges(const float* src, float* dst, const Ranges& R, cudaStream_t s);
void launch_set_beta(Scalars* sc, cudaStream_t s);  // beta_f from the (all-part) sums
void launch_set_rho_inf(Scalars* sc, cudaStream_t s);  // rho = inf (beta = 0 on the first iteration)
// copy nbytes (a multiple of 4) between device and mapped host memory by a kernel (no copy
// engine: small transfers never queue behind a caller's large copies)
void launch_copy_words(const void* src, void* dst, size_t nbytes, cudaStream_t s);
void launch_pupdate(const float* z, float* p, const Ranges& R, const Scalars* sc, bool use_beta, cudaStream_t s,
                    int grid);  // p = z + beta p in place
void launch_mask_copy(const float* src, const uint32_t* act, float* dst, int64_t n, cudaStream_t s);  // nat -> slots
void launch_copy_to_nat(const float* src, float* dst, const Ranges& R, cudaStream_t s);  // slots -> nat, owned
void launch_permute_f32(const float* src, float* dst, int64_t n, int nf, bool to_slots, cudaStream_t s);
void launch_permute_u8(const uint8_t* src, uint8_t* dst, int64_t n, bool to_slots, cudaStream_t s);
void launch_build_mask(const float* coef, int64_t n, uint32_t* act, cudaStream_t s);

// smoother kernels (direct.cu, rbfused.cu, subcycle.cu)
struct SmoothArgs {
  const int4* tile;
  const int* nbr;
  const int* parent;
  const float* coef;    // SoA per tile: planes c, c_x-, c_y-, c_z- (cidx)
  const float* glayer_val;
  const int* glayer;
  Fld u;                // level values read (in place: also written)
  Fld uc;               // rest buffer of every level (ghost sources, prolongation parents)
  const float* ustar;   // inner-indexed u* (prolongation)
  float* ustar_w;       // inner-indexed u* output (restrict stage)
  Fld b;                // leaf = PCG residual r, inner = FAS rhs
  float beta, alpha;    // restriction: b^{l-1} = beta R r, R = P^T / alpha
  int std_form;         // Alg. 2: u^{l-1} := 0 and u* := 0 at restriction (no Avg, no FAS rhs)
  float pro_scale;      // prolongation: u += pro_scale (u^{l-1} - u*) (Alg. 2: beta; Alg. 4: 1)
  int pro_active_only;  // prolong only from active parents (GMG comparison mode: a solid coarse
                        // cell can have fluid children and a nonzero u*; DESIGN reading 20)
  int NL;
  const int* order;     // tiles of the level in rank order (slab-major), or nullptr: the level's
                        // tiles by index, ord_nleaf leaves from ord_leaf0 then inners from ord_inner0
  int ord_leaf0, ord_nleaf, ord_inner0;
  int n;                // tiles in the level
  int first_tile;       // k_fasrhs: first inner tile of the level
  int stage[1];         // bit0 colour, bits1.. mode
  // direct coarsest solve (coarsest = 1): u^0 = M0 b^0 over the c0n level-0 cells (cell
  // k*512 + slot of level-0 tile c0tile[k]); M0 row-major f32 [c0n][c0n]; c0n = 0: smoothing
  const float* c0M;
  const int* c0tile;
  int c0n;
  double* rz_partial;   // SM_PLAIN_RZ (the last pass of M on a uniform tree): per-warp fp64
                        // partials of (r, z) over the tile's cells (PCG Alg. 1 line 12)
};
void launch_fasrhs(const SmoothArgs& a, int ninner, cudaStream_t s);
void launch_pass_direct(const SmoothArgs& a, cudaStream_t s, int cpt);
bool pass_v3_on();  // the 128-bit row pass on big levels (not OCTMG_PASS_V=2)
// (r, z) and beta from the SM_PLAIN_RZ pass's 2 partials per tile (fixed order)
void launch_rz_finish(const double* partial, int64_t n, double* scratch, Scalars* sc, cudaStream_t s);
void launch_restrict_direct(const SmoothArgs& a, cudaStream_t s, int v2);  // 0 staged, 6 / 8: k_restrict_v2 min CTAs/SM
void launch_prolong(const SmoothArgs& a, cudaStream_t s);
int subcycle_max_tiles();
int subcycle_max_level();
void launch_subcycle(const SmoothArgs& base, int L, int K, int fas_first, const octmg_mg_params& prm,
                     const int* order_all, const int* lvl_off, const int* lvl_n, const int* ib, const int* ic,
                     cudaStream_t s);

// the coarsest complete levels as dense grids in shared memory (coarse_dense.cu)
constexpr int CD_MAXL = 3;
octmg_status build_coarse_dense(Hier& h, int Kmax, cudaStream_t s);  // sets h.cd_K (-1: not applicable)
void launch_coarse_dense(const Hier& h, int K, int fas_first, float* u_inner, float* b_inner, cudaStream_t s);
octmg_status build_coarse_cluster(Hier& h, cudaStream_t s);  // sets h.cc_K = 2 (levels 0-2 in a cluster) or -1
void launch_coarse_cluster(const Hier& h, int fas_first, float* u_inner, float* b_inner, cudaStream_t s);

// direct coarsest solve (coarsest.cu)
constexpr int C0_MAX_CELLS = 4096;
octmg_status build_coarse_direct(Hier& h, cudaStream_t s);  // M0 of level 0 (setup)
void launch_coarse_direct(const SmoothArgs& a, cudaStream_t s);  // u^0 = M0 b^0 (one launch)

// setup kernels (setup.cu)
struct SetupArgs;
octmg_status assemble_leaf_coefs(Hier& h, const uint8_t* kind, const float* fbeta, const float* ffrac,
                                 cudaStream_t s);  // + coarsen_all + the leaf row sums d
octmg_status coarsen_all(Hier& h, cudaStream_t s);  // literal Alg. 3 if h.prm.coarsen_literal

// projection operators (projection.cu)
octmg_status divergence(const Hier& h, const float* frac, const float* u6, float* b, cudaStream_t s);
octmg_status subtract_gradient(const Hier& h, const uint8_t* kind, const float* fbeta, const float* frac,
                               const float* p, float* u6, cudaStream_t s);

// cut-cell geometry of the tank scene (geometry.cu)
octmg_status tank_fields(const Tree& T, const double* centre, double radius, uint8_t* kind, float* frac, float* b,
                         cudaStream_t s);
octmg_status tank_fields_inner(const Tree& T, const double* centre, double radius, uint8_t* kind, float* frac,
                               cudaStream_t s);  // the same geometry on the inner tiles (GMG mode)

// narrow-band refinement of the sphere-surface test grids on the device (band.cu)
octmg_status band_tiles(const int32_t* ext, int l0, int extra, const double* centre, double radius, int repair,
                        octmg_tile* out_host, int64_t cap, int64_t* n_out, cudaStream_t s);

// 2:1 grading repair of a leaf-tile list (grade.cpp, host)
octmg_status grade_repair(const octmg_tile* in, int64_t n, const int32_t* ext, std::vector<octmg_tile>& out);

// tree build (tree.cu)
octmg_status build_tree(const octmg_tree_desc* desc, const octmg_tile* tiles, int64_t n, cudaStream_t s,
                        Tree* t);

// ------------------------------------------------------------------------------------
// Hierarchy (coefficients + multigrid work buffers + PCG state)
// ------------------------------------------------------------------------------------
struct Op {
  int kind;    // 0 smoother stage, 1 FAS rhs, 2 zero coarse leaves, 3 prolongation, 4 sub-cycle,
               // (5, 6: retired fused-RB kinds), 7 halo exchange of level
               // `level` of u, 8 broadcast of the restricted partition-parent level,
               // (9: the retired cooperative coarse grid)
  int level;
  int stage;   // bit0 colour, bits1.. mode (SM_*)
  int in_buf = 0, out_buf = 0;
};

struct Hier {
  Tree* tree = nullptr;
  octmg_mg_params prm{};
  float* coef = nullptr;         // [T*2048] SoA per tile: c, cxm, cym, czm planes (cidx)
  float* ccoef = nullptr;        // the records the cycle uses: = coef, or (GMG comparison mode) a
                                 // copy with the inner tiles' records assembled from the grid
  // GMG comparison mode inputs (octmg_setup_hierarchy_gmg; read during setup only)
  const uint8_t* gmg_kind = nullptr;   // [NI*512] inner cells' kinds (natural cell order)
  const float* gmg_beta = nullptr;     // [6][NI*512] or null (= 1)
  const float* gmg_frac = nullptr;     // [6][NI*512] or null (= 1)
  uint32_t* act = nullptr;       // [NL*512/32] activity bitmask of the leaf cells
  float* glayer_val = nullptr;   // [n_glayers*64]
  int2* ifaces = nullptr;        // (inner tile, face) layers the composite apply reads as children means
  int n_ifaces = 0;
  float* pbar = nullptr;         // [NI*512] those means (only the listed face layers are written)
  int* dtile = nullptr;          // [NL] leaf row sums d (flux-form apply): tile's row in dval, or -1 (all d = 0)
  float* dval = nullptr;         // [n_dtiles*512] d of those tiles (slot order)
  int n_dtiles = 0;
  // multigrid buffers
  float* z = nullptr;            // [NL*512] leaf part of the cycle's u (buffer A) = M output
  float* uinA = nullptr;         // [NI*512] inner part of u (buffer A)
  float* binner = nullptr;       // [NI*512]
  float* ustar = nullptr;        // [NI*512]
  float* r = nullptr;            // [NL*512] PCG residual = leaf part of the cycle rhs
  float* xs = nullptr;           // [NL*512] PCG iterate (slot order; copied to the caller's x)
  // PCG
  float* p0 = nullptr;
  float* p1 = nullptr;
  float* q = nullptr;
  double* partial = nullptr;     // reduction partials
  size_t n_partial = 0;
  unsigned* counter = nullptr;   // last-block counters (one per reduction slot)
  Scalars* sc = nullptr;         // device scalars
  Scalars* sc_host = nullptr;    // mapped pinned mirror (host pointer)
  Scalars* sc_host_dev = nullptr;  // its device pointer (written by launch_copy_words)
  double n_active = 0;
  int any_dirichlet = 0;
  // per-level tile orders (this part's tiles at partitioned levels)
  int* order = nullptr;          // [T] per level: tiles in rank order (segment at lvl_order_off)
  int lvl_order_off[MAXL + 1] = {};
  int lvl_n[MAXL + 1] = {};
  bool lvl_ghost[MAXL + 1] = {};
  int lvl_nreg[MAXL + 1] = {};    // tiles of the level without a ghost face (first in its order segment)  // the level has T-junction (ghost) tiles (anywhere, all parts)
  int pass_cpt = 4;              // colour cells per thread of the direct pass (OCTMG_PASS_CPT)
  bool pass_v2 = true;           // k_pass_v2 on the small levels (the round-1 k_pass_direct is retired)
  int pass_big = 1024;           // levels with >= pass_big tiles run pass_cpt cells/thread, smaller ones 1 (OCTMG_PASS_BIG)
  bool direct_order = true;      // level kernels take tiles by index (OCTMG_TILE_ORDER=slab: the order array)
  bool restrict_red = true;      // red-row restriction on ghost-free levels (OCTMG_RESTRICT_RED=0: off)
  int restrict_row = -1;         // row-form restriction: -1 on levels with ghost tiles, 0 never, 1 always (OCTMG_RESTRICT_ROW)
  int restrict_v2 = 6;           // k_restrict_v2 (x-pairs) at >= 6 CTAs/SM
  int sub_K = -1;                // top level of the on-chip coarse sub-cycle (-1: none)
  int cd_K = -1;                 // top level of the dense shared-memory coarse cycle (coarse_dense.cu; -1: none)
  int cd_total = 0;              // its cells (levels 0..cd_K)
  int cd_lv[CD_MAXL + 1][4] = {};  // per level: nx, ny, nz, first cell
  int* cd_map = nullptr;         // tile maps of those levels
  std::vector<int> cd_moff;      // per level: offset of its tile map
  float* cd_coef = nullptr;      // dense coefficient planes
  int cd_threads = 512;          // threads of its CTA
  int cc_K = -1;                 // 2: levels 0..2 in one thread-block cluster (k_coarse_cluster), else -1
  int* cc_map = nullptr;         // its level-2 tile map
  float* cc_coef = nullptr;      // its level-2 slab coefficient planes
  size_t cc_smem = 0;            // its dynamic shared memory per CTA
  float* c0M = nullptr;          // direct coarsest solve: M0 [c0n][c0n] (coarsest = 1)
  int* c0tile = nullptr;         // its level-0 tiles
  int c0n = 0;
  // profiling
  bool profiling = false;
  struct Ev { int cls; double bytes; cudaEvent_t a, b; int level; };
  std::vector<Ev> events;
  std::vector<cudaEvent_t> event_pool;
  size_t event_next = 0;
  double prof_ms[KC_COUNT] = {};
  int64_t prof_cnt[KC_COUNT] = {};
  double prof_bytes[KC_COUNT] = {};
  double prof_lvl_ms[MAXL + 1][KC_COUNT] = {};   // the same per level of the multigrid op
  int64_t prof_lvl_cnt[MAXL + 1][KC_COUNT] = {};
  double prof_lvl_bytes[MAXL + 1][KC_COUNT] = {};
  // partition (multi-part): this part's rank, owned ranges
  int rank = 0, nranks = 1;
  int lg = 0;                          // partition level (levels < lg replicated)
  int own_lb[MAXL + 1] = {}, own_lc[MAXL + 1] = {};  // owned leaf tiles per level
  int own_ib[MAXL + 1] = {}, own_ic[MAXL + 1] = {};  // owned inner tiles per level
  Ranges own_cells;                    // owned leaf cells (float4 units)
  int* apply_tiles = nullptr;          // owned leaf tiles
  int n_apply_tiles = 0;
  double n_active_local = 0;
  std::vector<void*> allocs;
  ~Hier();
};

struct PartPlanHolder;
struct Comm;

// A solver instance: one part (single GPU, or one rank of an NCCL job) or several parts
// in one process (loopback partition on one GPU, for testing the distributed path).
// state of the device-side PCG loop (OCTMG_GRAPH_LOOP=1): written by the loop's check
// kernel, read by the host once per solve
constexpr int LOOP_HCAP = 512;
struct LoopState {
  double bn, rtol, rel;
  int k, max_iters, status;  // status: 0 running/converged, 9 breakdown, 8 non-finite, 10 max iters
  int converged;
  double hist[LOOP_HCAP];
};
void launch_pcg_check(Scalars* sc, LoopState* ls, unsigned long long handle, cudaStream_t s);

struct Group {
  std::vector<Hier*> parts;
  Comm* comm = nullptr;
  PartPlanHolder* plan = nullptr;
  std::vector<Op> ops;                 // identical for every part
  cudaGraphExec_t graph = nullptr;
  cudaStream_t graph_stream = nullptr;
  cudaGraphExec_t loop_graph = nullptr;  // the whole PCG loop as a conditional-while graph
  LoopState* loop = nullptr;             // device
  LoopState* loop_host = nullptr;        // mapped pinned (host pointer)
  LoopState* loop_host_dev = nullptr;    // its device pointer
  int loop_ns = -1;                      // null-space flag the loop graph was built with
  bool rz_fused = false;                 // (r, z) summed by the last pass of M (build_schedule)
  bool loop_unavailable = false;         // building the loop graph failed: host-driven loop
  int64_t launches = 0;
  ~Group();
};

}  // namespace octmg

struct octmg_tree {
  octmg::Tree t;
};
struct octmg_hier {
  octmg::Group g;
};
