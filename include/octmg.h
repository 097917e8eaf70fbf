/*
 * octmg.h — C ABI of the B200-native (sm_100a) matrix-free multigrid-preconditioned CG
 * solver for  -div(beta grad p) = b  on graded adaptive octrees with cut cells.
 *
 * Method: arXiv 2604.18886 (Wang, Sun, Zhu), "Matrix-Free Multigrid with Algebraically
 * Consistent Coarsening on Adaptive Octrees".  Citations "P:Lnnn" are lines of that
 * paper's PAPER.md (section / equation / algorithm named beside each).
 *
 * Conventions
 *  - Tiles are 8x8x8 cells.  At tile level l the domain has ext[a] * 2^l tiles
 *    along axis a and the cell edge is h_l = 2^-l / 8 in units of a level-0 tile.
 *  - Leaf-slot order (all user vectors): leaf tiles sorted by (level descending, Morton
 *    key ascending; Morton interleaves bits with x in the lowest bit of each triple), then
 *    cells x + 8y + 64z within a tile.  octmg_tree_export(OCTMG_EXPORT_TILES) returns that
 *    order; slot = tile_index * 512 + cell.
 *  - Face order: x-, x+, y-, y+, z-, z+.
 *  - Right-hand side convention: A p = b with A ~ -div(beta grad) * V (volume-integrated,
 *    symmetric-positive sign), Eq. 1-3.  For div(beta grad p) = f pass
 *    b_i = -f_i V_i.
 *  - Vectors are fp32 device arrays; dot products accumulate in fp64.
 *  - Ownership: the library owns every internal device allocation; caller buffers are
 *    borrowed for the duration of a call.  All device work is issued on the caller's
 *    stream; calls are asynchronous unless stated otherwise.  A handle is not
 *    thread-safe (one call at a time).
 *  - Errors: every entry point returns an octmg_status; octmg_last_error() gives a
 *    thread-local message.  No C++ exception crosses the ABI.  A failed call leaves no
 *    handle allocated.
 */
#ifndef OCTMG_H
#define OCTMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* cudaStream_t without including the CUDA headers; NULL = legacy default stream. */
typedef struct CUstream_st* octmg_stream;

typedef enum {
  OCTMG_OK = 0,
  OCTMG_E_INVALID = 1,     /* bad argument, level or coordinate out of range            */
  OCTMG_E_OVERLAP = 2,     /* duplicate leaf tiles, or a leaf that contains another     */
  OCTMG_E_GAP = 3,         /* leaf tiles do not cover the domain                        */
  OCTMG_E_NOT_GRADED = 4,  /* two face-adjacent leaves differ by > 1 level     */
  OCTMG_E_OOM = 5,         /* device allocation failed                                  */
  OCTMG_E_CUDA = 6,        /* any other CUDA runtime error                              */
  OCTMG_E_NCCL = 7,        /* reserved (multi-GPU)                                      */
  OCTMG_E_NONFINITE = 8,   /* non-finite value in b or in a PCG scalar                  */
  OCTMG_E_BREAKDOWN = 9,   /* p.Ap <= 0 in PCG; the last good iterate is kept           */
  OCTMG_E_MAXITER = 10     /* not converged within max_iters (report.converged = 0)     */
} octmg_status;

/* Thread-local description of the last failure (never NULL). */
const char* octmg_last_error(void);
/* Library version string. */
const char* octmg_version(void);

typedef struct octmg_tree octmg_tree;
typedef struct octmg_hier octmg_hier;

/* A LEAF tile: level l and tile coordinates (i, j, k) at that level. */
typedef struct {
  int32_t level, i, j, k;
} octmg_tile;

typedef struct {
  int32_t ext[3];      /* domain size in level-0 tiles; (1,1,1) = unit cube              */
  uint8_t wall_bc[6];  /* per domain face x-,x+,y-,y+,z-,z+: 0 Neumann, 1 Dirichlet p=0
                          at the centre of a virtual wall cell of the boundary cell's
                          size (P:L328-330 ghost-fluid Dirichlet)                         */
  int32_t grade_repair;/* 0: ungraded input is rejected with NOT_GRADED; 1: the list is first
                          repaired on the host (octmg_grade_repair_host)                 */
  int32_t rank, nranks;/* this process's rank and the number of ranks (1 = single GPU)    */
  void* nccl_comm;     /* ncclComm_t over the nranks GPUs (octmg_nccl_comm_init), or NULL
                          when nranks == 1.  The leaf-tile list is replicated on all ranks;
                          the partition is deterministic.                    */
} octmg_tree_desc;

/*
 * Build the octree tables on the GPU from the host list of leaf tiles (P:L548-550,
 * "recompute the six same-level neighbors for each tile"): validates range,
 * overlap, coverage (exact integer volume) and 2:1 face grading; sorts tiles into the
 * canonical order; derives inner tiles (all strict ancestors of leaves), per-level
 * segments, the 6-neighbour table (>= 0 same-level tile, -1 domain wall, -2 - c when the
 * neighbour position is a ghost whose coarse leaf tile is c), parent and child tables.
 * leaf_tiles_host: n entries, any order, host memory (copied).  Synchronises `stream`.
 */
octmg_status octmg_build_tree(const octmg_tree_desc* desc, const octmg_tile* leaf_tiles_host,
                              int64_t n, octmg_stream stream, octmg_tree** out);

#define OCTMG_MAX_LEVELS 16
typedef struct {
  int32_t levels;          /* L + 1 (level 0 .. L, L = finest leaf level)                 */
  int32_t n_leaf_tiles;    /* NL; leaf tiles are tile indices [0, NL)                     */
  int32_t n_inner_tiles;   /* NI; inner tiles are tile indices [NL, NL + NI)              */
  int64_t n_leaf_cells;    /* NL * 512 = length of every user vector                      */
  int32_t leaf_begin[OCTMG_MAX_LEVELS], leaf_count[OCTMG_MAX_LEVELS];
  int32_t inner_begin[OCTMG_MAX_LEVELS], inner_count[OCTMG_MAX_LEVELS];
  int32_t n_ghost_layers;  /* T-junction (+face toward a ghost) coefficient layers        */
} octmg_tree_info;
octmg_status octmg_tree_info_get(const octmg_tree* tree, octmg_tree_info* out);

/* Copy canonical tables to host (bit-exact contract; int32):
 *  TILES  (NL+NI) x 4 (level,i,j,k)   NBR (NL+NI) x 6   PARENT (NL+NI) (-1 at level 0)
 *  CHILD  NI x 8 (octant dx + 2dy + 4dz)                 bytes must equal the size. */
enum { OCTMG_EXPORT_TILES = 0, OCTMG_EXPORT_NBR = 1, OCTMG_EXPORT_PARENT = 2, OCTMG_EXPORT_CHILD = 3 };
octmg_status octmg_tree_export(const octmg_tree* tree, int32_t what, void* host_dst, size_t bytes);

typedef struct {
  float alpha;          /* restriction scaling, R = P^T / alpha; 2   */
  float beta_overshoot; /* MG overshoot beta (not the PDE face_beta), at restriction (Alg. 4 line 10); 2   */
  int32_t mu;           /* cycle index: 1 V-cycle, 2 W-cycle                   */
  int32_t nu_pre;       /* RBGS iterations (red+black) before coarsening: 2        */
  int32_t nu_post;      /* RBGS iterations after (opposite colour order): 2                 */
  int32_t nu_coarsest;  /* RBGS iterations at level 0, two opposite-order halves: 10        */
  int32_t form;         /* 0: FAS-style mu-cycle, Alg. 4, beta at restriction;
                           1: standard mu-cycle, Alg. 2, beta at prolongation,
                           zero coarse initial guess — uniform trees only (every leaf at the
                           finest level), else OCTMG_E_INVALID                                */
  int32_t coarsen_literal; /* 1: Alg. 3 exactly as printed (the non-diagonal
                           branch without the activity test); 0 (default): with the test,
                           so that Alg. 3 equals R A P over the fluid unknowns (DESIGN.md
                           reading 3)                                                        */
  int32_t coarsest;     /* level-0 step of the cycle (Alg. 4 line 4): 0 (default)
                           nu_coarsest RBGS iterations; 1 "or direct solve":
                           u^0 = M0 b^0 with M0 the solution operator of the level-0
                           system over its active cells, precomputed at setup (exact
                           inverse on components coupled to a Dirichlet cell or wall; the
                           minimum-norm solution on floating pure-Neumann components,
                           DESIGN.md reading 9b).  Needs <= 4096 level-0 cells (ext product
                           <= 8), else OCTMG_E_INVALID                                       */
  int32_t reserved0;
  int64_t gather_below_cells; /* multi-GPU: the partition level lg is the
                           coarsest level (<= the coarsest leaf level) with >= 8 tiles per
                           rank and >= gather_below_cells cells; the levels below it are not
                           partitioned — every rank holds and smooths them redundantly after
                           an all-gather of the restricted partition parents (0 = the default
                           threshold, 2^21 cells; 1 = partition as deep as 8 tiles per rank
                           allow; single part: ignored)                                      */
} octmg_mg_params;

/*
 * Assemble the compact matrix-free coefficients (c, c_x-, c_y-, c_z-) of every leaf cell
 * (Eq. 3; ghost-fluid kinds; T-junction faces, Eqs. 9-10,
 * P:L641-648) and coarsen every inner cell bottom-up with Alg. 3 (with the
 * activity test on the off-diagonal branch so that it equals R A P over fluid DOFs).
 *  kind:      device u8[N], 0 fluid, 1 Dirichlet (p = 0), 2 Neumann (solid)
 *  face_beta: device f32[6][N] or NULL (= 1): beta on each face of each leaf cell
 *  face_frac: device f32[6][N] or NULL (= 1): fluid area fraction S / h^2 of each face
 *  Face conductance kappa = beta * frac * h.  Authority: the +side cell's -face entry on
 *  same-level faces, the fine side's entries on T-junction faces, the cell's own entry
 *  on domain faces.  params: NULL = defaults above.  Inputs are read during the call only.
 */
octmg_status octmg_setup_hierarchy(octmg_tree* tree, const uint8_t* kind, const float* face_beta,
                                   const float* face_frac, const octmg_mg_params* params,
                                   octmg_stream stream, octmg_hier** out);

/*
 * Partitioned hierarchy of `nparts` parts living in this process on the current device
 * ("loopback" transport: halo exchanges are device copies between the parts).  Same
 * partition, schedule and kernels as an nparts-rank NCCL job; used to test the
 * distributed path on one GPU.  Vectors passed to the solver calls are global leaf-slot
 * vectors; each part reads/writes its owned cells.
 */
octmg_status octmg_setup_hierarchy_loopback(octmg_tree* tree, int32_t nparts, const uint8_t* kind,
                                            const float* face_beta, const float* face_frac,
                                            const octmg_mg_params* params, octmg_stream stream,
                                            octmg_hier** out);

/*
 * GMG comparison mode (Fig. 12): the
 * cycle's coarse operators "given directly by the grid discretization" instead of
 * Alg. 3 — every inner cell's record (c, c_x-, c_y-, c_z-) assembled by Eq. 3 (P:L303-316,
 * kinds P:L318-335) at its own level from its own kind and face weights and those of its
 * same-level neighbours (leaf inputs for leaf cells).  Only the preconditioner changes: the
 * leaf records, and so the composite operator octmg_apply / octmg_pcg_solve solve with, are
 * those of octmg_setup_hierarchy (a T-junction face keeps its Alg. 3 coupling there).  In
 * fluid-only domains both constructions coincide; next to solid cells the grid
 * records ignore the sub-cell structure, which is what makes GMG stall on cut cells (Fig. 12).
 *  kind, face_beta, face_frac: as octmg_setup_hierarchy (leaf cells).
 *  kind_inner:      device u8[NI*512], the inner cells' kinds (inner tiles in canonical order,
 *                   cells x + 8y + 64z) — e.g. octmg_tank_fields_inner.
 *  face_beta_inner, face_frac_inner: device f32[6][NI*512] or NULL (= 1).
 * Single-part hierarchies only (OCTMG_E_INVALID for a multi-rank tree).  Inputs are read
 * during the call only.  Costs a second coefficient store (the cycle's).
 */
octmg_status octmg_setup_hierarchy_gmg(octmg_tree* tree, const uint8_t* kind, const float* face_beta,
                                       const float* face_frac, const uint8_t* kind_inner,
                                       const float* face_beta_inner, const float* face_frac_inner,
                                       const octmg_mg_params* params, octmg_stream stream, octmg_hier** out);

/* Partition of part `part` (0 for an NCCL rank): partition level lg (levels < lg are
 * replicated), rank, nranks, and per level the owned leaf tiles [begin, begin+count). */
octmg_status octmg_partition_info(const octmg_hier* h, int32_t part, int32_t* lg, int32_t* rank,
                                  int32_t* nranks, int32_t* own_leaf_begin, int32_t* own_leaf_count);

/* NCCL bootstrap for a multi-GPU job (libnccl.so.2 is loaded on first use): rank 0 calls
 * octmg_nccl_unique_id (128 bytes), broadcasts it (e.g. via torch.distributed), every rank
 * calls octmg_nccl_comm_init on its device.  The solver calls of an nranks > 1 hierarchy
 * are collective: every rank must issue them in the same order.  Each rank's output
 * vectors hold its owned cells. */
octmg_status octmg_nccl_unique_id(void* out128);
octmg_status octmg_nccl_comm_init(int32_t rank, int32_t nranks, const void* id128, void** comm);
void octmg_nccl_comm_destroy(void* comm);

/* Host-only partition planner (no device needed): from the canonical tree tables (as
 * exported by octmg_tree_export; level_counts = 4 int32 per level l = 0..L: leaf_begin,
 * leaf_count, inner_begin, inner_count), the partition level lg, the owner rank of every
 * tile (-1 = replicated, level < lg) and the halo item lists: n_items_out[(l*nranks +
 * from)*nranks + to] items of (tile, kind) pairs concatenated in that order into items_out
 * (kind 0..5 = face layer of that face, 6 = whole tile).  items_cap = max item count.
 * gather_below_cells: as octmg_mg_params.gather_below_cells (0 = the default threshold). */
octmg_status octmg_partition_plan_host(const int32_t* tiles4, const int32_t* nbr, const int32_t* parent,
                                       const int32_t* child, int32_t NL, int32_t NI, int32_t L,
                                       const int32_t* level_counts, int32_t nranks, int32_t* lg_out,
                                       int32_t* owner_out, int32_t* n_items_out, int32_t* items_out,
                                       int64_t items_cap, int64_t gather_below_cells);

/*
 * Narrow-band leaf tiles around a sphere surface on the device (P:L1224-1229,
 * the Table 1 / Sec. 5.3-5.4 grids): starting from every level-l0 tile of the ext[0] x
 * ext[1] x ext[2] domain, a tile whose box strictly intersects the sphere surface (distance
 * from `centre3` to the box: d_min < radius < d_max; coordinates in level-0 tile units) is
 * refined, down to level l0 + extra; the others stay leaves.  grade_repair = 1 then refines,
 * to fixpoint, every leaf face-adjacent to a leaf two or more levels finer, the
 * unique minimal 2:1-graded refinement.  Dense per-level occupancy bitmaps on the device
 * (fp64 box test without FMA contraction: the same tile set as an IEEE host computation).
 * out_host: cap entries of host memory receiving the leaves in unspecified order (feed them
 * to octmg_build_tree), or NULL to count only; *n_out = the leaf count (OCTMG_E_INVALID if it
 * exceeds cap).
 * Synchronises `stream`.
 */
octmg_status octmg_band_tiles(const int32_t* ext3, int32_t l0, int32_t extra, const double* centre3, double radius,
                             int32_t grade_repair, octmg_tile* out_host, int64_t cap, int64_t* n_out,
                             octmg_stream stream);

/*
 * Cut-cell fields of the static tank scene: a solid sphere
 * obstacle (centre, radius in level-0 tile units; radius <= 0: none) in a tank with solid
 * bottom and side walls and an open top y = ext_y.  For every leaf cell (leaf-slot order),
 * on the device: kind (2 Neumann/solid where the SDF phi = |x - centre| - radius < 0 at the
 * cell centre, else 0 fluid; ghost-fluid classification P:L318-320), face_frac[6][N] the
 * fluid area fraction of each face from the SDF sampled at its 4 corners by
 * marching squares, a saddle split when the face-centre sample is solid;
 * tank walls 0, the open top 1; and b = h^2 (w_y+ - w_y-) on fluid cells (0 on solid),
 * the volume-integrated divergence of a unit downward velocity.  fp64 arithmetic, fp32
 * outputs.  kind, face_frac, b: device buffers of N, 6N, N elements (caller-owned).
 */
octmg_status octmg_tank_fields(const octmg_tree* tree, const double* centre3, double radius, uint8_t* kind,
                               float* face_frac, float* b, octmg_stream stream);

/* The same tank geometry on the inner cells (each at its own level): kinds and face
 * fractions for octmg_setup_hierarchy_gmg.  kind_inner: device u8[NI*512], face_frac_inner:
 * device f32[6][NI*512] (inner tiles in canonical order, cells x + 8y + 64z; caller-owned). */
octmg_status octmg_tank_fields_inner(const octmg_tree* tree, const double* centre3, double radius,
                                     uint8_t* kind_inner, float* face_frac_inner, octmg_stream stream);

/*
 * Projection operators on the composite octree (after the pressure solve
 * "apply the pressure gradient to project the velocity field and measure the divergence";
 * SPEC S:L170-178).  Face velocities u6: device f32[6][N], u6[f][i] = the velocity
 * component along the +axis of face f (x-,x+,y-,y+,z-,z+) on that face of leaf cell i
 * (both cells of a shared face hold a copy); face_frac: device f32[6][N] fluid fractions
 * (NULL = 1), S = frac h^2.  Single-part hierarchies only (OCTMG_E_INVALID otherwise).
 *
 * octmg_divergence: b_i = -(sum over the faces of i of the outward flux s_f u S), s_f = -1
 * on - faces and +1 on + faces, on every active leaf cell (0 on inactive cells) — the
 * right-hand side convention of the solver (for u = (0,-1,0) in the tank it is the
 * h^2 (w_y+ - w_y-) of octmg_tank_fields).  A coarse leaf's face toward finer cells sums
 * the fine cells' entries (the finer side is authoritative, as for the coefficients).
 * b: device f32[N].
 *
 * octmg_subtract_gradient: u6 -= G p in place: on every face of every active leaf cell with
 * S > 0, u += s_f F_f / S where F_f is the composite operator's flux through that face
 * (the face's share of the diagonal times p_i plus the coupling times the neighbour value,
 * T-junction ghosts by Eq. 12), so that divergence(u - G p) = divergence(u) -
 * A p: after a converged solve of A p = divergence(u) the projected field's divergence is
 * the solver's residual.  kind, face_beta, face_frac: the arrays given to
 * octmg_setup_hierarchy (face_beta / face_frac NULL = 1).  p: device f32[N].
 */
octmg_status octmg_divergence(const octmg_hier* h, const float* face_frac, const float* u6, float* b,
                              octmg_stream stream);
octmg_status octmg_subtract_gradient(const octmg_hier* h, const uint8_t* kind, const float* face_beta,
                                     const float* face_frac, const float* p, float* u6, octmg_stream stream);

/*
 * 2:1 face-grading repair on the host (no device needed, SPEC S:L82;
 * grading P:L548-550): every leaf tile that covers an in-domain face-neighbour position of
 * a leaf two or more levels finer is replaced by its 8 children, to fixpoint (the least
 * graded refinement of the input; the order of the input does not matter).  tiles: n leaf
 * tiles (host); ext3: the domain in level-0 tiles; out: host array of cap tiles (any
 * order).  *n_out = the repaired count; if cap is too small nothing is written and the
 * call fails with OCTMG_E_INVALID (call again with *n_out).
 */
octmg_status octmg_grade_repair_host(const octmg_tile* tiles, int64_t n, const int32_t* ext3, octmg_tile* out,
                                     int64_t cap, int64_t* n_out);

/*
 * Allocator hook: every persistent device buffer of the handles created afterwards (tree
 * tables, coefficient store, multigrid and PCG buffers, halo buffers) is obtained with
 * alloc(bytes, stream, ctx) and returned with release(ptr, stream, ctx) (stream = NULL:
 * the legacy default stream), e.g. to draw from PyTorch's caching allocator.  Each
 * pointer is released through the allocator that made it, so the hook may change between
 * handles.  Short-lived setup temporaries still use cudaMalloc(Async).  NULL, NULL restores
 * cudaMalloc / cudaFree.  alloc returns NULL on failure (the call then fails with
 * OCTMG_E_OOM).  Process-wide; thread-safe.
 */
typedef void* (*octmg_alloc_fn)(size_t bytes, octmg_stream stream, void* ctx);
typedef void (*octmg_free_fn)(void* ptr, octmg_stream stream, void* ctx);
octmg_status octmg_set_allocator(octmg_alloc_fn alloc, octmg_free_fn release, void* ctx);

/* Host copy of the coefficient store: (NL+NI)*512 records of 4 floats (c, cxm, cym, czm)
 * in tile order, cells x + 8y + 64z within a tile (the library's internal colour-split,
 * structure-of-arrays layout is converted).  Synchronises `stream` of the last call. */
octmg_status octmg_hier_export_coefs(const octmg_hier* h, float* host_dst, size_t bytes);
/* The same export of the records the cycle uses (differs from the above only for a GMG
 * comparison-mode hierarchy, octmg_setup_hierarchy_gmg: its inner records). */
octmg_status octmg_hier_export_cycle_coefs(const octmg_hier* h, float* host_dst, size_t bytes);

/* y = A x, the composite operator over all leaf cells (T-junction ghosts, Eq. 12,
 * P:L661-665; inner neighbour value = mean of its active children).  x, y are
 * device f32[N]; y is 0 on inactive cells; x's inactive entries are ignored. */
octmg_status octmg_apply(octmg_hier* h, const float* x, float* y, octmg_stream stream);

/* u = M b: one FAS-style mu-cycle (Alg. 4) from a zero initial guess.
 * b, u are device f32[N]; b's inactive entries are ignored; u is 0 on inactive cells. */
octmg_status octmg_vcycle(octmg_hier* h, const float* b, float* u, octmg_stream stream);

typedef struct {
  double rtol;          /* stop when ||r||_2 <= rtol * ||r_0||_2 (active cells); 1e-6    */
  int32_t max_iters;    /* 200                                                            */
  int32_t nullspace;    /* -1 auto (no Dirichlet wall or cell), 0 off, 1 project residual
                           to zero mean after Alg. 1 lines 4 and 11              */
} octmg_solve_params;

typedef struct {
  int32_t iters;        /* PCG iterations performed (= A applications = M applications)  */
  int32_t converged;
  double rel_residual;  /* ||r_k|| / ||r_0|| (recursive residual)                         */
  double bnorm;         /* ||r_0||                                                        */
  int32_t status;       /* octmg_status of the solve                                      */
  double* history;      /* optional host array: relative residual after each iteration   */
  int32_t history_cap;
  int64_t kernel_launches; /* device kernels launched by this solve (graph nodes counted) */
  int32_t history_len;  /* entries of history written: min(iters, history_cap), and at most
                           512 in the device-side loop                                    */
  int32_t device_loop;  /* 1: the solve ran as the device-side conditional-graph loop;
                           0: the host-driven loop                                        */
} octmg_solve_report;

/*
 * Alg. 1: x0 = 0, r0 = b (masked to active cells, projected if nullspace),
 * z = M r, CG recurrences with fp64 scalars kept on the device.  The whole loop runs as
 * ONE CUDA graph with a conditional while node whose stopping test (Alg. 1 line 8) runs on
 * the device: one host synchronisation per solve; a partitioned hierarchy captures its
 * transport's halo exchanges and fp64 scalar allreduces into the same body.  Environment
 * OCTMG_GRAPH_LOOP=0, profiling, or a transport / driver that cannot be captured: the
 * host-driven loop (the same kernels, one scalar read per iteration).  The null-space
 * projection of the updated r is fused into the x / r update (its mean from the projected r's
 * sum and the apply's sum of A p, the same projection up to rounding); on trees whose leaves
 * all lie on the finest level (r, z) is summed by the last colour pass of M.
 * b (read-only) and x (overwritten) are device f32[N].  Synchronises `stream` before
 * returning.  report may be NULL.
 */
octmg_status octmg_pcg_solve(octmg_hier* h, const float* b, float* x, const octmg_solve_params* params,
                             octmg_solve_report* report, octmg_stream stream);

/*
 * Multigrid as a standalone solver (use beta = 1, "to prevent
 * oscillations"): x_0 = 0, r_0 = b (masked, projected if nullspace), then
 *   z_k = M r_k;  x_{k+1} = x_k + z_k;  r_{k+1} = r_k - A z_k
 * until ||r_k|| <= rtol ||r_0|| (tested like Alg. 1 line 8).  M is the hierarchy's cycle
 * (its mg params, including beta).  Same buffers, report and synchronisation as
 * octmg_pcg_solve; report.iters = cycles applied.
 */
octmg_status octmg_mg_solve(octmg_hier* h, const float* b, float* x, const octmg_solve_params* params,
                            octmg_solve_report* report, octmg_stream stream);

/* Per-kernel-class device time of the work issued since the last reset while profiling
 * is on (CUDA events bracketing each launch on the launch stream; CUDA-graph replay is
 * disabled while profiling), with the launch count and the ALGORITHMIC bytes those
 * launches must move at minimum (e.g. 20 B per cell for an RBGS
 * colour pass in the colour-split cell order: the other colour's u and coupling planes,
 * its own colour's b and coefficient record, its own u written).  names/ms/counts/bytes:
 * arrays of cap entries (any may be NULL); *n = number of classes.  Synchronises. */
octmg_status octmg_profile_enable(octmg_hier* h, int32_t on);
octmg_status octmg_profile_read(octmg_hier* h, const char** names, double* ms, int64_t* counts,
                                double* bytes, int32_t cap, int32_t* n);
/* The same restricted to the multigrid work of one level (0 = coarsest; the classes in
 * octmg_profile_read's order; the PCG vector kernels have no level and are not counted).
 * Accumulates since the last octmg_profile_enable, like octmg_profile_read.  Synchronises. */
octmg_status octmg_profile_read_level(octmg_hier* h, int32_t level, double* ms, int64_t* counts, double* bytes,
                                      int32_t cap, int32_t* n);

void octmg_hier_destroy(octmg_hier* h);
void octmg_tree_destroy(octmg_tree* tree);

#ifdef __cplusplus
}
#endif
#endif /* OCTMG_H */
