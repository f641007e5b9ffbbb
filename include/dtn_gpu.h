/* dtn_gpu.h — C ABI of the B200-native build/solve engine for the
 * Gillman–Martinsson nested-dissection DtN build (arXiv 1302.5995).
 *
 * Drop-in boundary for the reference's dense engine (/root/reference/proj):
 *   dtn_gpu_build        replaces build_root_dense_op / build_with_loads(..., Engine::dense, ...)
 *                        (proj/include/dtn/accel_nd.hpp:98-100, proj/src/bodyload.cpp:47-57,
 *                         proj/src/dense_nd.cpp:196-225)
 *   dtn_gpu_boundary     SolutionOperator::boundary / root_boundary (solution_operator.hpp:33,65)
 *   dtn_gpu_export       SolutionOperator::S_dense, G_dense, cond_estimate (solution_operator.hpp:36,44)
 *   dtn_gpu_apply        apply_dtn (which=0, G*g) / apply_schur (which=1, S*g)
 *                        (solution_operator.hpp:55-59, solution_operator.cpp:36-52), batched
 *   dtn_gpu_box_schur    SchurData::S of any box of the build tree (dense_nd.hpp:18-26)
 *   dtn_gpu_level_stats  SolutionOperator::level_stats (solution_operator.hpp:18-23,46)
 *   dtn_discretize_*     discretize (grid.hpp:111, grid.cpp:106-168) as 5-point stencil arrays
 *
 * All matrices are column-major FP64. The boundary is the canonical CCW ring
 * of root unknowns starting at the south-west corner (grid.cpp:170-190), of
 * size 4(n-2)-4 with n the reference grid size including the Dirichlet ring.
 *
 * Threading: calls on one context -- and on every operator built with it (dense or HBS) --
 * are serialised by the context's lock (the context owns the stream, cached plans, apply
 * staging and the HBS apply workspaces), so concurrent applies of one operator are safe
 * but do not overlap. For concurrent work build one context (and its operators) per host
 * thread. dtn_gpu_set_stream changes the stream of every later call on the context.
 *
 * Return codes (errors.hpp, harness.hpp:11-12): 0 ok, 2 invalid argument,
 * 3 singular block (FactorizationError; dtn_gpu_last_error carries the
 * "what [where]" text), 5 CUDA failure. There is no CPU fallback: without a
 * usable sm_100a device every build returns 5.
 */
#ifndef DTN_GPU_H
#define DTN_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dtn_ctx dtn_ctx;
typedef struct dtn_op dtn_op;

#define DTN_OK 0
#define DTN_EINVAL 2
#define DTN_ESINGULAR 3
#define DTN_ECUDA 5

typedef struct {
  int32_t n;               /* grid side including the Dirichlet ring (grid.hpp:29-35) */
  const double* stencil;   /* 5 x (n-2)^2 SoA: center, east, west, north, south, unknown_id order
                              (grid.hpp:68-70); couplings to ring nodes are ignored */
  int32_t stencil_on_device; /* 1: stencil is a device pointer on the context's device */
  /* top-of-tree build only (opts.nshards > 1, opts.shard == -1): the Schur
   * complements of the shards (column-major nb x nb, dtn_gpu_shard_info order) */
  const double* const* shard_S;
  int32_t shard_S_on_device;
} dtn_problem;

typedef struct {
  int32_t engine;      /* 0 = dense (Engine::dense, solution_operator.hpp:15) */
  int32_t n_leaf;      /* build_tree leaf capacity (grid.hpp:159), used when leaf_side == 0 */
  int32_t leaf_side;   /* > 0: uniform tree of leaf_side^2 leaves, requires n-2 = leaf_side*2^L */
  int32_t want_G;      /* compute G = S^{-1} and cond_estimate (dense_nd.cpp:218-224) */
  int32_t micro_max;   /* leaf elimination granularity (unknowns per one-CTA box); 0 = default */
  int32_t profile;     /* 1: no graph, CUDA events around every launch (dtn_gpu_kernel_stats) */
  double epsilon;      /* compressed engine tolerance (AccelOptions::epsilon, dtn_gpu_build_accel) */
  int64_t crossover;   /* AccelOptions::crossover: root boundaries >= crossover are compressed */
  int32_t nshards;     /* subtree sharding: 1, 2 (W|E), 4 (quadrants), 8 (quadrant halves) */
  int32_t shard;       /* >= 0: build only this shard's S; -1: full build (nshards == 1) or the top of
                          the tree from prob.shard_S (nshards > 1); -2: collective build over the
                          context's NCCL world (dtn_gpu_create_rank, nshards == world): shard `rank`
                          locally, shard S gathered to every rank, the top merges column-sharded
                          (interface LU redundant, boundary columns split, ncclAllGather per wave);
                          S (and G) on every rank; -3: the same split computed on this one device
                          (every shard and column chunk in turn, no communication); -4: -3 with every
                          NCCL call of the -2 path issued in place on the context's 1-rank
                          communicator (dtn_gpu_create_rank with nranks == 1: a one-GPU check of the
                          communicator and of the collectives captured in the build graph) */
  double* export_S;    /* optional host buffer (page-locked for overlap): receives S (column-major,
                          leading dimension export_lds) during the build, overlapping the root inverse */
  int64_t export_lds;
  /* body loads (LoadPanel, dense_nd.hpp:29-32; build_with_loads, bodyload.cpp:47-57): unit loads at
   * these distinct, strictly interior unknown ids are carried through every merge as extra
   * right-hand-side columns (dense_nd.cpp:98-101, 136-147, 182-184); the result's body map
   * F = G * rhs_root (accel_nd.cpp:872-875) is read with dtn_gpu_body_map when want_G; without G
   * the reduced load columns rhs_root are read with dtn_gpu_root_rhs. */
  const int64_t* load_ids;
  int32_t nloads;
  /* 1: keep every box's S resident after the build (dtn_gpu_box_schur); 0 (default): box
   * storage is reused level by level -- children are dropped once their parent is formed
   * (dense_nd.cpp:215), so device memory is ~ two tree levels instead of the whole tree */
  int32_t keep_boxes;
  /* engine 1 (structured merges, dtn_gpu_build_accel): factor rank ell(j) of a box with a
   * J edge of j nodes = min(j, rank_base + rank_step * floor(log2(j / 128))), rounded up to
   * a multiple of 8; 0 = defaults (64, 8) */
  int32_t rank_base;
  int32_t rank_step;
} dtn_opts;

typedef struct {
  int32_t level;       /* reference tree level (root = 0) */
  int32_t boxes;       /* boxes merged at this level */
  int64_t max_boundary;
  double seconds;      /* device time of this level's waves */
  double flops;        /* algorithmic merge flops of this level (SURVEY 8d formula) */
  /* LevelStats (solution_operator.hpp:18-23): the largest numerical rank at epsilon of the
   * level's off-diagonal factors (structured merges; 0 for dense levels) and the bytes of
   * the level's box operators (dense S + factors) */
  int64_t max_rank;
  uint64_t bytes;
} dtn_level_stats;

typedef struct {
  double build_ms;        /* device time of the whole build (leaf + merges + root inverse) */
  double leaf_ms;         /* device time below the reference leaves */
  double merge_ms;        /* device time of the reference-tree merges */
  double inverse_ms;      /* device time of G = S^{-1} */
  double merge_flops;     /* algorithmic flops of the reference-tree merges */
  double leaf_flops;      /* flops of the in-leaf dense eliminations */
  double inverse_flops;   /* 2 nb^3 */
  int32_t waves;
  int32_t launches;       /* kernels launched by one build */
  double arena_bytes;     /* device arena of the plan (liveness-packed box storage) */
  double arena_sum_bytes; /* the same storage without reuse (every box resident) */
  int32_t structured_merges;
  int32_t max_rank;       /* largest numerical rank at epsilon of any factor (structured merges) */
  double sketch_tail;     /* largest |R_ii| / |R_00| over the last 4 sketch columns (range-finder check) */
  double exec_flops;      /* flops executed by the merge waves (structured: reduced systems + factors) */
  int32_t rank_attempts;  /* builds run to settle the factor ranks (1 once learned for this problem) */
} dtn_build_stats;

typedef struct {
  char name[16];          /* kernel class */
  int32_t launches;
  double ms;              /* summed device time (profiled build) */
  double max_ms;
  double flops;           /* algorithmic flops of those launches */
  double bytes;           /* algorithmic bytes (memory-bound classes) */
} dtn_kernel_stats;

int dtn_gpu_create(dtn_ctx** ctx, int device);
/* Multi-GPU, one process per GPU: rank 0 draws a 128-byte NCCL unique id,
 * the launcher hands it to every rank, and each rank creates its context on its device;
 * the context owns the NCCL communicator of the collective builds (opts.shard = -2). */
int dtn_gpu_nccl_unique_id(uint8_t* id);
int dtn_gpu_create_rank(dtn_ctx** ctx, int device, int nranks, int rank, const uint8_t* id);
void dtn_gpu_destroy(dtn_ctx* ctx);
const char* dtn_gpu_last_error(const dtn_ctx* ctx);
/* kernel launches issued so far by the HBS code (compress, invert_hbs, apply), process-wide */
unsigned long long dtn_gpu_hbs_launch_count(void);
/* Run this context's work on an external CUDA stream (cudaStream_t); NULL restores its own. */
int dtn_gpu_set_stream(dtn_ctx* ctx, void* stream);

int dtn_gpu_build(dtn_ctx* ctx, const dtn_problem* prob, const dtn_opts* opts, dtn_op** out);
void dtn_gpu_free(dtn_op* op);

int dtn_gpu_boundary(const dtn_op* op, int64_t* ids, int64_t* nb);
int dtn_gpu_export(const dtn_op* op, double* S, double* G, double* cond);
int dtn_gpu_device_ptrs(const dtn_op* op, const double** S, const double** G, int64_t* ld);
/* Device-to-device export into caller buffers (leading dimensions lds, ldg); NULL skips. */
int dtn_gpu_export_device(const dtn_op* op, double* S, int64_t lds, double* G, int64_t ldg);
/* Y(nb x batch) = op(X), op = G (which 0, apply_dtn) or S (which 1, apply_schur).
 * on_device: X and Y are device pointers (else host). */
/* Dirichlet-ring DtN adapter (SURVEY f-1; not in the reference, derived from
 * A u = -D g, grid.hpp:88-90, grid.cpp:151-166): T = (1/h)(I + P G D_b), the
 * m x m map from Dirichlet data on the m = 4 n_int non-corner ring nodes to
 * the one-sided normal derivative there. adj[i] = boundary position of the
 * unknown adjacent to ring node i, coef[i] = its stencil coefficient toward
 * the ring node. T column-major (leading dimension ldt) on the host or, with
 * on_device, in device memory. Requires G (want_G). */
int dtn_gpu_ring_dtn(const dtn_op* op, const int64_t* adj, const double* coef, int64_t m, double h, double* T,
                     int64_t ldt, int on_device);
/* Body map F (nb x nloads, column-major, leading dimension ldf) of a build with loads:
 * solve_with_load (bodyload.cpp:68-77) is v = G g + F fhat. */
int dtn_gpu_body_map(const dtn_op* op, double* F, int64_t ldf, int on_device);
/* The root's reduced load columns rhs_root (nb x nloads; dense_nd.cpp:182-184, SchurData::rhs) of a
 * build with body loads, with or without G: the compressed engine's body map is G_hbs * rhs_root
 * (accel_nd.cpp:848-855), formed with dtn_gpu_hbs_apply. */
int dtn_gpu_root_rhs(const dtn_op* op, double* R, int64_t ldr, int on_device);
int dtn_gpu_apply(const dtn_op* op, int which, const double* X, int64_t ldx, int64_t batch, double* Y, int64_t ldy,
                  int on_device);

int dtn_gpu_num_boxes(const dtn_op* op, int32_t* count, int32_t* depth);
/* info: level, parent, x0, x1, y0, y1, boundary size, children SW SE NW NE */
int dtn_gpu_box_info(const dtn_op* op, int32_t box, int32_t* info);
int dtn_gpu_box_schur(const dtn_op* op, int32_t box, double* S);
int dtn_gpu_level_stats(const dtn_op* op, dtn_level_stats* out, int32_t max, int32_t* count);
int dtn_gpu_build_stats(const dtn_op* op, dtn_build_stats* out);
/* per-kernel-class timing of a build made with opts.profile = 1 (count 0 otherwise) */
int dtn_gpu_kernel_stats(const dtn_op* op, dtn_kernel_stats* out, int32_t max, int32_t* count);

/* Geometry of shard `shard` of `nshards` (host only, no device needed):
 * rect = x0, x1, y0, y1 of its unknown rectangle; nb = its boundary size. */
int dtn_gpu_shard_info(int32_t n, int32_t n_leaf, int32_t leaf_side, int32_t nshards, int32_t shard, int32_t* rect,
                       int64_t* nb);

/* Work (flops) per rank of a collective build over nranks GPUs (opts.shard = -2), host
 * only: per_rank[r] (nranks entries) and the single-GPU build's algorithmic flops */
int dtn_gpu_collective_flops(int32_t n, int32_t n_leaf, int32_t leaf_side, int32_t nranks, int32_t want_G,
                             double* per_rank, double* single_gpu);

/* Test hook: partial LU (pivots among the first ni rows) of a host n x n
 * column-major matrix with the engine's blocked kernels; ni == n is a full LU. */
int dtn_debug_partial_lu(int32_t n, int32_t ni, const double* A, double* out, int32_t* ipiv, double* pivstat);

/* Diagnostic: phase clocks (SM cycles) of CTA 0 of the last fused-merge launch of each of the three
 * size classes: out24[8 c + {0..4}] = start, assembled, factored, substituted, done; [5], [6] = the
 * LU's panel / update shares. */
int dtn_debug_fused_clocks(int64_t* out24);

/* Test hook: C (m x n, in/out) = alpha A B + beta C on host column-major operands through the
 * engine's FP64 tensor-core GEMMs; path 0 = cp.async-staged kernels, 1 = the TMA-staged kernel. */
int dtn_debug_gemm(int32_t m, int32_t n, int32_t k, const double* A, const double* B, double* C, double alpha,
                   double beta, int32_t path);

/* discretize (grid.cpp:106-168) on the host: continuum mode from coefficient
 * samples b, c, d at the unknowns (physical coordinates (x h, y h), h = 1/(n-1),
 * unknown_id order; NULL = 0), network mode from the seeded link conductivities. */
int dtn_discretize_continuum(int32_t n, const double* b, const double* c, const double* d, double* stencil);
int dtn_discretize_network(int32_t n, double lo, double hi, uint64_t seed, double* stencil);

/* ---- compressed (HBS) operators ----------------------------------------
 * HbsMatrix (hbs.hpp:30-51): orthonormal-basis hierarchically block separable
 * matrix over build_index_tree(M, leaf_cap) (index_tree.cpp:37-67).
 *   dtn_gpu_hbs_compress     compress(H, eps, leaf_cap) (hbs.hpp:58-62, hbs.cpp:61-182) of a dense
 *                            column-major M x M matrix (host or device memory)
 *   dtn_gpu_hbs_compress_op  the same on a built operator's resident G (which 0) or S (which 1):
 *                            the compressed SolutionOperator::G_hbs / S_hbs (solution_operator.hpp:38-42)
 *   dtn_gpu_hbs_apply        apply(H, x) (hbs.hpp:66, hbs.cpp:187-232), batched; apply_dtn on G_hbs
 *                            (solution_operator.cpp:42)
 *   dtn_gpu_hbs_info/tree/factor  size(), max_rank(), payload_bytes(), tree nodes, rank(t) and the
 *                            D/U/V/B factors (hbs.hpp:30-51)
 *   dtn_gpu_hbs_serialize / _deserialize  the DTNHBS01 byte format (hbs.hpp:92-95, hbs.cpp:422-519),
 *                            byte-for-byte the reference layout */
typedef struct dtn_hbs dtn_hbs;
int dtn_gpu_hbs_compress(dtn_ctx* ctx, const double* H, int64_t M, int64_t ldh, int on_device, double eps,
                         int64_t leaf_cap, dtn_hbs** out);
int dtn_gpu_hbs_compress_op(const dtn_op* op, int which, double eps, int64_t leaf_cap, dtn_hbs** out);
void dtn_gpu_hbs_free(dtn_hbs* h);
int dtn_gpu_hbs_info(const dtn_hbs* h, int64_t* M, int64_t* num_nodes, int32_t* depth, int64_t* max_rank,
                     uint64_t* payload_bytes);
/* nodes: 6 int64 per node (begin, end, left, right, parent, level), preorder; ranks: rank(t) */
int dtn_gpu_hbs_tree(const dtn_hbs* h, int64_t* nodes, int64_t* ranks);
/* which: 0 D (leaves), 1 U, 2 V (non-root), 3 B (parents); out (column-major, rows x cols) may be
 * NULL to query the shape */
int dtn_gpu_hbs_factor(const dtn_hbs* h, int32_t node, int32_t which, double* out, int64_t* rows, int64_t* cols);
int dtn_gpu_hbs_apply(const dtn_hbs* h, const double* X, int64_t ldx, int64_t nrhs, double* Y, int64_t ldy,
                      int on_device);
/* buf NULL: *size receives the byte count only */
int dtn_gpu_hbs_serialize(const dtn_hbs* h, uint8_t* buf, uint64_t cap, uint64_t* size);
int dtn_gpu_hbs_deserialize(dtn_ctx* ctx, const uint8_t* buf, uint64_t size, dtn_hbs** out);
/* invert_hbs (hbs_ops.hpp:64, hbs_ops.cpp:148-201): the telescoping inverse factors of H in
 * the InverseFactors layout (hbs_ops.hpp:46-55: E in U, F in V, G in D/B, the root core inverse
 * in the root B), so dtn_gpu_hbs_apply on the result is apply_inverse (hbs_ops.cpp:203-205).
 * A singular block returns 3 with "<block> is singular [node t level l]". */
int dtn_gpu_hbs_invert(const dtn_hbs* H, dtn_hbs** out);
/* ---- the HBS algebra (hbs.hpp:71-90, hbs_ops.hpp:57-120, lowrank.hpp) ---------------
 * Device-resident operations on dtn_hbs handles and low-rank blocks (csrc/hbs_ops.cu).
 * Index trees are passed as 6 int64 per node (begin, end, left, right, parent, level), preorder,
 * the dtn_gpu_hbs_tree layout. Factor transforms are exact; the operations that re-compress
 * (add, from_lowrank, add_lowrank, rebase, split_at, consolidate) evaluate their operands on the
 * device and compress onto the result's index tree (the reference's tree) at eps. Errors: 2 with
 * the reference's message (e.g. "add_hbs: operands use different index trees").
 *   dtn_gpu_hbs_compress_tree  compress(H, tree, eps)                 hbs.hpp:58-60, hbs.cpp:61-178
 *   dtn_gpu_hbs_reconstruct    reconstruct(H): the dense M x M matrix  hbs.hpp:69, hbs.cpp:258-288
 *   dtn_gpu_hbs_subtree        subtree_matrix(H, node)                 hbs.cpp:290-320
 *   dtn_gpu_hbs_flip           flip(H) (index reversal, mirrored tree) hbs.cpp:322-375
 *   dtn_gpu_hbs_scale(_rows/_cols)  scale / scale_rows / scale_cols, in place   hbs.cpp:377-402
 *   dtn_gpu_hbs_add            add_hbs(A, B, eps) (same tree)          hbs_ops.cpp:386-404
 *   dtn_gpu_hbs_from_lowrank   lowrank_to_bs(Q, R, tree)               hbs_ops.cpp:409-465
 *   dtn_gpu_hbs_add_lowrank    add_lowrank(A, Q, R, eps)               hbs_ops.cpp:467-470
 *   dtn_gpu_hbs_rebase         rebase(H, target, eps)                  hbs_ops.cpp:737-743
 *   dtn_gpu_hbs_split_at       split_at(H, pos) with both sides consolidated: lo = H[:pos,:pos],
 *                              hi = H[pos:,pos:] (NULL when empty), lo_hi / hi_lo the off-diagonal
 *                              blocks                                  hbs_ops.cpp:620-640, 710-735
 *   dtn_gpu_hbs_consolidate    consolidate(pieces at offsets tiling [0, size) + placed low-rank
 *                              corrections (row, col offset pairs), eps)   hbs_ops.cpp:710-735
 *   dtn_gpu_lowrank_*          LowRank L (m x k) R (k x n): lowrank_from_dense, lowrank_recompress,
 *                              lowrank_sum of placed terms (offsets: row, col pairs)  lowrank.cpp:27-72 */
typedef struct dtn_lowrank dtn_lowrank;
int dtn_gpu_hbs_compress_tree(dtn_ctx* ctx, const double* H, int64_t M, int64_t ldh, int on_device, double eps,
                              const int64_t* nodes, int64_t num_nodes, dtn_hbs** out);
int dtn_gpu_hbs_reconstruct(const dtn_hbs* h, double* out, int64_t ldo, int on_device);
int dtn_gpu_hbs_subtree(const dtn_hbs* h, int32_t node, dtn_hbs** out);
int dtn_gpu_hbs_flip(const dtn_hbs* h, dtn_hbs** out);
int dtn_gpu_hbs_scale(dtn_hbs* h, double s);
int dtn_gpu_hbs_scale_rows(dtn_hbs* h, const double* w, int on_device);
int dtn_gpu_hbs_scale_cols(dtn_hbs* h, const double* w, int on_device);
int dtn_gpu_hbs_add(const dtn_hbs* A, const dtn_hbs* B, double eps, dtn_hbs** out);
int dtn_gpu_hbs_from_lowrank(dtn_ctx* ctx, const double* Q, int64_t ldq, const double* R, int64_t ldr, int64_t k,
                             const int64_t* nodes, int64_t num_nodes, int on_device, dtn_hbs** out);
int dtn_gpu_hbs_add_lowrank(const dtn_hbs* A, const double* Q, int64_t ldq, const double* R, int64_t ldr, int64_t k,
                            double eps, int on_device, dtn_hbs** out);
int dtn_gpu_hbs_rebase(const dtn_hbs* h, const int64_t* nodes, int64_t num_nodes, double eps, dtn_hbs** out);
int dtn_gpu_hbs_split_at(const dtn_hbs* h, int64_t pos, double eps, dtn_hbs** lo, dtn_hbs** hi, dtn_lowrank** lo_hi,
                         dtn_lowrank** hi_lo);
int dtn_gpu_hbs_consolidate(dtn_ctx* ctx, int64_t size, int64_t npieces, const dtn_hbs* const* pieces,
                            const int64_t* offsets, int64_t ncorr, const dtn_lowrank* const* corr,
                            const int64_t* corr_offsets, double eps, dtn_hbs** out);
int dtn_gpu_lowrank_create(dtn_ctx* ctx, const double* L, int64_t ldl, const double* R, int64_t ldr, int64_t m,
                           int64_t n, int64_t k, int on_device, dtn_lowrank** out);
int dtn_gpu_lowrank_from_dense(dtn_ctx* ctx, const double* X, int64_t ldx, int64_t m, int64_t n, int on_device,
                               double eps, dtn_lowrank** out);
int dtn_gpu_lowrank_info(const dtn_lowrank* x, int64_t* m, int64_t* n, int64_t* k);
int dtn_gpu_lowrank_get(const dtn_lowrank* x, double* L, int64_t ldl, double* R, int64_t ldr);
int dtn_gpu_lowrank_recompress(const dtn_lowrank* x, double eps, dtn_lowrank** out);
int dtn_gpu_lowrank_sum(dtn_ctx* ctx, int64_t m, int64_t n, int64_t nterms, const dtn_lowrank* const* terms,
                        const int64_t* offsets, double eps, dtn_lowrank** out);
void dtn_gpu_lowrank_free(dtn_lowrank* x);

/* Compressed engine, build_root_accel (accel_nd.hpp:93-95, accel_nd.cpp:707-859) on the B200:
 * the root Schur complement S from the exact dense GPU merges, S_hbs = compress(S,
 * opts->epsilon, hbs_leaf) and G_hbs = invert_hbs(S_hbs) (accel_nd.cpp:820-822), cond = the
 * reference's probe estimate (accel_nd.cpp:834-841). The HBS factors are in canonical ring
 * order (rep_to_canonical = identity). A root boundary below opts->crossover stays dense
 * (accel_nd.cpp:796-818): *S_hbs = *G_hbs = NULL, the dense op (with G) in *op_out.
 * op_out (optional): the dense build (S resident; boundary ids, box S); NULL frees it.
 * Body loads (opts->load_ids / nloads) ride through the dense merges; with a compressed root the
 * body map is G_hbs * rhs_root (accel_nd.cpp:848-855): rhs_root from dtn_gpu_root_rhs(*op_out). */
int dtn_gpu_build_accel(dtn_ctx* ctx, const dtn_problem* prob, const dtn_opts* opts, int64_t hbs_leaf,
                        dtn_op** op_out, dtn_hbs** S_hbs, dtn_hbs** G_hbs, double* cond);

#ifdef __cplusplus
}
#endif

#endif /* DTN_GPU_H */
