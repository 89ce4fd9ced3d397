/*
 * scvt_b200.h — C ABI of the B200-native SCVT energy/gradient + Lloyd-P-LBFGS hot path.
 *
 * The reference (`scvtmesh` 0.1.0, pure Python) has no FFI: its drop-in boundary is the
 * duck-typed evaluator protocol consumed by `optimizer.minimize`
 * (/root/reference/pkg/src/scvtmesh/optimizer.py:278-391) and implemented by
 * `MeshEvaluator.evaluate` (pipeline.py:261-279).  Each entry point below replaces one piece
 * of that protocol or of the optimizer's vector algebra; the citation names the reference
 * code it stands in for.  The Python package `paper_1709_06924_b200` binds these with ctypes
 * (see INTEGRATION.md), exactly as a maintainer would bind them from the reference.
 *
 * Conventions
 *   - All array pointers are DEVICE pointers to caller-owned, contiguous float64 / int64
 *     buffers (row-major (n,3) for points/vectors).  The library never frees caller memory.
 *   - Scalars documented as "host out" are written to host memory; those calls synchronise
 *     the context's stream.  All other calls are stream-ordered on the context stream.
 *   - Return value: SCVT_OK (0) or one of the status codes below (1:1 with scvtmesh.errors).
 *     `scvt_last_error` gives the message.  One context per (process, device).
 */
#ifndef SCVT_B200_H
#define SCVT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum scvt_status {
    SCVT_OK = 0,
    SCVT_ERR_INSUFFICIENT_POINTS = 1, /* InsufficientPointsError  delaunay.py:189-199        */
    SCVT_ERR_DEGENERATE_TRIANGLE = 2, /* DegenerateTriangleError  delaunay.py:157-160        */
    SCVT_ERR_COVERAGE = 3,            /* CoverageError            delaunay.py:295-302        */
    SCVT_ERR_CENTROID_AT_ORIGIN = 4,  /* CentroidAtOriginError    optimizer.py:240-246       */
    SCVT_ERR_NONPOSITIVE_DIAGONAL = 5,/* NonpositiveDiagonalError cvt_core.py:176-189        */
    SCVT_ERR_NON_DESCENT = 6,         /* NonDescentError          optimizer.py:165-166       */
    SCVT_ERR_LINE_SEARCH = 7,         /* LineSearchFailure        optimizer.py:190-192       */
    SCVT_ERR_POLE_AMBIGUITY = 8,      /* PoleAmbiguityError       density.py:82-90           */
    SCVT_ERR_CONFIG = 9,              /* ConfigError / ValueError                             */
    SCVT_ERR_CAPACITY = 10,           /* n > n_max, valence/polygon capacity exceeded          */
    SCVT_ERR_CUDA = 11,               /* CUDA runtime failure                                  */
    SCVT_ERR_NCCL = 12,               /* collective failure (multi-GPU plumbing)               */
    SCVT_ERR_FACTORIZATION = 13       /* FactorizationError       cvt_core.py:218-236        */
};

/* density kinds (density.py:116-129 + BASELINE tanh^4 variants, DECISIONS.md D3/D4) */
enum scvt_density_kind {
    SCVT_DENSITY_CONST = 0,   /* rho = 1                                                      */
    SCVT_DENSITY_X3 = 1,      /* (1-g) z^4 + g                                                */
    SCVT_DENSITY_X16 = 2,     /* reference tanh plateau, elliptical distance (density.py:100) */
    SCVT_DENSITY_TANH = 3,    /* reference tanh plateau, geodesic distance (x64 / 'tanh')     */
    SCVT_DENSITY_TANH4 = 4,   /* (((1-g)/2)(tanh((b-d)/a)+1)+g)^4, one centre                 */
    SCVT_DENSITY_TANH4X2 = 5  /* same, d = min over two centres                               */
};

typedef struct scvt_config {
    int32_t density_kind;     /* enum scvt_density_kind                                        */
    int32_t measure;          /* 0 = "flat", 1 = "sphere"  (cvt_core.py:67-92)                 */
    double gamma, beta, alpha;
    double center[6];         /* one or two unit centres (x,y,z)                               */
    double w_lon, w_lat;      /* x16 only                                                      */
    int32_t n_nodes;          /* composite rule size = 4^depth * Q  (<= SCVT_MAX_NODES)        */
    int32_t lbfgs_m;          /* correction pairs kept (optimizer.py:79-90)                    */
    const double* node_l1;    /* HOST arrays [n_nodes]: barycentric (l1, l2) of each composite */
    const double* node_l2;    /*   node relative to the fan sub-triangle (v0, v1, v2) and its  */
    const double* node_w;     /*   weight  w_q / 4^depth  (geometry.py:142-185 + 383-407)      */
    /* optional piecewise-polynomial form of rho^(1/4) for the tanh4 kinds (NULL = evaluate
     * the closed form with atan2/tanh per node).  HOST array [2][table_intervals]
     * [table_degree+1]: branch 0 in x = |y - c|, branch 1 in x = |y + c|, x in [0, sqrt 2],
     * interval width table_width, local variable tau = 2 (x/w - k) - 1, monomial coeffs. */
    int32_t table_intervals;
    int32_t table_degree;     /* must equal SCVT_TABLE_DEGREE                               */
    double table_width;
    const double* table_coef;
} scvt_config;

#define SCVT_TABLE_DEGREE 6

#define SCVT_MAX_NODES 2304
#define SCVT_MAX_DEGREE 32

typedef struct scvt_ctx scvt_ctx;

/* lifecycle ---------------------------------------------------------------------------- */
int scvt_create(scvt_ctx** ctx, int device, int64_t n_max, const scvt_config* cfg);
int scvt_destroy(scvt_ctx* ctx);
const char* scvt_last_error(const scvt_ctx* ctx);
/* cudaStream_t as void*; NULL = legacy default stream */
int scvt_set_stream(scvt_ctx* ctx, void* stream);
/* library version string */
const char* scvt_version(void);

/* triangulation ------------------------------------------------------------------------
 * Replaces convex_hull_delaunay (delaunay.py:181-202) incl. _ccw_outward/_canonical_sort
 * (133-147, 172-178): writes the canonical (2n-4, 3) int64 triangle list (CCW seen from
 * outside, min-ID first, lexicographically sorted) and one flag byte per triangle
 * (1 = an edge of it failed the FP64 in-circle filter: cocircular candidate).
 * stats_host[0..7] = {triangle count, flagged triangles, max valence, filter-undecided
 * directed edges, symbolic-perturbation tie-breaks, max candidate passes of one cell,
 * cells that needed the unsorted sweep, 32-point batches those sweeps visited}. */
int scvt_triangulate(scvt_ctx* ctx, const double* z, int64_t n, int64_t* tri_out,
                     uint8_t* flags_out, int64_t* stats_host);

/* evaluation ---------------------------------------------------------------------------
 * Consecutive evaluations of the same n reuse the previous cycles when the robust certificate
 * (consistency, orientation, local Delaunay on every edge) still holds at the new positions;
 * edges failing only the in-circle test are repaired by Lawson edge flips (env SCVT_NO_FLIPS=1:
 * rebuilt instead), other failing neighbourhoods are rebuilt, and every touched cell is
 * certified again, so the result is always THE Delaunay triangulation (env SCVT_NO_REUSE=1
 * disables the reuse).
 * Replaces MeshEvaluator.evaluate (pipeline.py:261-279) = triangulation + Voronoi fans
 * (delaunay.py:337-380) + depth-d subdivision (383-407) + cell_quadrature
 * (cvt_core.py:55-117) + gradient assembly.  Outputs (device): grad (n,3) =
 * 2(c.z)z - 2c, first (n,3) = c, mass (n,) = m (may be NULL), lloyd_diag (n,) = 2 c.z.
 * scalars_host[0..2] = {energy, grad_norm, obtuse triangle count}. */
int scvt_evaluate(scvt_ctx* ctx, const double* z, int64_t n, double* grad, double* first,
                  double* mass, double* lloyd_diag, double* scalars_host);

/* scvt_evaluate plus, in the same fixed-shape reduction: scalars_host[3] = min lloyd_diag (the
 * nonpositive-diagonal test of cvt_core.py:184) and, when q3/norms are given (a line-search
 * trial at v = z + alpha q3, norms = |v|), scalars_host[4] = sum g.(q3/|v|) (optimizer.py:330).
 * scalars_host must hold 5 doubles. */
int scvt_evaluate_ex(scvt_ctx* ctx, const double* z, int64_t n, double* grad, double* first,
                     double* mass, double* lloyd_diag, const double* q3, const double* norms,
                     double* scalars_host);

/* scvt_evaluate_ex for a line-search trial that also STAGES the correction pair the optimizer
 * would push if it accepts this point (s = z - z_old, y = grad - g_old; optimizer.py:351-353):
 * the pair's scalars (y.s, s.s, y.y, max|s| and the products with the stored pairs) are reduced
 * with the evaluation's and come back in the same host read, so that
 * scvt_history_commit_staged needs no kernel pass and no host round trip.  A later evaluation,
 * scvt_history_push or scvt_history_clear drops the staged pair. */
int scvt_evaluate_staged(scvt_ctx* ctx, const double* z, int64_t n, double* grad, double* first,
                         double* mass, double* lloyd_diag, const double* q3, const double* norms,
                         const double* z_old, const double* g_old, double* scalars_host);

/* Moments only over an externally supplied canonical triangulation (T,3) int64 — used by
 * parity tests to isolate the quadrature from the triangulation. Same outputs as above. */
int scvt_evaluate_on_triangles(scvt_ctx* ctx, const double* z, int64_t n,
                               const int64_t* triangles, int64_t t, double* grad,
                               double* first, double* mass, double* lloyd_diag,
                               double* scalars_host);

/* Per-cell energy E_i = sum over the cell's fan sub-triangles of int rho |y - z_i|^2 (the
 * terms cvt_core.py:97-100 sums into the scalar energy) of the last single-GPU evaluation,
 * copied into energy_out (n doubles, device memory).  Parity tests compare it per cell. */
int scvt_cell_energy(scvt_ctx* ctx, int64_t n, double* energy_out);

/* sharded evaluation (one process per GPU) -------------------------------------------------
 * The generators are split into `nshards` equal ranges of the cube-map bucket order; shard s
 * owns rows [s*R, (s+1)*R) with R = scvt_shard_rows(n, nshards).  Per evaluation:
 *   scvt_shard_cells    grid (replicated) + cells of the owned generators -> cyc_send
 *                       int32 [R][34] = {id, valence, 32 neighbour ids}   (id -1 = padding)
 *   <caller all-gathers cyc_send -> cyc_all [nshards*R][34]>
 *   scvt_shard_moments  certificate of the owned cells against all cycles, owned fan
 *                       quadrature -> res_send f64 [R][8] = {id, m, c(3), E, obtuse, 0};
 *                       status_host = device status bits (0 = ok)
 *   <caller all-reduces status (max); nonzero -> scvt_shard_status maps it to a code>
 *   <caller all-gathers res_send -> res_all [nshards*R][8]>
 *   scvt_shard_finish   scatter to id order, gradient epilogue and the fixed-shape
 *                       reductions -> identical outputs to scvt_evaluate, bitwise, for any
 *                       shard count.
 * Stands in for the reference's region path (pipeline.py:171-242: partition, per-region
 * triangulation on a worker pool, gather in fixed region order). */
int64_t scvt_shard_rows(int64_t n, int nshards);
int scvt_shard_cells(scvt_ctx* ctx, const double* z, int64_t n, int shard, int nshards,
                     int32_t* cyc_send);
/* cyc_all may be NULL after the reuse rounds below certified the context's cycles */
int scvt_shard_moments(scvt_ctx* ctx, const double* z, int64_t n, int shard, int nshards,
                       const int32_t* cyc_all, double* res_send, int32_t* status_host);

/* sharded cycle reuse: the single-GPU reuse loop (previous evaluation's cycles certified at
 * the new positions, failing cells rebuilt, re-certified) split at its exchanges.  After a
 * successful evaluation every rank holds all n certified cycles, identically.  Per round r:
 *   scvt_shard_recheck  r = 0: grid (replicated) and the certificate of the owned cells
 *                       against the held cycles; r > 0: the owned cells of the last plan's
 *                       re-check list.  bad_out int32[n]: 1 for every generator of a failing
 *                       triangle seen by this shard.  *ready_host = 0 at r = 0 when the context
 *                       holds no cycles for n points (take the scvt_shard_cells path).
 *   <caller all-reduces bad_out (max) -> bad_all>
 *   scvt_shard_plan     bad set, the next round's re-check list (bad cells and their
 *                       current neighbours) and counts_host int64[nshards+1] = bad cells per
 *                       shard, total.  Identical on every rank.  Total 0: certified, call
 *                       scvt_shard_moments(cyc_all = NULL).
 *   scvt_shard_rebuild  rebuild this shard's bad cells -> rows_send int32[cap][34] (cap = max
 *                       per-shard count; padding id -1)
 *   <caller all-gathers rows_send -> rows [nshards*cap][34]>
 *   scvt_shard_install  write the gathered rows into the held cycles
 * Bad set, re-check lists and rebuilt cells equal the single-GPU loop's, so the certified
 * triangulation (unique) and every output are bitwise those of scvt_evaluate. */
int scvt_shard_recheck(scvt_ctx* ctx, const double* z, int64_t n, int shard, int nshards,
                       int round, int32_t* bad_out, int32_t* ready_host);
/* before the rounds: the flip repair of the held cycles, replicated on every rank (the
 * cycles are replicated and the repair is deterministic, so no exchange is needed).
 * *nbad_host = 0: certified, call scvt_shard_moments(cyc_all = NULL); > 0: cells left for the
 * rounds above; -1: no held cycles for n points (or reuse/flips disabled). */
int scvt_shard_flip(scvt_ctx* ctx, const double* z, int64_t n, int32_t* nbad_host);
/* the same repair with the certificate pass sharded: each rank runs the flip-mode certificate
 * of its owned cells -> cand_send int32 [cap][4] ({i, a, b, c} per non-Delaunay edge) and
 * counts_host = {candidates (> cap: overflow; -1: no held cycles), bad cells};
 * <caller all-gathers the counts; any bad cell or overflow -> the rounds above; else it
 * all-gathers cand_send (padded to the largest count) -> cand_all [nshards*cap][4]>;
 * scvt_shard_flip_rounds then runs the (replicated, deterministic) flip rounds on the
 * concatenated candidates; *nbad_host = 0: certified. */
int scvt_shard_flip_detect(scvt_ctx* ctx, const double* z, int64_t n, int shard, int nshards,
                           int32_t* cand_send, int64_t cap, int32_t* counts_host);
int scvt_shard_flip_rounds(scvt_ctx* ctx, const double* z, int64_t n, int nshards,
                           const int32_t* cand_all, int64_t cap, const int64_t* counts,
                           int32_t* nbad_host);
int scvt_shard_plan(scvt_ctx* ctx, int64_t n, int nshards, const int32_t* bad_all,
                    int64_t* counts_host);
int scvt_shard_rebuild(scvt_ctx* ctx, int64_t n, int shard, int nshards, int64_t cap,
                       int32_t* rows_send);
int scvt_shard_install(scvt_ctx* ctx, int64_t n, const int32_t* rows, int64_t nrows);
/* scvt_shard_moments for certified held cycles (cyc_all == NULL) without a host read: k_quad
 * takes the shard's incidence count from the device and the status word is copied to
 * status_dev (device, 1 int32) for the caller's all-gather of the ranks' status words. */
int scvt_shard_moments_async(scvt_ctx* ctx, const double* z, int64_t n, int shard, int nshards,
                             double* res_send, int32_t* status_dev);
int scvt_shard_status(scvt_ctx* ctx, int32_t status);
int scvt_shard_finish(scvt_ctx* ctx, const double* z, int64_t n, int nshards,
                      const double* res_all, double* grad, double* first, double* mass,
                      double* lloyd_diag, double* scalars_host);
/* as scvt_shard_finish with the extra scalars of scvt_evaluate_ex (5 doubles) */
int scvt_shard_finish_ex(scvt_ctx* ctx, const double* z, int64_t n, int nshards,
                         const double* res_all, double* grad, double* first, double* mass,
                         double* lloyd_diag, const double* q3, const double* norms,
                         double* scalars_host);

/* arithmetic-layout slices (multi-GPU optimizer algebra) -----------------------------------
 * The generator ids are cut into SCVT_CHUNKS fixed chunks of ceil(n / SCVT_CHUNKS) ids; rank r
 * of W (W divides SCVT_CHUNKS) owns the chunks [r C/W, (r+1) C/W), i.e. the ids [lo, hi) of
 * scvt_slice_range.  Its LBFGS vectors (grad, first, lloyd_diag, q3, norms, the history ring)
 * hold only those rows (slice-local: index 0 = id lo); positions stay replicated.  Every
 * reduction of the optimizer is written per chunk into a caller-owned partials buffer
 * red f64 [nval][SCVT_CHUNKS] that is zero outside the owned chunks; the caller sums the
 * buffers over the ranks (all-reduce SUM — each entry has exactly one non-zero contributor,
 * so the sum is exact) and the next call reduces the SCVT_CHUNKS partials in a fixed order.
 * Every scalar is therefore bitwise the same for any W, and the single-GPU entry points run
 * the same kernels with W = 1.  Replaces the paper's distributed LBFGS dot products
 * (the reference's optimizer.py:147-167 and 340-355 on one process).
 *   evaluation   scvt_slice_finish (5 values) -> <sum> -> scvt_slice_scalars
 *   direction    scvt_slice_gram (nval values, 0 with an empty history) -> <sum> ->
 *                scvt_slice_combine (2 values: q.g, g.q3) -> <sum> -> scvt_reduce_chunks
 *   fallback     scvt_slice_tangent (1 value: g.q3) -> <sum> -> scvt_reduce_chunks
 *   history      scvt_slice_history_pair (nval = 4 + 2K values) -> <sum> ->
 *                scvt_slice_history_commit (curvature test, ring commit, movement)
 *   trial point  scvt_trial_point on the slice rows, then the caller all-gathers z_t. */
#define SCVT_CHUNKS 1184
int scvt_slice_range(int64_t n, int rank, int world, int64_t* lo, int64_t* hi);
/* scatter of the gathered shard results (res_all of scvt_shard_moments) to this slice,
 * gradient epilogue; 5 values: E, |g|^2, obtuse, min lloyd_diag, sum g.(q3/norms) */
int scvt_slice_finish(scvt_ctx* ctx, const double* z, int64_t n, int nshards,
                      const double* res_all, int rank, int world, double* grad, double* first,
                      double* mass, double* lloyd_diag, const double* q3, const double* norms,
                      double* red);
/* scalars_host[5] = {energy, |g|, obtuse, min lloyd_diag, dphi} (as scvt_evaluate_ex) */
int scvt_slice_scalars(scvt_ctx* ctx, const double* red, double* scalars_host);
int scvt_slice_gram(scvt_ctx* ctx, const double* g, const double* lloyd_diag, double gamma,
                    int64_t n, int rank, int world, double* red, int32_t* nval_host);
/* red may alias red_gram (the recursion consumes it first, stream-ordered) */
int scvt_slice_combine(scvt_ctx* ctx, const double* g, const double* lloyd_diag, double gamma,
                       const double* z, int64_t n, int rank, int world, const double* red_gram,
                       double* q3, double* red);
int scvt_slice_tangent(scvt_ctx* ctx, const double* q, const double* z, const double* g,
                       int64_t n, int rank, int world, double* q3, double* red);
int scvt_slice_history_pair(scvt_ctx* ctx, const double* z_old, const double* z_new,
                            const double* g_old, const double* g_new, int64_t n, int rank,
                            int world, double* red, int32_t* nval_host);
int scvt_slice_history_commit(scvt_ctx* ctx, const double* red, int64_t n, int rank, int world,
                              int32_t* pushed_host, double* movement_host);
/* fixed-order reduction of nval values (ops[v]: 0 sum, 1 max, 2 min; NULL = all sums) */
int scvt_reduce_chunks(scvt_ctx* ctx, const double* red, int32_t nval, const uint8_t* ops,
                       double* out_host);

/* covering migration (region-mode bookkeeping; partition.py:123-164, pipeline.py:163-167,
 * 244-259, optimizer.py:377-381) ----------------------------------------------------------
 * geometric cell of every point = argmax_c z.centers[c] (ties to the lowest index).
 * fresh != 0: arithmetic[i] = geometric cell (assign_points without a frozen layout);
 * otherwise *class_host = 0 in-place, 1 neighbor-move (every moved point's geometric cell is a
 * one-level neighbour of its arithmetic cell: bit (a, g) of the row-major p x ceil(p/32)
 * uint32 `adjacency` bitmap), 2 out-of-range (detect_migration). */
int scvt_migration(scvt_ctx* ctx, const double* z, int64_t n, const double* centers, int32_t p,
                   const uint32_t* adjacency, int32_t* arithmetic, int32_t fresh,
                   int32_t* class_host);

/* region-path fallback decision (MeshEvaluator.fallbacks, pipeline.py:127-128, 244-259),
 * right after the evaluation of these n points: *fail_host = 0 when the reference's region
 * path would succeed for the covering (centers (p,3), one-level `adjacency` bitmap as above,
 * eps_proj of the stereographic projection), else a bit set: 1 a Delaunay triangle at an
 * owned generator is not kept by select_region_triangles (CoverageError, truncated fan),
 * 2 a member near its region's projection antipode (AntipodeError), 4 a region with owned
 * points has < 3 members (InsufficientPointsError); region_fail_host (p host ints, may be
 * NULL) gets the bits of every region (0 for regions without owned points, which the
 * reference does not triangulate).  p <= 128.  Moments do not depend on it (the
 * reference falls back to the global path, which this library always evaluates). */
int scvt_region_cover(scvt_ctx* ctx, const double* z, int64_t n, const double* centers,
                      int32_t p, const uint32_t* adjacency, double eps_proj, int32_t* fail_host,
                      int32_t* region_fail_host);   /* optional: the bits per region (p) */

/* graph Laplacian preconditioner (methods laplacian-a6 / laplacian-m2) ---------------------
 * LaplacianPreconditioner (cvt_core.py:192-240): a_ij = -int_{T_ij u T_ji} rho over the fan
 * sub-triangles next to edge ij, zero row sums.  scvt_laplacian, right after the evaluation of
 * these n points, writes the weights aligned with the context's cycles: wsym (n, 32) f64 =
 * w_ij + w_ji for the neighbour in cycle slot t, diag (n,) = row sums, and a copy of the
 * cycles themselves (nbr_out (n, 32) int32, deg_out (n,)) that the solve takes as the matrix's
 * sparsity.  The caller forms the
 * perturbed diagonal dpert (m2: 1.01 diag, a6: diag + 1e-6).  scvt_laplacian_solve solves
 * A_pert x = b for the three coordinate columns of b (n,3) by conjugate gradients with
 * fixed-order reductions until |r_c| <= tol |b_c| (the reference factors with SuperLU; an
 * indefinite matrix or no convergence -> SCVT_ERR_FACTORIZATION). */
int scvt_laplacian(scvt_ctx* ctx, int64_t n, double* wsym, double* diag, int32_t* nbr_out,
                   int32_t* deg_out);
int scvt_laplacian_solve(scvt_ctx* ctx, int64_t n, const int32_t* nbr, const int32_t* deg,
                         const double* wsym, const double* dpert, const double* b, double* x,
                         double tol, int32_t max_iter, int32_t* iters_host);
/* two_loop_direction (optimizer.py:147-167) around a general initial inverse: backward loop
 * (q = g - sum a_k y_k, newest first), caller applies h0, forward loop + negation;
 * qg_host = q.g */
int scvt_twoloop_backward(scvt_ctx* ctx, const double* g, int64_t n, double* q);
int scvt_twoloop_forward(scvt_ctx* ctx, double* q, const double* g, int64_t n, double* qg_host);

/* optimizer vector algebra -------------------------------------------------------------
 * CorrectionHistory (optimizer.py:79-114): ring of at most lbfgs_m (s, y) pairs held on
 * the device inside ctx. */
int scvt_history_clear(scvt_ctx* ctx);
int scvt_history_size(scvt_ctx* ctx, int32_t* size_host);
/* gamma = y.s / y.y of the newest pair, 1 when empty (optimizer.py:109-114); host out */
int scvt_history_gamma(scvt_ctx* ctx, double* gamma_host);
/* s = z_new - z_old, y = g_new - g_old; push unless y.s <= 1e-14 |s||y| (optimizer.py:98-104,
 * 351-353).  pushed_host = 1/0; movement_host = max |z_new - z_old| (optimizer.py:355). */
int scvt_history_push(scvt_ctx* ctx, const double* z_old, const double* z_new,
                      const double* g_old, const double* g_new, int64_t n,
                      int32_t* pushed_host, double* movement_host);
/* scvt_history_push of the pair staged by scvt_evaluate_staged(z_new -> g_new): same outputs,
 * same curvature test; SCVT_ERR_CONFIG when no pair is staged for exactly these buffers and
 * this history state (the caller then uses scvt_history_push). */
int scvt_history_commit_staged(scvt_ctx* ctx, const double* z_new, const double* g_new,
                               int64_t n, int32_t* pushed_host, double* movement_host);
/* two_loop_direction (optimizer.py:147-167): q = -H g with h0 = diag(1/lloyd_diag) blockwise
 * when inv_diag_src != NULL (LloydDiagonal, optimizer.py:127-134; the ARRAY passed is
 * lloyd_diag itself, inverted on the fly), else gamma*I (GammaIdentity, 117-124).
 * qg_host = q.g (caller raises NonDescentError when >= 0). */
int scvt_lbfgs_direction(scvt_ctx* ctx, const double* g, const double* lloyd_diag,
                         double gamma, int64_t n, double* q_out, double* qg_host);
/* Fused two_loop_direction + tangent projection (optimizer.py:147-167, 322-333) in Gram form:
 * one pass computes s_i.g, y_i.H0 g, y_i.H0 y_j, g.H0 g (y_i.s_j is kept from the pushes), a
 * one-block kernel runs the scalar recursion, one pass forms q, q3 = q - (q.z)z and the sums.
 * out_host[0] = q.g (descent test), out_host[1] = dphi0 = sum g.q3.  h0 as for
 * scvt_lbfgs_direction (lloyd_diag != NULL: LloydDiagonal, else gamma*I). */
int scvt_lbfgs_direction_tangent(scvt_ctx* ctx, const double* g, const double* lloyd_diag,
                                 double gamma, const double* z, int64_t n, double* q3_out,
                                 double* out_host);
/* q3 = q - (q.z) z rowwise (optimizer.py:322-323); dphi0_host = sum g.q3 (333) */
/* as scvt_lbfgs_direction_tangent without the host wait: the two scalars are copied to
 * pinned memory behind the kernels; scvt_direction_result waits for that copy only (the
 * caller may enqueue the first line-search trial in between) */
int scvt_lbfgs_direction_tangent_async(scvt_ctx* ctx, const double* g, const double* lloyd_diag,
                                       double gamma, const double* z, int64_t n, double* q3);
int scvt_direction_result(scvt_ctx* ctx, double* out_host);
int scvt_tangent_project(scvt_ctx* ctx, const double* q, const double* z, const double* g,
                         int64_t n, double* q3_out, double* dphi0_host);
/* v = z + alpha q3; norms = |v|; zt = v / norms (optimizer.py:325-328) */
int scvt_trial_point(scvt_ctx* ctx, const double* z, const double* q3, double alpha, int64_t n,
                     double* zt_out, double* norms_out);
/* d = sum g . (q3 / norms) (optimizer.py:330); host out */
int scvt_directional_derivative(scvt_ctx* ctx, const double* g, const double* q3,
                                const double* norms, int64_t n, double* d_host);
/* lloyd_step (optimizer.py:240-246): z = c / |c|, SCVT_ERR_CENTROID_AT_ORIGIN if |c| <= 1e-12 */
int scvt_lloyd_step(scvt_ctx* ctx, const double* first, int64_t n, double* z_out);
/* min over v[0..len) (host out) — nonpositive-diagonal test (cvt_core.py:184) */
int scvt_min(scvt_ctx* ctx, const double* v, int64_t len, double* min_host);
/* max |a - b| over len doubles (host out) — movement of the Lloyd method (optimizer.py:355) */
int scvt_max_abs_diff(scvt_ctx* ctx, const double* a, const double* b, int64_t len,
                      double* max_host);
/* y = a * x over len doubles (the -gamma g fallback, optimizer.py:321) */
int scvt_scale(scvt_ctx* ctx, double a, const double* x, int64_t len, double* y);
/* normalise rows of (n,3) in place (optimizer.py:290) */
int scvt_normalize_rows(scvt_ctx* ctx, double* z, int64_t n);

/* live CUDA-event timing of the evaluation kernels (bench roofline).  When enabled, every
 * scvt_evaluate records events around the cell-construction kernels, the quadrature kernel
 * and the whole evaluation on the context stream; read accumulates them:
 * ms_out[0..2] / counts_out[0..2] = {cells, quadrature, evaluate}. */
int scvt_profile_enable(scvt_ctx* ctx, int on);
int scvt_profile_read(scvt_ctx* ctx, double* ms_out, int64_t* counts_out, int reset);
/* cell-builder work counters accumulated while profiling is enabled:
 * out12 = {cells, candidate passes, points scanned, candidates sorted, clips, radius rounds,
 *          max 32-point sweep batches of one cell, max clips of one cell,
 *          evaluations whose previous cycles were certified and reused, cells rebuilt by
 *          reuse, certificate passes run by reuse,
 *          max points scanned by one cell | (max candidate passes of one cell << 40)} */
int scvt_profile_counters(scvt_ctx* ctx, int64_t* out12, int reset);
/* flip repair of reused cycles: {evaluations that ran it, flip rounds, flips, evaluations that
 * left candidates open and rebuilt those cells} since the last reset */
int scvt_profile_flips(scvt_ctx* ctx, int64_t* out4, int reset);
/* measured FP64 DFMA throughput of `device` in TFLOP/s (2 FLOPs per FMA): the FP64
 * roofline denominator, which MEASURED_PEAKS.json does not carry */
int scvt_fp64_peak(int device, double* tflops_out);

/* launches of library kernels since the context was created (bench accounting) */
int64_t scvt_launch_count(const scvt_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* SCVT_B200_H */
