/*
 * mdsx.h — C-ABI of the B200-native big-data MDS hot path (libmdsx.so).
 *
 * Every entry point takes caller-owned DEVICE pointers (row-major, explicit
 * leading dimension), plain sizes and a cudaStream_t passed as void*; it
 * enqueues work on that stream and returns an mdsx_status.  Arrays marked
 * "host" are read on the host before the call returns.  Nothing here ever
 * frees caller memory; each handle owns its own device workspace.  Calls on
 * one handle are serialised (a lock) and stream-ordered against each other (the
 * stream of a call waits for the previous call's last work), so a handle may
 * be shared by several host threads and streams.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/scalemds):
 *   mdsx_classical_pieces   <- classical_mds_from_data via _piece_mds
 *                              (classical.py:153-160, algorithms.py:115-119),
 *                              batched over every piece of a plan
 *   mdsx_classical_delta    <- classical_mds (classical.py:109-150)
 *   mdsx_sqdist_self        <- euclidean_distance_matrix (linalg.py:61-82)
 *   mdsx_sqdist_cross       <- cross_squared_distances (linalg.py:85-104)
 *   mdsx_double_center      <- double_center (linalg.py:107-121)
 *   mdsx_sym_eigvals        <- the full spectrum of symmetric_eigen / eigvalsh
 *                              (linalg.py:149-169) used by classical_mds
 *   mdsx_gower_context      <- gower_context (algorithms.py:193-217)
 *   mdsx_gower_interpolate  <- gower_interpolate (algorithms.py:220-242)
 *   mdsx_gower_tiles, mdsx_landmark_overwrite, mdsx_interp_recenter
 *                           <- interpolation_mds's interpolate / landmark overwrite /
 *                              _recentered steps (algorithms.py:262-274), for rows
 *                              spread over ranks
 *   mdsx_procrustes_fit     <- fit_procrustes (procrustes.py:53-78), batched
 *   mdsx_procrustes_apply   <- apply_procrustes (procrustes.py:99-105), batched
 *   mdsx_divide_conquer     <- divide_and_conquer_mds (algorithms.py:128-172)
 *   mdsx_interpolation      <- interpolation_mds (algorithms.py:245-274)
 *   mdsx_recenter           <- _recentered (algorithms.py:122-125)
 *   mdsx_scatter_rows       <- points[root.indices] = block (algorithms.py:341-342)
 *   mdsx_fast_finish        <- the root's child alignment (algorithms.py:310-311) +
 *                              points[root.indices] = block (:341-342) + _recentered
 *                              (:122-125) in one pass
 *   mdsx_fast_mds           <- fast_mds (algorithms.py:285-348) for plans with form-0
 *                              leaves (the BASELINE shapes), one call
 *   mdsx_divide_conquer_sharded, mdsx_fast_mds_sharded
 *                           <- the same for one rank's share of the pieces, the column
 *                              mean gathered over the ranks inside the call
 * Other fast_mds plans (algorithms.py:323-348) are composed from mdsx_classical_pieces,
 * mdsx_procrustes_fit/apply and mdsx_fast_finish (or mdsx_scatter_rows +
 * mdsx_recenter) by the host.
 */
#ifndef MDSX_H
#define MDSX_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the host shim maps them onto scalemds.errors (errors.py:4-41). */
enum mdsx_status {
  MDSX_OK = 0,
  MDSX_PARAM = 1,          /* ParamError */
  MDSX_SHAPE = 2,          /* ShapeError */
  MDSX_INVALID_INPUT = 3,  /* InvalidInputError */
  MDSX_NUMERICAL = 4,      /* NumericalError */
  MDSX_DEGENERATE = 5,     /* DegenerateRankError */
  MDSX_CUDA = 6,           /* CUDA runtime failure */
  MDSX_UNSUPPORTED = 7,    /* shape outside what this build handles */
  MDSX_FORMAT = 8          /* FormatError: a file does not match its declared format */
};

/* Element type of data matrices: the reference coerces to float64
 * (linalg.py:30); float32 storage is read and widened to float64 in-kernel. */
enum mdsx_dtype { MDSX_F64 = 0, MDSX_F32 = 1 };

/* Per-piece status record written by the batched classical-MDS kernels. */
typedef struct mdsx_piece_status {
  int32_t code;        /* mdsx_status */
  int32_t index;       /* DegenerateRank: 1-based failing eigenvalue index */
  double value;        /* DegenerateRank: the failing eigenvalue (snapped) */
} mdsx_piece_status;

typedef struct mdsx_handle mdsx_handle;

int mdsx_create(int device, mdsx_handle** out);
void mdsx_destroy(mdsx_handle* h);
const char* mdsx_last_error(const mdsx_handle* h);
/* Number of kernels this handle has launched since creation. */
int64_t mdsx_launch_count(const mdsx_handle* h);
int mdsx_version(void);
/* Per-kernel CUDA-event timing of this handle's launches (off by default).
 * mdsx_timing_report synchronises on the recorded events and returns the
 * length of the report "<kernel> <total_ms> <count> <work>\n"... (work: executed
 * flops credited by the launcher, 0 when not counted); with a buffer
 * (cap bytes, NUL-terminated) it also copies the report and resets it. */
int mdsx_timing_enable(mdsx_handle* h, int on);
int64_t mdsx_timing_report(mdsx_handle* h, char* buf, int64_t cap);
/* The launches timed since the last report, one line each: "kernel start_ms
 * end_ms" relative to the first launch's start event (a timeline of the piece
 * pipeline's two streams); does not consume them.  Returns the text length. */
int64_t mdsx_timing_trace(mdsx_handle* h, char* buf, int64_t cap);

/* Copy `bytes` from a PAGEABLE host array (e.g. the numpy array the reference
 * API receives, linalg.py:28-38) to device memory, staged through page-locked
 * chunk buffers by `threads` host threads (0 = half the cores) so host
 * memcpy and PCIe DMA overlap.  Returns once the source has been read; the
 * device writes are ordered on `stream` like cudaMemcpyAsync. */
int mdsx_h2d(mdsx_handle* h, void* dst, const void* src, int64_t bytes, int32_t threads,
             void* stream);

/* ---- column compaction of wide inputs ---------------------------------------
 * Columns that are zero in every row contribute exactly zero to every Gram,
 * eigenvector, mean, point and Gower term, so the algorithms may run on the
 * matrix of the active columns (same configuration).  mdsx_active_columns:
 * one pass over the n x p matrix (device), the indices of the columns with a
 * nonzero (or non-finite) entry in ascending order written to the HOST array
 * cols (p entries), their number to *count; synchronous.
 * mdsx_gather_columns: out (n x ldo, device, same dtype) = the columns
 * cols[0..pa) (device array) of data, zero columns pa..ldo-1. */
int mdsx_active_columns(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n,
                        int32_t p, int32_t* cols, int32_t* count, void* stream);
int mdsx_gather_columns(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n,
                        const int32_t* cols, int32_t pa, int64_t ldo, void* out, void* stream);

/* ---- dense primitives (function-level seams) ---------------------------- */
/* out (m x m, ldo) = squared distances between rows of x (m x p, ld);
 * symmetrised, clamped at 0, exact-zero diagonal. */
int mdsx_sqdist_self(mdsx_handle* h, const void* x, int dtype, int64_t ld,
                     int64_t m, int32_t p, double* out, int64_t ldo, void* stream);
/* out (ma x mb, ldo) = squared distances rows(a) x rows(b), clamped at 0. */
int mdsx_sqdist_cross(mdsx_handle* h, const void* a, int64_t lda, int64_t ma,
                      const void* b, int64_t ldb, int64_t mb, int dtype, int32_t p,
                      double* out, int64_t ldo, void* stream);
/* q (m x m) = -1/2 (d - rowmean_i - rowmean_j + grandmean), symmetrised. */
int mdsx_double_center(mdsx_handle* h, const double* delta, int64_t m, double* q,
                       void* stream);

/* ---- batched classical MDS of the pieces of a plan ---------------------- */
/* Piece j is rows row_idx[piece_off[j] .. piece_off[j+1]) of data (n x p).
 * points  (total x r): configuration of every piece, piece order, rows in
 *                      row_idx order, canonical column signs (linalg.py:139-146)
 * estimates (npieces x r): lambda_i / m_j   gof (npieces x 2): G1, G2
 * status (npieces): per-piece mdsx_piece_status.
 * piece_off is a HOST array of npieces+1 offsets. */
int mdsx_classical_pieces(mdsx_handle* h, const void* data, int dtype, int64_t ld,
                          int32_t p, const int64_t* row_idx, const int64_t* piece_off,
                          int32_t npieces, int32_t r, double* points, double* estimates,
                          double* gof, mdsx_piece_status* status, void* stream);

/* Every eigenvalue (ascending, n doubles into w) of the symmetric n x n
 * device matrix a (row-major, full storage; a is not modified): Householder
 * tridiagonalisation + bisection.  Replaces the full-spectrum eigvalsh /
 * dsyevd that classical_mds needs for G1/G2 and the DegenerateRank rule
 * (classical.py:88-150, linalg.py:149-169) beyond the in-kernel Jacobi size. */
int mdsx_sym_eigvals(mdsx_handle* h, const double* a, int64_t n, double* w, void* stream);

/* Validity flags of a squared-distance matrix (linalg.py:41-58), OR-ed into
 * *flags (device int32, caller-zeroed): 1 non-finite, 2 asymmetric,
 * 4 nonzero diagonal, 8 negative entries (tolerance 1e-9 max(|d|max, 1)). */
int mdsx_delta_check(mdsx_handle* h, const double* delta, int64_t m, int32_t* flags, void* stream);

/* Classical MDS of a precomputed squared-distance matrix (m x m). */
int mdsx_classical_delta(mdsx_handle* h, const double* delta, int64_t m, int32_t r,
                         double* points, double* estimates, double* gof,
                         mdsx_piece_status* status, void* stream);

/* ---- Gower interpolation ------------------------------------------------ */
/* Context packed as doubles: [mean(p) | M(p x r) | v(r) | S(r x r) | q(l)],
 * size mdsx_gower_context_size(l, p, r).  base rows are data[base_idx[j]]
 * (base_idx may be NULL: rows 0..l-1), base_config is (l x r). cond (1 double,
 * device) receives the covariance condition estimate; flag (1 int32, device)
 * 0 ok, 1 condition > 1e12, 2 covariance not positive definite. */
int64_t mdsx_gower_context_size(int64_t l, int32_t p, int32_t r);
int mdsx_gower_context(mdsx_handle* h, const void* data, int dtype, int64_t ld, int32_t p,
                       const int64_t* base_idx, int64_t l, const double* base_config,
                       int32_t r, double* ctx, double* cond, int32_t* flag, void* stream);
/* out (m x r, ldo) = Gower coordinates of rows data[0..m) in the base frame;
 * *nonfinite (device int32, caller-zeroed) is set if an input is not finite. */
/* flags: MDSX_GOWER_CENTRED = the context's base configuration has zero
 * column means (true for interpolation_mds's landmark MDS): v ~ 0, so the
 * squared norms of fp32 rows may be formed on the fp32 pipe. */
#define MDSX_GOWER_CENTRED 1
int mdsx_gower_interpolate(mdsx_handle* h, const double* ctx, int64_t l, int32_t p, int32_t r,
                           const void* rows, int dtype, int64_t ld, int64_t m,
                           double* out, int64_t ldo, int32_t* nonfinite, int32_t flags,
                           void* stream);
/* The three steps of interpolation_mds after the landmark context
 * (algorithms.py:262-274), for callers that spread the rows over ranks
 * (distributed.ShardedInterpolation).  mdsx_interpolation runs the same steps
 * in one call with per-CTA column sums; the tile sums here make the result
 * independent of how the rows are spread (bitwise, for any number of ranks):
 *  - mdsx_gower_tiles: as mdsx_gower_interpolate for dense (ld = p), 16-byte
 *    aligned rows with packed output, plus tile_sums[t * r + c] = column sums of
 *    out over tile t (mdsx_gower_tile_rows rows per tile; MDSX_UNSUPPORTED for
 *    other layouts).  A rank's rows must start on a tile boundary for the
 *    tiles to be the same as the single-call's.
 *  - mdsx_landmark_overwrite: out[pos[i]] = base[s], corr[s] = base[s] - old,
 *    s = sel[i] (sel NULL: i), for the nl landmarks held here; corr (l x r,
 *    sample order) is zeroed first, so summing the ranks' corr is exact.
 *  - mdsx_interp_recenter: out[0..m) -= (sum of tile_sums (all ranks' tiles in
 *    row order) + sum of corr) / n_total, in a fixed order. */
int32_t mdsx_gower_tile_rows(mdsx_handle* h, int dtype, int32_t p, int32_t r);
int mdsx_gower_tiles(mdsx_handle* h, const double* ctx, int64_t l, int32_t p, int32_t r,
                     const void* rows, int dtype, int64_t m, double* out, double* tile_sums,
                     int32_t* nonfinite, int32_t flags, void* stream);
int mdsx_landmark_overwrite(mdsx_handle* h, const double* base, int64_t l, int32_t r,
                            const int64_t* sel, const int64_t* pos, int64_t nl, double* out,
                            double* corr, void* stream);
int mdsx_interp_recenter(mdsx_handle* h, const double* tile_sums, int64_t ntiles,
                         const double* corr, int64_t l, int32_t r, int64_t n_total, double* out,
                         int64_t m, void* stream);

/* ---- Procrustes ----------------------------------------------------------- */
/* Job j aligns src rows src_rows[job_off[j]..job_off[j+1]) of src (ld = r)
 * onto tgt rows tgt_rows[...] of tgt.  job_off is a HOST array.
 * rot (njobs x r x r), trans (njobs x r), loss (njobs), degenerate (njobs). */
int mdsx_procrustes_fit(mdsx_handle* h, const double* tgt, const int64_t* tgt_rows,
                        const double* src, const int64_t* src_rows, const int64_t* job_off,
                        int32_t njobs, int32_t r, double* rot, double* trans, double* loss,
                        int32_t* degenerate, void* stream);
/* In place: buf[start_j + i] = buf[start_j + i] @ rot_j + trans_j for
 * i < len_j.  start/len are DEVICE arrays of njobs int64. */
int mdsx_procrustes_apply(mdsx_handle* h, double* buf, int32_t r, const int64_t* start,
                          const int64_t* len, int32_t njobs, int64_t max_len,
                          const double* rot, const double* trans, void* stream);

/* ---- stitching / finishing ------------------------------------------------ */
/* out[idx[i]] = src[i] (rows of r doubles), i < n. */
int mdsx_scatter_rows(mdsx_handle* h, const double* src, const int64_t* idx, int64_t n,
                      int32_t r, double* out, void* stream);
/* points (n x r) -= column means (fixed-order, deterministic reduction). */
int mdsx_recenter(mdsx_handle* h, double* points, int64_t n, int32_t r, void* stream);
/* fast_mds (algorithms.py:285-348) in one call for plans whose leaves are
 * all form 0 (more rows than features) with p <= 128, r <= 16 and 16-byte
 * aligned rows: classical MDS of every leaf and alignment set (eigenpairs;
 * points only for the alignment sets and the tracked rows), the Procrustes
 * fits level by level (deepest first), and ONE pass over the leaf rows
 * writing out[out_idx[i]] = (x - mu_leaf) U_leaf T_tot + t_tot (- the column
 * mean when recenter != 0, algorithms.py:122-125).  The plan arrays come
 * from the host flattener (paper_2007_11919_b200.plans.fast_route). */
typedef struct mdsx_fast_plan {
  int32_t npieces, n_leaves, nlevels;
  const int64_t* piece_off;   /* host, npieces + 1: leaves (DFS order) then alignment sets */
  const int64_t* row_idx;     /* device, piece_off[npieces] data rows */
  const int64_t* out_idx;     /* device, piece_off[n_leaves]: output row of every leaf row */
  int64_t ntracked;
  const int64_t* trk_row;     /* device: data row of every tracked row */
  const int32_t* trk_leaf;    /* device: its leaf */
  const int32_t* level_njobs; /* host, nlevels (deepest first) */
  const int64_t* job_off;     /* host, per level njobs + 1 entries, concatenated */
  const int64_t* job_src;     /* device: tracked-row ids of each job's samples, concatenated */
  const int64_t* job_tgt;     /* device: alignment-set point rows (targets), concatenated */
  const int32_t* trk_job;     /* device, nlevels x ntracked: job at that level or -1 */
  const int32_t* leaf_job;    /* device, nlevels x n_leaves: job at that level or -1 */
} mdsx_fast_plan;
int mdsx_fast_mds(mdsx_handle* h, const void* data, int dtype, int64_t ld, int32_t p,
                  const mdsx_fast_plan* plan, int32_t r, int64_t n_out, int32_t recenter,
                  double* out, double* estimates, double* gof, mdsx_piece_status* status,
                  void* stream);

/* out[order[i]] = P[i] @ rot_j + trans_j - mean for the rows i of job j
 * (HOST job_off: njobs+1 offsets covering 0..n), mean = the column mean of
 * the result (from per-job sums pushed through each fit; fixed order). */
int mdsx_fast_finish(mdsx_handle* h, const double* P, int32_t r, const int64_t* job_off,
                     int32_t njobs, const double* rot, const double* trans,
                     const int64_t* order, int64_t n, double* out, void* stream);

/* ---- whole algorithms ------------------------------------------------------ */
/* divide_and_conquer_mds with an explicit plan (partition.py:184-214 layout:
 * every subset = c connecting rows then own rows).  out (n x r) in original
 * row order, re-centred (callers handle the n <= l passthrough with
 * mdsx_classical_pieces, as algorithms.py:142-143 does).  Per-piece estimates/gof/status as in
 * mdsx_classical_pieces; the host aggregates them in plan order. */
int mdsx_divide_conquer(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n,
                        int32_t p, const int64_t* row_idx, const int64_t* piece_off,
                        int32_t npieces, int32_t c, int32_t r, double* out,
                        double* estimates, double* gof, mdsx_piece_status* status,
                        void* stream);
/* mdsx_divide_conquer with flags: MDSX_NO_RECENTER leaves the column means in
 * place (a sharded run re-centres with globally reduced sums).  The anchor is
 * piece 0 of the given (sub-)plan. */
#define MDSX_NO_RECENTER 1
int mdsx_divide_conquer_ex(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n,
                           int32_t p, const int64_t* row_idx, const int64_t* piece_off,
                           int32_t npieces, int32_t c, int32_t r, double* out,
                           double* estimates, double* gof, mdsx_piece_status* status,
                           int32_t flags, void* stream);
/* One rank's share of a sharded divide_and_conquer_mds: the subsets of this
 * call (piece 0 = the anchor, recomputed by every rank) are solved, fitted and
 * composed as in mdsx_divide_conquer; their column-sum contributions
 * (npieces x r) are copied to contrib_local and gather(ctx, stream) is called
 * on the host thread: it must enqueue on `stream` the collective that fills
 * contrib_global (npieces_total x r) with every subset's contribution in
 * global subset order.  The mean over n_total rows then follows in the same
 * fixed order on every rank (results independent of the number of ranks and
 * equal to the unsharded call), and the output pass writes this call's rows
 * re-centred.  MDSX_UNSUPPORTED unless the fused output route applies. */
typedef int (*mdsx_gather_fn)(void* ctx, void* stream);
int mdsx_divide_conquer_sharded(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n,
                                int32_t p, const int64_t* row_idx, const int64_t* piece_off,
                                int32_t npieces, int32_t c, int32_t r, double* out,
                                double* estimates, double* gof, mdsx_piece_status* status,
                                int64_t n_total, int32_t npieces_total, double* contrib_local,
                                double* contrib_global, mdsx_gather_fn gather, void* ctx,
                                void* stream);
/* mdsx_fast_mds for one rank's share of a sharded fast MDS (distributed.py):
 * the plan holds the rank's level-1 subtrees (plus the root's alignment set);
 * its n_leaves leaf contributions go to contrib_local, gather() fills
 * contrib_global (nleaves_total x r, global leaf order) on the call's stream,
 * and the output pass writes the rank's rows (leaf order) re-centred by the
 * mean over n_total rows -- bitwise the unsharded call's rows. */
int mdsx_fast_mds_sharded(mdsx_handle* h, const void* data, int dtype, int64_t ld, int32_t p,
                          const mdsx_fast_plan* plan, int32_t r, int64_t n_out, double* out,
                          double* estimates, double* gof, mdsx_piece_status* status,
                          int64_t n_total, int32_t nleaves_total, double* contrib_local,
                          double* contrib_global, mdsx_gather_fn gather, void* ctx, void* stream);
/* Column sums of points[idx[seg_off[j] .. seg_off[j+1])] per segment j
 * (sums: nseg x r, device; seg_off: device).  Fixed-order reductions, so a
 * sharded run that sums the same segments in the same order is independent
 * of the number of ranks. */
/* idx == NULL: the rows are the offsets themselves (contiguous segments). */
int mdsx_segment_colsums(mdsx_handle* h, const double* points, const int64_t* idx,
                         const int64_t* seg_off, int32_t nseg, int32_t r, double* sums,
                         void* stream);
/* points[idx[i]] -= shift (r doubles, device), i < n; idx == NULL: rows 0..n-1. */
int mdsx_shift_rows(mdsx_handle* h, double* points, const int64_t* idx, int64_t n, int32_t r,
                    const double* shift, void* stream);

/* interpolation_mds with an explicit landmark sample (sample_idx, device, l).
 * out (n x r) in original row order, re-centred; estimates (r), gof (2),
 * status (1) describe the landmark MDS; cond (1) the covariance condition;
 * flags (2 int32, device, caller-zeroed): [0] context flag as in
 * mdsx_gower_context, [1] non-finite input seen. */
int mdsx_interpolation(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n,
                       int32_t p, const int64_t* sample_idx, int64_t l, int32_t r,
                       double* out, double* estimates, double* gof,
                       mdsx_piece_status* status, double* cond, int32_t* flags,
                       void* stream);

/* ---- harness metric (simulation.py:83-108) --------------------------------
 * aligned_correlations: Procrustes-align the configuration `points` (n x r,
 * f64, device) onto `dominant` (n x r, dtype, row stride ld, device: e.g. the
 * first r columns of the data matrix) and return the per-column Pearson
 * correlations corr (r, device).  One pass over the rows (shifted column sums
 * and the 2r x 2r Gram, fixed-order reductions), then the rotation from the
 * centred cross-product by the warp SVD of the Procrustes kernels; the aligned
 * matrix is never formed.  rotation (r x r, device) may be NULL; zero_var
 * (1 int32, device) is set to 1 when a column has zero variance (the caller
 * raises MetricError).  1 <= r <= 16. */
int mdsx_aligned_correlations(mdsx_handle* h, const double* points, int64_t n, int32_t r,
                              const void* dominant, int32_t dtype, int64_t ld, double* corr,
                              double* rotation, int32_t* zero_var, void* stream);

/* ---- host planner ------------------------------------------------------ */
/* In-place random permutation of a[0..n) bit-identical to numpy's
 * Generator.permutation on a PCG64 bit generator whose state is passed as
 * state = {state_hi, state_lo, inc_hi, inc_lo}, has_uint32, uinteger and
 * advanced in place (the permutation draws of partition.py:204-213, 225-231
 * and 258-264).  Host memory only; no device. */
int mdsx_plan_permute(int64_t* a, int64_t n, uint64_t* state, int32_t* has_uint32,
                      uint32_t* uinteger);
/* Generator.choice(pops[i], min(s, pops[i]), replace=False) for i = 0..npop-1
 * in sequence on the same PCG64 state (the sampling positions of
 * partition.py:258-264), bit-identical to numpy; out[i * s ..] receives the
 * picks (unsorted).  MDSX_UNSUPPORTED when a population needs a path numpy
 * takes only for k == pop. */
int mdsx_plan_choices(const int64_t* pops, int32_t npop, int32_t s, int64_t* out,
                      uint64_t* state, int32_t* has_uint32, uint32_t* uinteger);

/* ---- file ingestion (replaces dataio.py:42-58, 68-82, 102-130) ----------
 * Host-side parsing; no device is needed except for mdsx_idx_load_images.
 * On failure `msg` (msg_len bytes, NUL-terminated) carries the reference's
 * FormatError text. */

/* IDX header check: expect_kind 3 = images (magic 0x00000803, dims count,
 * height, width; dataio.py:42-58) or 1 = labels (magic 0x00000801, dim count;
 * dataio.py:68-82).  Validates the magic and the payload size against the file
 * size.  height/width are set to 1 for labels. */
int mdsx_idx_probe(const char* path, int32_t expect_kind, int64_t* count, int32_t* height,
                   int32_t* width, char* msg, int64_t msg_len);

/* Stream an IDX image payload straight into a device matrix `out`
 * (count x height*width, row-major, dtype MDSX_F64 / MDSX_F32), each element
 * scale * pixel: the file is read in chunks into two pinned buffers, the
 * unsigned bytes cross PCIe (1/8 of the float64 volume) and a kernel widens
 * them on the device; reads of chunk i+1 overlap the copy and kernel of chunk i.
 * Synchronises `stream` before returning (the pinned buffers are released). */
int mdsx_idx_load_images(mdsx_handle* h, const char* path, void* out, int dtype, double scale,
                         void* stream);

/* Numeric CSV (dataio.py:102-130), two calls: with out == NULL it counts the
 * data rows and the fields of the first data row (rows, cols); with out (rows x
 * cols doubles, host) it parses every field (correctly rounded, Python float()
 * syntax: surrounding whitespace and double quotes stripped, inf/nan accepted,
 * no hexadecimal) with `threads` host threads and reports the FIRST bad line in
 * file order: "ragged row at line N: expected W fields, got K" / "invalid
 * number at line N: ..." / "no data rows" (MDSX_FORMAT). */
int mdsx_csv_read(const char* path, int32_t has_header, int32_t threads, double* out,
                  int64_t* rows, int64_t* cols, char* msg, int64_t msg_len);

#ifdef __cplusplus
}
#endif
#endif /* MDSX_H */
