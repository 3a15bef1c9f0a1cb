// C-ABI entry points and the handle runtime (workspace, staging, errors).
#include "mdsx_common.cuh"

#include <cstdlib>

#include <algorithm>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

namespace mdsx {
int launch_procrustes_fit(mdsx_handle* h, const double* tgt, const int64_t* tgt_rows,
                          const double* src, const int64_t* src_rows, const int64_t* job_off_dev,
                          int njobs, int r, double* rot, double* trans, double* loss,
                          int32_t* degenerate, cudaStream_t st, bool redo_only = false);
bool dc_fit_ok(int r, int c, int p);
int launch_dc_fit(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                  const int64_t* row_idx, const PieceDesc* pd, int npieces, int r, int c,
                  const double* mu, const double* U, double* Pc, double* rot, double* trans,
                  double* loss, int32_t* degen, double* Uc, double* tvec, double* contrib,
                  int32_t* pending, cudaStream_t st);
int launch_apply(mdsx_handle* h, double* buf, int r, const int64_t* start, const int64_t* len,
                 int njobs, int64_t max_len, const double* rot, const double* trans,
                 cudaStream_t st);
int launch_dc_stitch(mdsx_handle* h, const double* P, const int64_t* row_idx, const int64_t* off,
                     int npieces, int64_t max_m, int c, int r, const double* rot,
                     const double* trans, double* out, cudaStream_t st, int64_t n_recenter,
                     double* ws, int first_identity = 1);
size_t dc_stitch_ws_bytes(int npieces, int r, int64_t max_m);
int launch_scatter(mdsx_handle* h, const double* src, const int64_t* idx, int64_t n, int r,
                   double* out, cudaStream_t st);
int launch_seg_colsum(mdsx_handle* h, const double* X, const int64_t* idx, const int64_t* off,
                      int nseg, int r, double* sums, cudaStream_t st);
int launch_shift_rows(mdsx_handle* h, double* X, const int64_t* idx, int64_t n, int r,
                      const double* shift, cudaStream_t st);
int corr_ws_doubles(int64_t n, int r, int num_sms);
int launch_aligned_corr(mdsx_handle* h, const double* X, int64_t n, int r, const void* D,
                        int dtype, int64_t ld, double* part, double* corr, double* rot,
                        int32_t* zero_var, cudaStream_t st);
size_t recenter_ws_bytes(int r);
int launch_recenter(mdsx_handle* h, double* X, int64_t n, int r, double* part, cudaStream_t st);
int launch_subtract_mean(mdsx_handle* h, double* X, int64_t n, int r, const double* part,
                         int nparts, const double* corr, cudaStream_t st, int64_t ndiv = 0);
int launch_landmark_overwrite(mdsx_handle* h, const double* base, const int64_t* idx, int64_t l,
                              int r, double* out, double* corr, cudaStream_t st);
int launch_landmark_corr(mdsx_handle* h, const double* base, const int64_t* sel,
                         const int64_t* pos, int64_t nl, int r, double* out, double* corr,
                         cudaStream_t st);
size_t fold_ws_bytes(int64_t na, int64_t nb, int r);
int launch_fold_sums(mdsx_handle* h, const double* A, int64_t na, const double* B, int64_t nb,
                     int r, double* ws, double** total, cudaStream_t st);
int gower_tile_rows(mdsx_handle* h, int dtype, int p, int r);
int launch_gower_bulk(mdsx_handle* h, const void* X, int dtype, int64_t m, int p, int r,
                      const double* mean, const double* M, const double* v, double* out,
                      double* colpart, int32_t* nonfinite, int* nparts, cudaStream_t st,
                      bool norm32 = false, bool tiles = false);
int launch_gower_context(mdsx_handle* h, const void* X, int dtype, int64_t ld, int p,
                         const int64_t* idx, int64_t l, const double* X1, int r, double* mean,
                         double* M, double* v, double* S, double* q, double* cond, int32_t* flag,
                         cudaStream_t st);
int launch_gower_affine(mdsx_handle* h, const void* X, int dtype, int64_t ld, int64_t m, int p,
                        int r, const double* mean, const double* M, const double* v, double* out,
                        int64_t ldo, int32_t* nonfinite, cudaStream_t st);
int launch_sqdist(mdsx_handle* h, const void* A, int64_t lda, int64_t ma, const void* B,
                  int64_t ldb, int64_t mb, int dtype, int p, double* na, double* nb, double* out,
                  int64_t ldo, int self, cudaStream_t st);
int launch_double_center(mdsx_handle* h, const double* D, int64_t m, double* mu, double* g,
                         double* Q, cudaStream_t st);
int launch_delta_check(mdsx_handle* h, const double* D, int64_t m, unsigned long long* mx,
                       int32_t* flags, cudaStream_t st);
int lanczos_kmax();
int lanczos_rmax();
size_t lanczos_smem_bytes(int kmax);
int launch_lanczos_smem(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r,
                        const double* A, double* U, double* lam, double* estimates, double* gof,
                        mdsx_piece_status* status, int full_basis, int only_flagged,
                        cudaStream_t st, const PtsEpi* epi = nullptr);
bool gram_piece_ok(const void* data, int dtype, int64_t ld, int p);
int launch_gram_piece(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                      const int64_t* row_idx, const PieceDesc* pd, int npieces, double* A,
                      double* mu, mdsx_piece_status* status, cudaStream_t st);
int launch_gram_combine(mdsx_handle* h, const PieceDesc* pd, const int4* rng, int npieces,
                        const PieceDesc* pd_split, const double* A_split, const double* mu_split,
                        const mdsx_piece_status* st_split, int p, double* A, double* mu,
                        mdsx_piece_status* status, cudaStream_t st);
int launch_gram_dmma(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                     const int64_t* row_idx, const PieceDesc* pd, const int4* tiles, int ntiles,
                     double* A, double* mu, mdsx_piece_status* status, cudaStream_t st);
int launch_jacobi_fallback(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r,
                           double* A, double* U, double* lam, double* estimates, double* gof,
                           mdsx_piece_status* status, cudaStream_t st);
size_t bk_ws_bytes(const std::vector<PieceDesc>& big);
int run_big_pieces(mdsx_handle* h, const std::vector<PieceDesc>& big, const double* A, int r,
                   double* Uout, double* lam_out, double* estimates, double* gof,
                   mdsx_piece_status* status, cudaStream_t st,
                   int (*put)(mdsx_handle*, void*, const void*, size_t, cudaStream_t));

// last error message of the calling thread (calls from several threads on one
// handle each read their own message)
static thread_local std::string t_last_error;
bool dc_out_route_ok(const void* data, int dtype, int64_t ld, int p, int r, int c);
size_t dc_out_ws_doubles(int npieces, int p, int r, int c, int64_t m0);
int launch_dc_points(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                     const int64_t* row_idx, const PieceDesc* pd, int npieces, int r, int c,
                     int64_t m0, const double* mu, double* U, double* Pc, double* Pa,
                     cudaStream_t st);
int launch_dc_conn(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                   const int64_t* row_idx, const PieceDesc* pd, int pbase, int count, int r, int c,
                   const double* mu, const double* U, double* Pc, cudaStream_t st);
int launch_dc_compose(mdsx_handle* h, const PieceDesc* pd, int pbase, int count, int p, int r, int c,
                      const double* U, const double* rot, const double* trans, const double* Pc,
                      double* Uc, double* tvec, double* contrib, cudaStream_t st,
                      const int32_t* pending = nullptr);
int launch_piece_out(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                     const int64_t* row_idx, const int64_t* out_idx, const PieceDesc* pd,
                     int npieces, int64_t max_m, int r, int c0, const double* mu, const double* Uc,
                     const double* tvec, const double* mean, double* out, cudaStream_t st);
int launch_dc_mean(mdsx_handle* h, const double* contrib, int npieces, int r, int64_t n,
                   double* mean, cudaStream_t st);
int launch_dc_recentre(mdsx_handle* h, const double* contrib, int npieces, int r, int64_t n,
                       double* mean, double* out, cudaStream_t st);
int launch_trk_points(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                      const int64_t* trk_row, const int32_t* trk_leaf, int64_t ntrk,
                      const PieceDesc* pd, int r, const double* mu, const double* U, double* P,
                      cudaStream_t st);
int launch_trk_apply(mdsx_handle* h, double* P, const int32_t* job, int64_t ntrk, int r,
                     const double* rot, const double* trans, cudaStream_t st);
int launch_fast_out(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                    const int64_t* row_idx, const int64_t* out_idx, const PieceDesc* pd, int nleaves,
                    int64_t max_m, int nlev, const int32_t* leaf_job, const int64_t* lev_jbase,
                    int r, const double* mu, const double* U, const double* rot, const double* trans,
                    double* Uc, double* tvec, double* contrib, double* mean, int64_t n_recenter,
                    double* out, cudaStream_t st, const ContribGather* shard = nullptr);
size_t points_ws_bytes(int npieces, int64_t max_m, int r);
size_t eigvals_ws_doubles(int64_t n);
int launch_sym_eigvals(mdsx_handle* h, const double* A, int64_t n, double* w, double* ws,
                       cudaStream_t st);

int fail(mdsx_handle* h, int code, const std::string& msg) {
  (void)h;
  t_last_error = msg;
  return code;
}

int cuda_check(mdsx_handle* h, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return MDSX_OK;
  return fail(h, MDSX_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void ws_reset(mdsx_handle* h) { h->ws_top = 0; }

cudaEvent_t pooled_event(mdsx_handle* h) {
  if (!h->event_pool.empty()) {
    cudaEvent_t e = h->event_pool.back();
    h->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Grow the workspace to hold `bytes` for this call (device sync on growth).
int ws_reserve(mdsx_handle* h, size_t bytes) {
  h->ws_top = 0;
  if (bytes <= h->ws_size) return MDSX_OK;
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cuda_check(h, e, "workspace sync");
  if (h->ws) cudaFree(h->ws);
  h->ws = nullptr;
  h->ws_size = 0;
  size_t want = std::max(bytes, (size_t)64 << 20);
  e = cudaMalloc(&h->ws, want);
  if (e != cudaSuccess) return cuda_check(h, e, "workspace cudaMalloc");
  h->ws_size = want;
  return MDSX_OK;
}

void* ws_alloc(mdsx_handle* h, size_t bytes, cudaStream_t) {
  const size_t b = align_up(bytes ? bytes : 1);
  if (h->ws_top + b > h->ws_size) {
    fail(h, MDSX_CUDA, "workspace overflow (internal sizing error)");
    return nullptr;
  }
  void* p = h->ws + h->ws_top;
  h->ws_top += b;
  return p;
}

// Small host->device uploads go through a pinned buffer; before reusing it we
// wait for the previous batch of copies (event) so the source stays valid.
struct Stager {
  mdsx_handle* h;
  cudaStream_t st;
  size_t top = 0;
  Stager(mdsx_handle* hh, cudaStream_t s) : h(hh), st(s) {}
  int begin(size_t total) {
    if (h->pinned_free) cudaEventSynchronize(h->pinned_free);
    total = align_up(total) + 4096;
    if (total > h->pinned_size) {
      if (h->pinned) cudaFreeHost(h->pinned);
      h->pinned = nullptr;
      h->pinned_size = 0;
      cudaError_t e = cudaMallocHost(&h->pinned, std::max(total, (size_t)1 << 20));
      if (e != cudaSuccess) return cuda_check(h, e, "cudaMallocHost");
      h->pinned_size = std::max(total, (size_t)1 << 20);
    }
    top = 0;
    return MDSX_OK;
  }
  int put(void* dst, const void* src, size_t bytes) {
    if (bytes == 0) return MDSX_OK;
    std::memcpy(h->pinned + top, src, bytes);
    cudaError_t e = cudaMemcpyAsync(dst, h->pinned + top, bytes, cudaMemcpyHostToDevice, st);
    top += align_up(bytes);
    return cuda_check(h, e, "cudaMemcpyAsync(H2D descriptors)");
  }
  int end() {
    if (!h->pinned_free) cudaEventCreateWithFlags(&h->pinned_free, cudaEventDisableTiming);
    return cuda_check(h, cudaEventRecord(h->pinned_free, st), "cudaEventRecord");
  }
};

// One-shot staged upload (waits for the previous staged copy to finish first).
static int stage_put(mdsx_handle* h, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  Stager sg(h, st);
  int rc = sg.begin(bytes);
  if (rc) return rc;
  if ((rc = sg.put(dst, src, bytes))) return rc;
  return sg.end();
}

int upload(mdsx_handle* h, void* dst, const void* src, size_t bytes, cudaStream_t st) {
  return stage_put(h, dst, src, bytes, st);
}

// ------------------------------------------------------ classical pipeline
struct ClassicalPlan {
  std::vector<PieceDesc> pd;
  std::vector<PieceDesc> pd_jac, pd_sub, pd_big;   // K3 split: Jacobi / Lanczos / block Krylov
  std::vector<PieceDesc> pd_f1;                    // form-1 pieces (separate means pass)
  std::vector<int4> tiles1;                        // form-1 Gram tiles (tiles: form 0, DMMA)
  int kmax_jac = 0, kmax_sub = 0;
  std::vector<int4> tiles;                         // form-0 tiles of pieces not in pd_g
  std::vector<PieceDesc> pd_g;                     // form 0, k <= 104: one CTA per piece
  std::vector<int4> tiles_g;                       // ... and their tiles (unaligned-data fallback)
  std::vector<int64_t> off;
  int kmax = 0;
  int64_t total = 0;
  size_t a_doubles = 0, u_doubles = 0;
  int64_t max_m = 0;
  // few large form-0 pieces (e.g. the landmark set of interpolation): each is
  // split into row ranges whose centred Grams are combined (gram_combine)
  std::vector<PieceDesc> pd_split;                 // virtual pieces (row sub-ranges)
  std::vector<int4> split_rng;                     // real piece j: (first split, count, j, 0)
  size_t split_a_doubles = 0;
};

static int plan_classical(mdsx_handle* h, int p, const int64_t* piece_off, int npieces, int r,
                          ClassicalPlan& cp) {
  if (npieces < 1) return fail(h, MDSX_PARAM, "no pieces");
  if (r < 1 || r > MDSX_MAX_R)
    return fail(h, MDSX_PARAM, "r must satisfy 1 <= r <= " + std::to_string(MDSX_MAX_R));
  cp.pd.resize(npieces);
  cp.off.assign(piece_off, piece_off + npieces + 1);
  int64_t a_off = 0, u_off = 0;
  for (int j = 0; j < npieces; ++j) {
    const int64_t m = piece_off[j + 1] - piece_off[j];
    if (m < 2 || r > m - 1)
      return fail(h, MDSX_PARAM, "r must satisfy 1 <= r <= n-1, got r=" + std::to_string(r) +
                                     ", n=" + std::to_string(m));
    if (m > 20000) return fail(h, MDSX_PARAM, "piece exceeds the exact-size guard (20000)");
    PieceDesc d{};
    d.row_off = piece_off[j];
    d.m = (int)m;
    d.form = (p < m) ? 0 : 1;
    d.k = d.form == 0 ? p : (int)m;
    d.a_off = a_off;
    d.u_off = u_off;
    d.pt_off = piece_off[j] - piece_off[0];
    d.id = j;
    a_off += (int64_t)d.k * d.k;
    u_off += (int64_t)d.k * r;
    cp.kmax = std::max(cp.kmax, d.k);
    // full Jacobi for small k or large r; Lanczos (top-r) up to 104; block Krylov above
    if (d.k > lanczos_kmax() && !(r > 12 && d.k <= MDSX_JACOBI_KMAX)) {
      cp.pd_big.push_back(d);
    } else if (d.k <= 32 || d.k > lanczos_kmax() || r > lanczos_rmax()) {
      cp.pd_jac.push_back(d);
      cp.kmax_jac = std::max(cp.kmax_jac, d.k);
    } else {
      cp.pd_sub.push_back(d);
      cp.kmax_sub = std::max(cp.kmax_sub, d.k);
    }
    cp.max_m = std::max<int64_t>(cp.max_m, m);
    cp.pd[j] = d;
    const int T = (d.k + 63) / 64;
    const bool small0 = d.form == 0 && d.k <= 104;
    if (small0) cp.pd_g.push_back(d);
    for (int ti = 0; ti < T; ++ti)
      for (int tj = 0; tj <= ti; ++tj)
        (d.form == 1 ? cp.tiles1 : small0 ? cp.tiles_g : cp.tiles).push_back(make_int4(j, ti, tj, 0));
    if (d.form == 1) cp.pd_f1.push_back(d);
  }
  cp.total = piece_off[npieces] - piece_off[0];
  cp.a_doubles = (size_t)a_off;
  cp.u_doubles = (size_t)u_off;
  // one CTA per piece leaves most SMs idle when there are only a few pieces:
  // split each into row ranges of >= 128 rows (two 64-row stages each)
  if (!cp.pd_g.empty() && (int)cp.pd_g.size() * 4 <= h->num_sms && !getenv("MDSX_NO_GRAM_SPLIT")) {
    bool big = true;
    for (const PieceDesc& d : cp.pd_g) big = big && d.m >= 512;
    if (big) {
      int64_t a2 = 0;
      for (const PieceDesc& d : cp.pd_g) {
        const int S = std::min(std::max(1, h->num_sms / (int)cp.pd_g.size()), std::min(32, d.m / 128));
        cp.split_rng.push_back(make_int4((int)cp.pd_split.size(), S, d.id, 0));
        for (int q = 0; q < S; ++q) {
          const int r0 = (int)((int64_t)d.m * q / S), r1 = (int)((int64_t)d.m * (q + 1) / S);
          PieceDesc v = d;
          v.row_off = d.row_off + r0;
          v.m = r1 - r0;
          v.a_off = a2;
          v.id = (int)cp.pd_split.size();
          a2 += (int64_t)d.k * d.k;
          cp.pd_split.push_back(v);
        }
      }
      cp.split_a_doubles = (size_t)a2;
    }
  }
  return MDSX_OK;
}

static size_t classical_ws_bytes(const ClassicalPlan& cp, int p, int r) {
  const size_t np = cp.pd.size();
  return 6 * align_up(np * sizeof(PieceDesc)) + align_up(cp.tiles.size() * sizeof(int4)) +
         align_up(cp.tiles_g.size() * sizeof(int4)) +
         align_up(cp.tiles1.size() * sizeof(int4)) +
         align_up(np * p * sizeof(double)) + align_up(cp.a_doubles * sizeof(double)) +
         align_up(cp.u_doubles * sizeof(double)) + align_up(np * r * sizeof(double)) +
         align_up(points_ws_bytes((int)np, cp.max_m, r)) + align_up(np * sizeof(int)) +
         (cp.pd_big.empty() ? 0 : bk_ws_bytes(cp.pd_big)) +
         (cp.pd_split.empty() ? 0
                              : align_up(cp.split_a_doubles * sizeof(double)) +
                                    align_up(cp.pd_split.size() * (size_t)p * sizeof(double)) +
                                    align_up(cp.pd_split.size() * sizeof(mdsx_piece_status)) +
                                    align_up(cp.pd_split.size() * sizeof(PieceDesc)) +
                                    align_up(cp.split_rng.size() * sizeof(int4)));
}

// Runs K2 -> K1 -> K3 -> points for all pieces.  Workspace must be reserved.
// Device buffers of a run_classical call that later stages of the same call
// reuse (workspace of this call).
struct ClassicalOut {
  PieceDesc* dpd = nullptr;
  double* mu = nullptr;
  double* U = nullptr;
  double* lam = nullptr;
  // called once per piece chunk [j0, j1) right after its eigenpairs, on the
  // stream that solved it (the piece pipeline's chunk streams, or the caller's
  // stream for the whole batch): later stages of a chunk overlap the next
  // chunk's eigensolver
  std::function<int(int, int, cudaStream_t)> after_chunk;
};

// points == nullptr: eigenpairs only (no point matrices, no points epilogue).
static int run_classical(mdsx_handle* h, const ClassicalPlan& cp, const void* data, int dtype,
                         int64_t ld, int p, const int64_t* row_idx, int r, double* points,
                         double* estimates, double* gof, mdsx_piece_status* status,
                         cudaStream_t st, ClassicalOut* co = nullptr) {
  const int np = (int)cp.pd.size();
  PieceDesc* dpd = (PieceDesc*)ws_alloc(h, np * sizeof(PieceDesc), st);
  PieceDesc* dpd_jac = (PieceDesc*)ws_alloc(h, np * sizeof(PieceDesc), st);
  PieceDesc* dpd_sub = (PieceDesc*)ws_alloc(h, np * sizeof(PieceDesc), st);
  PieceDesc* dpd_f1 = (PieceDesc*)ws_alloc(h, np * sizeof(PieceDesc), st);
  PieceDesc* dpd_g = (PieceDesc*)ws_alloc(h, np * sizeof(PieceDesc), st);
  const bool piece_gram = gram_piece_ok(data, dtype, ld, p);
  std::vector<int4> tiles0 = cp.tiles;
  if (!piece_gram) tiles0.insert(tiles0.end(), cp.tiles_g.begin(), cp.tiles_g.end());
  int4* dtiles = (int4*)ws_alloc(h, tiles0.size() * sizeof(int4), st);
  int4* dtiles1 = (int4*)ws_alloc(h, cp.tiles1.size() * sizeof(int4), st);
  double* mu = (double*)ws_alloc(h, (size_t)np * p * sizeof(double), st);
  double* A = (double*)ws_alloc(h, cp.a_doubles * sizeof(double), st);
  double* U = (double*)ws_alloc(h, cp.u_doubles * sizeof(double), st);
  double* lam = (double*)ws_alloc(h, (size_t)np * r * sizeof(double), st);
  double2* cand = (double2*)ws_alloc(h, points_ws_bytes(np, cp.max_m, r), st);
  if (!dpd || !dtiles || !mu || !A || !U || !lam || !cand) return MDSX_CUDA;
  if (co) { co->dpd = dpd; co->mu = mu; co->U = U; co->lam = lam; }
  const int nsplit = (int)cp.pd_split.size();
  double* A_sp = nullptr;
  double* mu_sp = nullptr;
  mdsx_piece_status* st_sp = nullptr;
  PieceDesc* dpd_sp = nullptr;
  int4* drng = nullptr;
  if (nsplit) {
    A_sp = (double*)ws_alloc(h, cp.split_a_doubles * sizeof(double), st);
    mu_sp = (double*)ws_alloc(h, (size_t)nsplit * p * sizeof(double), st);
    st_sp = (mdsx_piece_status*)ws_alloc(h, nsplit * sizeof(mdsx_piece_status), st);
    dpd_sp = (PieceDesc*)ws_alloc(h, nsplit * sizeof(PieceDesc), st);
    drng = (int4*)ws_alloc(h, cp.split_rng.size() * sizeof(int4), st);
    if (!A_sp || !mu_sp || !st_sp || !dpd_sp || !drng) return MDSX_CUDA;
  }
  const std::vector<PieceDesc>& pd = cp.pd;  // row_off indexes row_idx directly
  const int64_t* ridx = row_idx;
  Stager sg(h, st);
  int rc = sg.begin(6 * np * sizeof(PieceDesc) + (tiles0.size() + cp.tiles1.size()) * sizeof(int4) +
                    nsplit * sizeof(PieceDesc) + cp.split_rng.size() * sizeof(int4) + 8192);
  if (rc) return rc;
  if ((rc = sg.put(dpd, pd.data(), np * sizeof(PieceDesc)))) return rc;
  if ((rc = sg.put(dpd_jac, cp.pd_jac.data(), cp.pd_jac.size() * sizeof(PieceDesc)))) return rc;
  if ((rc = sg.put(dpd_sub, cp.pd_sub.data(), cp.pd_sub.size() * sizeof(PieceDesc)))) return rc;
  if ((rc = sg.put(dtiles, tiles0.data(), tiles0.size() * sizeof(int4)))) return rc;
  if (piece_gram && (rc = sg.put(dpd_g, cp.pd_g.data(), cp.pd_g.size() * sizeof(PieceDesc))))
    return rc;
  if ((rc = sg.put(dpd_f1, cp.pd_f1.data(), cp.pd_f1.size() * sizeof(PieceDesc)))) return rc;
  if ((rc = sg.put(dtiles1, cp.tiles1.data(), cp.tiles1.size() * sizeof(int4)))) return rc;
  if (nsplit) {
    if ((rc = sg.put(dpd_sp, cp.pd_split.data(), nsplit * sizeof(PieceDesc)))) return rc;
    if ((rc = sg.put(drng, cp.split_rng.data(), cp.split_rng.size() * sizeof(int4)))) return rc;
  }
  if ((rc = sg.end())) return rc;
  if ((rc = cuda_check(h, cudaMemsetAsync(status, 0, np * sizeof(mdsx_piece_status), st), "memset")))
    return rc;
  // Piece pipeline (the BASELINE D&C / fast shapes: every piece form 0 with
  // k <= 104, Lanczos route): chunks of pieces alternate between the caller's
  // stream and a second one, so one chunk's latency-bound eigensolver runs
  // next to another chunk's HBM / tensor-bound Gram and points kernels.
  // Same kernels and per-piece arithmetic, so results are unchanged.
  {
    const char* pc = getenv("MDSX_PIPE_CHUNKS");
    const bool simple = piece_gram && cp.pd_jac.empty() && cp.pd_big.empty() && cp.pd_f1.empty() &&
                        (int)cp.pd_g.size() == np && (int)cp.pd_sub.size() == np;
    int nc = pc ? atoi(pc) : 2;                       // measured best on dc2 / fast3
    const bool serial = getenv("MDSX_PIPE_SERIAL") != nullptr;
    nc = std::min(nc, np / (2 * h->num_sms));          // >= two waves of pieces per chunk
    if (pc == nullptr && nc > 2) nc = 2;
    // fused points epilogue in the Lanczos kernel (aligned rows, r <= 10): each
    // CTA streams its piece's rows right after its eigenvectors, next to the
    // other CTA's Krylov phase; the points kernel then only takes the pieces
    // the epilogue left pending (Jacobi fallback / non-finite input)
    const size_t es = dtype == MDSX_F32 ? 4 : 8;
    const bool fuse = simple && r <= 10 && data != nullptr && points != nullptr && ((size_t)p * es) % 16 == 0 &&
                      ((size_t)ld * es) % 16 == 0 && (reinterpret_cast<uintptr_t>(data) & 15) == 0 &&
                      !getenv("MDSX_POINTS_TILED") && !getenv("MDSX_NO_FUSE");
    int* pending = fuse ? (int*)ws_alloc(h, (size_t)np * sizeof(int), st) : nullptr;
    if (fuse && !pending) return MDSX_CUDA;
    PtsEpi epi{data, dtype == MDSX_F32 ? 1 : 0, ld, p, ridx, mu, points, pending};
    if (simple && nc > 1) {
      nc = std::min(nc, 4);
      if (!h->pipe[0]) {
        for (int c = 0; c < 4; ++c) {
          if ((rc = cuda_check(h, cudaStreamCreateWithFlags(&h->pipe[c], cudaStreamNonBlocking),
                               "stream")))
            return rc;
          cudaEventCreateWithFlags(&h->ev_pj[c], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
      }
      cudaEventRecord(h->ev_fork, st);
      for (int c = 0; c < nc && !serial; ++c) cudaStreamWaitEvent(h->pipe[c], h->ev_fork, 0);
      for (int c = 0; c < nc; ++c) {
        const int j0 = (int)((int64_t)np * c / nc), j1 = (int)((int64_t)np * (c + 1) / nc);
        const int n = j1 - j0;
        // MDSX_PIPE_SERIAL: every chunk on the caller's stream (same kernels and
        // chunks, no overlap) -- bench.py's per-kernel timing pass
        cudaStream_t s = serial ? st : h->pipe[c];
        if ((rc = launch_gram_piece(h, data, dtype, ld, p, ridx, dpd + j0, n, A, mu, status, s)))
          return rc;
        if ((rc = launch_lanczos_smem(h, dpd + j0, n, cp.kmax_sub, r, A, U, lam, estimates, gof,
                                      status, 0, 0, s, fuse ? &epi : nullptr)))
          return rc;
        if ((rc = launch_jacobi_fallback(h, dpd + j0, n, cp.kmax_sub, r, A, U, lam, estimates, gof,
                                         status, s)))
          return rc;
        if (points && (rc = launch_points(h, data, dtype, ld, p, ridx, dpd + j0, n, cp.max_m, r, mu,
                                          U, lam, points, cand, s, true, pending)))
          return rc;
        if (co && co->after_chunk && (rc = co->after_chunk(j0, j1, s))) return rc;
      }
      for (int c = 0; c < nc && !serial; ++c) {
        cudaEventRecord(h->ev_pj[c], h->pipe[c]);
        if ((rc = cuda_check(h, cudaStreamWaitEvent(st, h->ev_pj[c], 0), "pipeline join"))) return rc;
      }
      return MDSX_OK;
    }
  }
  // form 0: DMMA Gram with fused shifted means;  form 1: means pass + row Gram
  if (piece_gram && nsplit) {
    // row-split Grams of the few large pieces, combined (Chan et al.) in fixed order
    if ((rc = cuda_check(h, cudaMemsetAsync(st_sp, 0, nsplit * sizeof(mdsx_piece_status), st),
                         "memset")))
      return rc;
    if ((rc = launch_gram_piece(h, data, dtype, ld, p, ridx, dpd_sp, nsplit, A_sp, mu_sp, st_sp, st)))
      return rc;
    if ((rc = launch_gram_combine(h, dpd_g, drng, (int)cp.split_rng.size(), dpd_sp, A_sp, mu_sp,
                                  st_sp, p, A, mu, status, st)))
      return rc;
  } else if (piece_gram && (rc = launch_gram_piece(h, data, dtype, ld, p, ridx, dpd_g,
                                                   (int)cp.pd_g.size(), A, mu, status, st))) {
    return rc;
  }
  if ((rc = launch_gram_dmma(h, data, dtype, ld, p, ridx, dpd, dtiles, (int)tiles0.size(), A, mu,
                             status, st)))
    return rc;
  if (!cp.pd_f1.empty()) {
    if ((rc = launch_piece_means(h, data, dtype, ld, p, ridx, dpd_f1, (int)cp.pd_f1.size(), mu,
                                 status, st)))
      return rc;
    if ((rc = launch_gram(h, data, dtype, ld, p, ridx, dpd, mu, dtiles1, (int)cp.tiles1.size(), A,
                          st)))
      return rc;
  }
  if (!cp.pd_jac.empty() &&
      (rc = launch_jacobi(h, dpd_jac, (int)cp.pd_jac.size(), cp.kmax_jac, r, A, U, lam, estimates,
                          gof, status, 1, st)))
    return rc;
  if (!cp.pd_sub.empty()) {
    if ((rc = launch_lanczos_smem(h, dpd_sub, (int)cp.pd_sub.size(), cp.kmax_sub, r, A, U, lam,
                                  estimates, gof, status, 0, 0, st)))
      return rc;
    if ((rc = launch_jacobi_fallback(h, dpd_sub, (int)cp.pd_sub.size(), cp.kmax_sub, r, A, U, lam,
                                     estimates, gof, status, st)))
      return rc;
  }
  if (!cp.pd_big.empty() &&
      (rc = run_big_pieces(h, cp.pd_big, A, r, U, lam, estimates, gof, status, st, stage_put)))
    return rc;
  if (co && co->after_chunk && (rc = co->after_chunk(0, np, st))) return rc;
  if (!points) return MDSX_OK;
  return launch_points(h, data, dtype, ld, p, ridx, dpd, np, cp.max_m, r, mu, U, lam, points,
                       cand, st, cp.pd_f1.empty());
}

}  // namespace mdsx

using namespace mdsx;

extern "C" {

int mdsx_version(void) { return 1; }

int mdsx_create(int device, mdsx_handle** out) {
  if (!out) return MDSX_PARAM;
  *out = nullptr;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return MDSX_CUDA;
  auto* h = new mdsx_handle();
  h->device = device;
  cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&h->max_smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  *out = h;
  return MDSX_OK;
}

void mdsx_destroy(mdsx_handle* h) {
  if (!h) return;
  cudaDeviceSynchronize();
  if (h->ws) cudaFree(h->ws);
  if (h->pinned) cudaFreeHost(h->pinned);
  if (h->pinned_free) cudaEventDestroy(h->pinned_free);
  for (auto& t : h->timed) { cudaEventDestroy(t.second.first); cudaEventDestroy(t.second.second); }
  for (auto e : h->event_pool) cudaEventDestroy(e);
  if (h->aux) cudaStreamDestroy(h->aux);
  for (int c = 0; c < 4; ++c) {
    if (h->pipe[c]) cudaStreamDestroy(h->pipe[c]);
    if (h->ev_pj[c]) cudaEventDestroy(h->ev_pj[c]);
  }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->ws_done) cudaEventDestroy(h->ws_done);
  if (h->ev_anchor) cudaEventDestroy(h->ev_anchor);
  delete h;
}

const char* mdsx_last_error(const mdsx_handle* h) { return h ? t_last_error.c_str() : "null handle"; }

int64_t mdsx_launch_count(const mdsx_handle* h) { return h ? h->launches : 0; }

int mdsx_timing_enable(mdsx_handle* h, int on) {
  if (!h) return MDSX_PARAM;
  std::lock_guard<std::recursive_mutex> lk(h->mu);
  h->timing = on != 0;
  return MDSX_OK;
}

int64_t mdsx_timing_trace(mdsx_handle* h, char* buf, int64_t cap) {
  if (!h) return -1;
  std::lock_guard<std::recursive_mutex> lk(h->mu);
  std::string out;
  if (!h->timed.empty()) {
    cudaEvent_t base = h->timed.front().second.first;
    for (auto& t : h->timed) {
      cudaEventSynchronize(t.second.second);
      float a = 0.f, b = 0.f;
      cudaEventElapsedTime(&a, base, t.second.first);
      cudaEventElapsedTime(&b, base, t.second.second);
      char line[160];
      snprintf(line, sizeof line, "%s %.4f %.4f\n", t.first, a, b);
      out += line;
    }
  }
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(out.size(), (size_t)cap - 1);
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int64_t)out.size();
}

int64_t mdsx_timing_report(mdsx_handle* h, char* buf, int64_t cap) {
  if (!h) return -1;
  std::lock_guard<std::recursive_mutex> lk(h->mu);
  // fold pending event pairs into the running per-kernel totals
  for (auto& t : h->timed) {
    cudaEventSynchronize(t.second.second);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.second.first, t.second.second);
    auto it = std::find_if(h->report.begin(), h->report.end(),
                           [&](auto& a) { return a.first == t.first; });
    if (it == h->report.end()) h->report.push_back({t.first, {ms, 1}});
    else { it->second.first += ms; it->second.second += 1; }
    h->event_pool.push_back(t.second.first);
    h->event_pool.push_back(t.second.second);
  }
  h->timed.clear();
  std::string out;
  for (auto& a : h->report) {
    double w = 0.0;
    for (auto& x : h->work)
      if (x.first == a.first) w = x.second;
    char wb[64];
    snprintf(wb, sizeof wb, "%.17g", w);
    out += a.first + " " + std::to_string(a.second.first) + " " + std::to_string(a.second.second) +
           " " + wb + "\n";
  }
  if (buf && cap > 0) {  // a call with a buffer consumes the totals
    const size_t n = std::min<size_t>(out.size(), (size_t)cap - 1);
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
    h->report.clear();
    h->work.clear();
  }
  return (int64_t)out.size();
}

int mdsx_sqdist_self(mdsx_handle* h, const void* x, int dtype, int64_t ld, int64_t m, int32_t p,
                     double* out, int64_t ldo, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (m < 1 || p < 1) return fail(h, MDSX_INVALID_INPUT, "data must be non-empty");
  const int64_t ta = (m + 63) / 64;                      // lower-triangle 64 x 64 tiles
  int rc = ws_reserve(h, align_up(m * sizeof(double)) + align_up(ta * (ta + 1) / 2 * 8) + 512);
  if (rc) return rc;
  double* na = (double*)ws_alloc(h, m * sizeof(double), st);
  return launch_sqdist(h, x, ld, m, x, ld, m, dtype, p, na, na, out, ldo, 1, st);
}

int mdsx_sqdist_cross(mdsx_handle* h, const void* a, int64_t lda, int64_t ma, const void* b,
                      int64_t ldb, int64_t mb, int dtype, int32_t p, double* out, int64_t ldo,
                      void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  int rc = ws_reserve(h, align_up(ma * sizeof(double)) + align_up(mb * sizeof(double)));
  if (rc) return rc;
  double* na = (double*)ws_alloc(h, ma * sizeof(double), st);
  double* nb = (double*)ws_alloc(h, mb * sizeof(double), st);
  return launch_sqdist(h, a, lda, ma, b, ldb, mb, dtype, p, na, nb, out, ldo, 0, st);
}

int mdsx_double_center(mdsx_handle* h, const double* delta, int64_t m, double* q, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  int rc = ws_reserve(h, align_up(m * sizeof(double)) + 256);
  if (rc) return rc;
  double* mu = (double*)ws_alloc(h, m * sizeof(double), st);
  double* g = (double*)ws_alloc(h, sizeof(double), st);
  return launch_double_center(h, delta, m, mu, g, q, st);
}

int mdsx_classical_pieces(mdsx_handle* h, const void* data, int dtype, int64_t ld, int32_t p,
                          const int64_t* row_idx, const int64_t* piece_off, int32_t npieces,
                          int32_t r, double* points, double* estimates, double* gof,
                          mdsx_piece_status* status, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  ClassicalPlan cp;
  int rc = plan_classical(h, p, piece_off, npieces, r, cp);
  if (rc) return rc;
  if ((rc = ws_reserve(h, classical_ws_bytes(cp, p, r)))) return rc;
  return run_classical(h, cp, data, dtype, ld, p, row_idx, r, points, estimates, gof, status, st);
}

int mdsx_classical_delta(mdsx_handle* h, const double* delta, int64_t m, int32_t r, double* points,
                         double* estimates, double* gof, mdsx_piece_status* status, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (r < 1 || r > m - 1 || r > MDSX_MAX_R)
    return fail(h, MDSX_PARAM, "r must satisfy 1 <= r <= n-1, got r=" + std::to_string(r) +
                                   ", n=" + std::to_string(m));
  const bool big = m > MDSX_JACOBI_KMAX;     // top-r by block Krylov (full spectrum: caller)
  if (big && r > 12)
    return fail(h, MDSX_UNSUPPORTED, "classical_mds(delta) with n > " +
                                         std::to_string(MDSX_JACOBI_KMAX) + " handles r <= 12");
  PieceDesc d{};
  d.m = (int)m; d.k = (int)m; d.form = 1;
  const std::vector<PieceDesc> bigv(big ? 1 : 0, d);
  const size_t need = align_up(sizeof(PieceDesc)) + align_up(m * m * sizeof(double)) * 2 +
                      align_up(m * r * sizeof(double)) + align_up(r * sizeof(double)) +
                      align_up(m * sizeof(double)) + align_up(points_ws_bytes(1, m, r)) + 512 + 256 +
                      (big ? bk_ws_bytes(bigv) : 0);
  int rc = ws_reserve(h, need);
  if (rc) return rc;
  PieceDesc* dpd = (PieceDesc*)ws_alloc(h, sizeof(PieceDesc), st);
  double* Q = (double*)ws_alloc(h, m * m * sizeof(double), st);
  double* U = (double*)ws_alloc(h, m * r * sizeof(double), st);
  double* lam = (double*)ws_alloc(h, r * sizeof(double), st);
  double* mu = (double*)ws_alloc(h, m * sizeof(double), st);
  double* g = (double*)ws_alloc(h, sizeof(double), st);
  double2* cand = (double2*)ws_alloc(h, points_ws_bytes(1, m, r), st);
  Stager sg(h, st);
  if ((rc = sg.begin(sizeof(PieceDesc)))) return rc;
  if ((rc = sg.put(dpd, &d, sizeof(PieceDesc)))) return rc;
  if ((rc = sg.end())) return rc;
  if ((rc = launch_double_center(h, delta, m, mu, g, Q, st))) return rc;
  if ((rc = cuda_check(h, cudaMemsetAsync(status, 0, sizeof(mdsx_piece_status), st), "memset")))
    return rc;
  if (big) {
    // largest algebraic eigenpairs of the (possibly indefinite) Q; the trivial
    // mode (Q 1 = 0) sits at eigenvalue 0 and is never among them unless the
    // spectrum is degenerate.  G1/G2 here are trace-based: the Python layer
    // replaces them (and the DegenerateRank decision) from the full spectrum.
    if ((rc = run_big_pieces(h, bigv, Q, r, U, lam, estimates, gof, status, st, stage_put)))
      return rc;
  } else if ((rc = launch_jacobi(h, dpd, 1, (int)m, r, Q, U, lam, estimates, gof, status, 1, st))) {
    return rc;
  }
  return launch_points(h, nullptr, MDSX_F64, 0, 0, nullptr, dpd, 1, m, r, nullptr, U, lam, points,
                       cand, st);
}

int mdsx_sym_eigvals(mdsx_handle* h, const double* a, int64_t n, double* w, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (n < 1) return fail(h, MDSX_SHAPE, "matrix must be non-empty");
  if (n > 20000) return fail(h, MDSX_PARAM, "n exceeds the exact-size guard (20000)");
  const size_t nd = eigvals_ws_doubles(n);
  int rc = ws_reserve(h, align_up(nd * sizeof(double)) + 256);
  if (rc) return rc;
  double* ws = (double*)ws_alloc(h, nd * sizeof(double), st);
  if (!ws) return MDSX_CUDA;
  return launch_sym_eigvals(h, a, n, w, ws, st);
}

int mdsx_delta_check(mdsx_handle* h, const double* delta, int64_t m, int32_t* flags, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  int rc = ws_reserve(h, 256);
  if (rc) return rc;
  auto* mx = (unsigned long long*)ws_alloc(h, sizeof(unsigned long long), st);
  if ((rc = cuda_check(h, cudaMemsetAsync(mx, 0, sizeof(unsigned long long), st), "memset")))
    return rc;
  return launch_delta_check(h, delta, m, mx, flags, st);
}

int64_t mdsx_gower_context_size(int64_t l, int32_t p, int32_t r) {
  return (int64_t)p + (int64_t)p * r + r + (int64_t)r * r + l;
}

int mdsx_gower_context(mdsx_handle* h, const void* data, int dtype, int64_t ld, int32_t p,
                       const int64_t* base_idx, int64_t l, const double* base_config, int32_t r,
                       double* ctx, double* cond, int32_t* flag, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (r < 1 || r > MDSX_MAX_R) return fail(h, MDSX_PARAM, "bad r");
  double* mean = ctx;
  double* M = mean + p;
  double* v = M + (int64_t)p * r;
  double* S = v + r;
  double* q = S + (int64_t)r * r;
  return launch_gower_context(h, data, dtype, ld, p, base_idx, l, base_config, r, mean, M, v, S, q,
                              cond, flag, st);
}

int mdsx_gower_interpolate(mdsx_handle* h, const double* ctx, int64_t l, int32_t p, int32_t r,
                           const void* rows, int dtype, int64_t ld, int64_t m, double* out,
                           int64_t ldo, int32_t* nonfinite, int32_t flags, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  int32_t* nf = nonfinite;
  const double* mean = ctx;
  const double* M = mean + p;
  const double* v = M + (int64_t)p * r;
  (void)l;
  if (m < 1) return MDSX_OK;
  // dense aligned rows, packed output: the bulk-copy streaming kernel (its
  // per-CTA column sums go to scratch); otherwise the per-row kernel
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  if (ld == p && ldo == r && r <= 16 && ((size_t)p * es) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(rows) & 15) == 0 &&
      h->num_sms * r * sizeof(double) <= recenter_ws_bytes(r)) {
    int rc = ws_reserve(h, recenter_ws_bytes(r) + 256);
    if (rc) return rc;
    double* part = (double*)ws_alloc(h, recenter_ws_bytes(r), st);
    int nparts = 0;
    const bool n32 = dtype == MDSX_F32 && (flags & MDSX_GOWER_CENTRED) && !getenv("MDSX_GOWER_NORM64");
    if ((rc = launch_gower_bulk(h, rows, dtype, m, p, r, mean, M, v, out, part, nf, &nparts, st,
                                n32)))
      return rc;
    if (nparts > 0) return MDSX_OK;
  }
  return launch_gower_affine(h, rows, dtype, ld, m, p, r, mean, M, v, out, ldo, nf, st);
}

static bool gower_tiles_fit(mdsx_handle* h, const void* rows, int dtype, int64_t ld, int p, int r) {
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  return ld == p && r <= 16 && ((size_t)p * es) % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(rows) & 15) == 0 && gower_tile_rows(h, dtype, p, r) > 0;
}

int32_t mdsx_gower_tile_rows(mdsx_handle* h, int dtype, int32_t p, int32_t r) {
  if (!h || p < 1 || r < 1) return 0;
  return gower_tile_rows(h, dtype, p, r);
}

int mdsx_gower_tiles(mdsx_handle* h, const double* ctx, int64_t l, int32_t p, int32_t r,
                     const void* rows, int dtype, int64_t m, double* out, double* tile_sums,
                     int32_t* nonfinite, int32_t flags, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  (void)l;
  if (!ctx || !out || !tile_sums || !nonfinite || m < 0) return fail(h, MDSX_PARAM, "bad gower tiles arguments");
  if (m > 0 && (!rows || !gower_tiles_fit(h, rows, dtype, p, p, r)))
    return fail(h, MDSX_UNSUPPORTED, "gower tiles: rows must be dense, 16-byte aligned, r <= 16");
  const double* mean = ctx;
  const double* M = mean + p;
  const double* v = M + (int64_t)p * r;
  int tile_rows = 0;
  const bool n32 = dtype == MDSX_F32 && (flags & MDSX_GOWER_CENTRED) && !getenv("MDSX_GOWER_NORM64");
  return launch_gower_bulk(h, rows, dtype, m, p, r, mean, M, v, out, tile_sums, nonfinite,
                           &tile_rows, st, n32, true);
}

int mdsx_landmark_overwrite(mdsx_handle* h, const double* base, int64_t l, int32_t r,
                            const int64_t* sel, const int64_t* pos, int64_t nl, double* out,
                            double* corr, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (!base || !corr || (nl > 0 && (!pos || !out)) || nl < 0 || nl > l || r < 1)
    return fail(h, MDSX_PARAM, "bad landmark overwrite arguments");
  int rc = cuda_check(h, cudaMemsetAsync(corr, 0, (size_t)l * r * sizeof(double), st), "memset");
  if (rc) return rc;
  return launch_landmark_corr(h, base, sel, pos, nl, r, out, corr, st);
}

int mdsx_interp_recenter(mdsx_handle* h, const double* tile_sums, int64_t ntiles,
                         const double* corr, int64_t l, int32_t r, int64_t n_total, double* out,
                         int64_t m, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if ((ntiles > 0 && !tile_sums) || !corr || n_total < 1 || m < 0 || r < 1 || r > MDSX_MAX_R)
    return fail(h, MDSX_PARAM, "bad recentre arguments");
  int rc = ws_reserve(h, fold_ws_bytes(ntiles, l, r) + 256);
  if (rc) return rc;
  double* ws = (double*)ws_alloc(h, fold_ws_bytes(ntiles, l, r), st);
  if (!ws) return MDSX_CUDA;
  double* total = nullptr;
  if ((rc = launch_fold_sums(h, tile_sums, ntiles, corr, l, r, ws, &total, st))) return rc;
  return launch_subtract_mean(h, out, m, r, total, 1, nullptr, st, n_total);
}

int mdsx_procrustes_fit(mdsx_handle* h, const double* tgt, const int64_t* tgt_rows,
                        const double* src, const int64_t* src_rows, const int64_t* job_off,
                        int32_t njobs, int32_t r, double* rot, double* trans, double* loss,
                        int32_t* degenerate, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (r < 1 || r > MDSX_MAX_R) return fail(h, MDSX_PARAM, "bad r");
  for (int j = 0; j < njobs; ++j)
    if (job_off[j + 1] - job_off[j] < 2)
      return fail(h, MDSX_SHAPE, "need at least 2 rows and 1 column");
  int rc = ws_reserve(h, align_up((size_t)(njobs + 1) * sizeof(int64_t)));
  if (rc) return rc;
  int64_t* doff = (int64_t*)ws_alloc(h, (size_t)(njobs + 1) * sizeof(int64_t), st);
  Stager sg(h, st);
  if ((rc = sg.begin((size_t)(njobs + 1) * sizeof(int64_t)))) return rc;
  if ((rc = sg.put(doff, job_off, (size_t)(njobs + 1) * sizeof(int64_t)))) return rc;
  if ((rc = sg.end())) return rc;
  return launch_procrustes_fit(h, tgt, tgt_rows, src, src_rows, doff, njobs, r, rot, trans, loss,
                               degenerate, st);
}

int mdsx_procrustes_apply(mdsx_handle* h, double* buf, int32_t r, const int64_t* start,
                          const int64_t* len, int32_t njobs, int64_t max_len, const double* rot,
                          const double* trans, void* stream) {
  MDSX_GUARD(h, as_stream(stream));
  if (r < 1 || r > MDSX_MAX_R) return fail(h, MDSX_PARAM, "bad r");
  return launch_apply(h, buf, r, start, len, njobs, max_len, rot, trans, as_stream(stream));
}

int mdsx_scatter_rows(mdsx_handle* h, const double* src, const int64_t* idx, int64_t n, int32_t r,
                      double* out, void* stream) {
  MDSX_GUARD(h, as_stream(stream));
  return launch_scatter(h, src, idx, n, r, out, as_stream(stream));
}

int mdsx_recenter(mdsx_handle* h, double* points, int64_t n, int32_t r, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (r < 1 || r > MDSX_MAX_R) return fail(h, MDSX_PARAM, "bad r");
  int rc = ws_reserve(h, recenter_ws_bytes(r));
  if (rc) return rc;
  double* part = (double*)ws_alloc(h, recenter_ws_bytes(r), st);
  return launch_recenter(h, points, n, r, part, st);
}

int mdsx_segment_colsums(mdsx_handle* h, const double* points, const int64_t* idx,
                         const int64_t* seg_off, int32_t nseg, int32_t r, double* sums,
                         void* stream) {
  MDSX_GUARD(h, as_stream(stream));
  if (r < 1 || r > MDSX_MAX_R) return fail(h, MDSX_PARAM, "bad r");
  return launch_seg_colsum(h, points, idx, seg_off, nseg, r, sums, as_stream(stream));
}

int mdsx_shift_rows(mdsx_handle* h, double* points, const int64_t* idx, int64_t n, int32_t r,
                    const double* shift, void* stream) {
  MDSX_GUARD(h, as_stream(stream));
  if (r < 1 || r > MDSX_MAX_R) return fail(h, MDSX_PARAM, "bad r");
  return launch_shift_rows(h, points, idx, n, r, shift, as_stream(stream));
}

int mdsx_divide_conquer(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n,
                        int32_t p, const int64_t* row_idx, const int64_t* piece_off,
                        int32_t npieces, int32_t c, int32_t r, double* out, double* estimates,
                        double* gof, mdsx_piece_status* status, void* stream) {
  return mdsx_divide_conquer_ex(h, data, dtype, ld, n, p, row_idx, piece_off, npieces, c, r, out,
                                estimates, gof, status, 0, stream);
}

using ShardOps = ContribGather;

static int dc_impl(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n, int32_t p,
                   const int64_t* row_idx, const int64_t* piece_off, int32_t npieces, int32_t c,
                   int32_t r, double* out, double* estimates, double* gof,
                   mdsx_piece_status* status, int32_t flags, cudaStream_t st, const ShardOps* shard);

int mdsx_divide_conquer_ex(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n,
                           int32_t p, const int64_t* row_idx, const int64_t* piece_off,
                           int32_t npieces, int32_t c, int32_t r, double* out, double* estimates,
                           double* gof, mdsx_piece_status* status, int32_t flags, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  return dc_impl(h, data, dtype, ld, n, p, row_idx, piece_off, npieces, c, r, out, estimates, gof,
                 status, flags, st, nullptr);
}

int mdsx_divide_conquer_sharded(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n,
                                int32_t p, const int64_t* row_idx, const int64_t* piece_off,
                                int32_t npieces, int32_t c, int32_t r, double* out,
                                double* estimates, double* gof, mdsx_piece_status* status,
                                int64_t n_total, int32_t npieces_total, double* contrib_local,
                                double* contrib_global, mdsx_gather_fn gather, void* ctx,
                                void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (!contrib_local || !contrib_global || !gather || npieces_total < npieces || n_total < n)
    return fail(h, MDSX_PARAM, "bad sharded D&C arguments");
  const ShardOps ops{contrib_local, contrib_global, npieces_total, n_total, gather, ctx};
  return dc_impl(h, data, dtype, ld, n, p, row_idx, piece_off, npieces, c, r, out, estimates, gof,
                 status, 0, st, &ops);
}

static int dc_impl(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n, int32_t p,
                   const int64_t* row_idx, const int64_t* piece_off, int32_t npieces, int32_t c,
                   int32_t r, double* out, double* estimates, double* gof,
                   mdsx_piece_status* status, int32_t flags, cudaStream_t st, const ShardOps* shard) {
  ClassicalPlan cp;
  int rc = plan_classical(h, p, piece_off, npieces, r, cp);
  if (rc) return rc;
  if (piece_off[0] != 0) return fail(h, MDSX_PARAM, "piece_off[0] must be 0");
  if (npieces > 1) {
    if (c < 2 || c < r) return fail(h, MDSX_PARAM, "c must be >= max(r, 2)");
    for (int j = 0; j < npieces; ++j)
      if (piece_off[j + 1] - piece_off[j] <= c) return fail(h, MDSX_PARAM, "l must exceed c");
  }
  const int nj = std::max(npieces - 1, 0);
  const size_t fit_rows = (size_t)nj * c;
  const bool rec = !(flags & MDSX_NO_RECENTER);
  // form-0 pieces, aligned rows: no per-piece point matrices -- anchor signs
  // and connecting-row points only, fits, then one fused output pass
  // (k_dcout.cu); otherwise points of every piece, fits, stitch
  if (npieces > 1 && cp.pd_f1.empty() && dc_out_route_ok(data, dtype, ld, p, r, c) &&
      !getenv("MDSX_DC_POINTS")) {
    const int64_t m0 = piece_off[1] - piece_off[0];
    const size_t need = classical_ws_bytes(cp, p, r) + align_up(dc_out_ws_doubles(npieces, p, r, c, m0) * 8) + 4096 +
                        align_up(fit_rows * sizeof(int64_t)) * 2 +
                        align_up((size_t)(nj + 1) * sizeof(int64_t)) +
                        align_up((size_t)nj * r * r * sizeof(double)) +
                        align_up((size_t)nj * r * sizeof(double)) + align_up(nj * sizeof(double)) +
                        align_up(nj * sizeof(int32_t)) + align_up(npieces * sizeof(int32_t)) + 8192;
    if ((rc = ws_reserve(h, need))) return rc;
    double* Pc = (double*)ws_alloc(h, (size_t)npieces * c * r * sizeof(double), st);
    double* Uc = (double*)ws_alloc(h, (size_t)npieces * p * r * sizeof(double), st);
    double* contrib = (double*)ws_alloc(h, (size_t)npieces * r * sizeof(double), st);
    double* tvec = (double*)ws_alloc(h, (size_t)npieces * r * sizeof(double), st);
    double* Pa = (double*)ws_alloc(h, (size_t)m0 * r * sizeof(double), st);
    double* mean = (double*)ws_alloc(h, 64 * sizeof(double), st);
    double* zero = (double*)ws_alloc(h, 64 * sizeof(double), st);
    double* rot = (double*)ws_alloc(h, (size_t)nj * r * r * sizeof(double), st);
    double* trans = (double*)ws_alloc(h, (size_t)nj * r * sizeof(double), st);
    int64_t* trows = (int64_t*)ws_alloc(h, fit_rows * sizeof(int64_t), st);
    int64_t* srows = (int64_t*)ws_alloc(h, fit_rows * sizeof(int64_t), st);
    int64_t* joff = (int64_t*)ws_alloc(h, (size_t)(nj + 1) * sizeof(int64_t), st);
    double* loss = (double*)ws_alloc(h, nj * sizeof(double), st);
    int32_t* degen = (int32_t*)ws_alloc(h, nj * sizeof(int32_t), st);
    int32_t* pending = (int32_t*)ws_alloc(h, (size_t)npieces * sizeof(int32_t), st);
    if (!Pc || !Uc || !contrib || !tvec || !Pa || !mean || !zero || !rot || !trans || !trows ||
        !srows || !joff || !loss || !degen || !pending)
      return MDSX_CUDA;
    std::vector<int64_t> ht(fit_rows), hs(fit_rows), hj(nj + 1);
    for (int j = 0; j < nj; ++j) {
      hj[j] = (int64_t)j * c;
      for (int t = 0; t < c; ++t) {
        ht[(size_t)j * c + t] = t;                              // anchor rows 0..c-1
        hs[(size_t)j * c + t] = (int64_t)(j + 1) * c + t;       // piece j+1 connecting rows
      }
    }
    hj[nj] = (int64_t)nj * c;
    {
      Stager sg(h, st);
      if ((rc = sg.begin(fit_rows * 16 + (nj + 1) * 8 + 1024))) return rc;
      if ((rc = sg.put(trows, ht.data(), fit_rows * sizeof(int64_t)))) return rc;
      if ((rc = sg.put(srows, hs.data(), fit_rows * sizeof(int64_t)))) return rc;
      if ((rc = sg.put(joff, hj.data(), (nj + 1) * sizeof(int64_t)))) return rc;
      if ((rc = sg.end())) return rc;
    }
    if ((rc = cuda_check(h, cudaMemsetAsync(zero, 0, 64 * sizeof(double), st), "memset"))) return rc;
    if (!h->ev_anchor) cudaEventCreateWithFlags(&h->ev_anchor, cudaEventDisableTiming);
    // per chunk of pieces, on the stream that solved it: anchor signs (chunk 0),
    // connecting points, fits, U' = U T, output rows (not yet re-centred)
    ClassicalOut co;
    // the anchor's signs and Procrustes targets right after its chunk's
    // eigenpairs (next to the other chunks' eigensolvers); the rest of the tail
    // once for every piece after the join: connecting points, fits, U' = U T,
    // then the column mean from the per-piece contributions, so the single
    // output pass writes the re-centred rows (no shift pass)
    co.after_chunk = [&](int j0, int j1, cudaStream_t s) -> int {
      (void)j1;
      if (j0 != 0) return MDSX_OK;
      return launch_dc_points(h, data, dtype, ld, p, row_idx, co.dpd, 1, r, c, m0, co.mu, co.U, Pc,
                              Pa, s);
    };
    if ((rc = run_classical(h, cp, data, dtype, ld, p, row_idx, r, nullptr, estimates, gof, status,
                            st, &co)))
      return rc;
    if (dc_fit_ok(r, c, p)) {
      // one warp per subset: connecting points, Newton-Schulz fit, composition;
      // fits it does not converge on: Jacobi fit + composition (pending mode)
      if ((rc = launch_dc_fit(h, data, dtype, ld, p, row_idx, co.dpd, npieces, r, c, co.mu, co.U, Pc,
                              rot, trans, loss, degen, Uc, tvec, contrib, pending, st)))
        return rc;
      if ((rc = launch_procrustes_fit(h, Pc, trows, Pc, srows, joff, npieces - 1, r, rot, trans,
                                      loss, degen, st, true)))
        return rc;
      if ((rc = launch_dc_compose(h, co.dpd, 0, npieces, p, r, c, co.U, rot, trans, Pc, Uc, tvec,
                                  contrib, st, pending)))
        return rc;
    } else {
      if ((rc = launch_dc_conn(h, data, dtype, ld, p, row_idx, co.dpd, 1, npieces - 1, r, c, co.mu,
                               co.U, Pc, st)))
        return rc;
      if ((rc = launch_procrustes_fit(h, Pc, trows, Pc, srows, joff, npieces - 1, r, rot, trans,
                                      loss, degen, st)))
        return rc;
      if ((rc = launch_dc_compose(h, co.dpd, 0, npieces, p, r, c, co.U, rot, trans, Pc, Uc, tvec,
                                  contrib, st)))
        return rc;
    }
    if (shard && shard->gather) {
      // sharded: every rank's contributions in global subset order (the
      // caller's collective), then the same fixed-order mean on every rank
      if ((rc = cuda_check(h, cudaMemcpyAsync(shard->local, contrib,
                                              (size_t)npieces * r * sizeof(double),
                                              cudaMemcpyDeviceToDevice, st), "contrib copy")))
        return rc;
      if (shard->gather(shard->ctx, st) != 0) return fail(h, MDSX_CUDA, "contribution gather failed");
      if ((rc = launch_dc_mean(h, shard->global, shard->total, r, shard->n_total, mean,
                               st)))
        return rc;
      return launch_piece_out(h, data, dtype, ld, p, row_idx, nullptr, co.dpd, npieces, cp.max_m, r, c,
                              co.mu, Uc, tvec, mean, out, st);
    }
    if (rec && (rc = launch_dc_mean(h, contrib, npieces, r, n, mean, st))) return rc;
    return launch_piece_out(h, data, dtype, ld, p, row_idx, nullptr, co.dpd, npieces, cp.max_m, r, c,
                            co.mu, Uc, tvec, rec ? mean : zero, out, st);
  }
  if (shard) return fail(h, MDSX_UNSUPPORTED, "sharded D&C needs the fused output route");
  const size_t need = classical_ws_bytes(cp, p, r) + align_up(cp.total * r * sizeof(double)) +
                      align_up(fit_rows * sizeof(int64_t)) * 2 +
                      align_up((size_t)(nj + 1) * sizeof(int64_t)) +
                      align_up((size_t)(npieces + 1) * sizeof(int64_t)) +
                      align_up((size_t)nj * r * r * sizeof(double)) +
                      align_up((size_t)nj * r * sizeof(double)) + align_up(nj * sizeof(double)) +
                      align_up(nj * sizeof(int32_t)) + align_up(dc_stitch_ws_bytes(npieces, r, cp.max_m)) + 4096;
  if ((rc = ws_reserve(h, need))) return rc;
  double* P = (double*)ws_alloc(h, cp.total * r * sizeof(double), st);
  if ((rc = run_classical(h, cp, data, dtype, ld, p, row_idx, r, P, estimates, gof, status, st)))
    return rc;
  int64_t* toff = (int64_t*)ws_alloc(h, (size_t)(npieces + 1) * sizeof(int64_t), st);
  double* rot = (double*)ws_alloc(h, (size_t)nj * r * r * sizeof(double), st);
  double* trans = (double*)ws_alloc(h, (size_t)nj * r * sizeof(double), st);
  if (nj > 0) {
    int64_t* trows = (int64_t*)ws_alloc(h, fit_rows * sizeof(int64_t), st);
    int64_t* srows = (int64_t*)ws_alloc(h, fit_rows * sizeof(int64_t), st);
    int64_t* joff = (int64_t*)ws_alloc(h, (size_t)(nj + 1) * sizeof(int64_t), st);
    double* loss = (double*)ws_alloc(h, nj * sizeof(double), st);
    int32_t* degen = (int32_t*)ws_alloc(h, nj * sizeof(int32_t), st);
    std::vector<int64_t> ht(fit_rows), hs(fit_rows), hj(nj + 1);
    for (int j = 0; j < nj; ++j) {
      hj[j] = (int64_t)j * c;
      for (int t = 0; t < c; ++t) {
        ht[(size_t)j * c + t] = t;                          // anchor: piece 1 rows 0..c-1
        hs[(size_t)j * c + t] = piece_off[j + 1] + t;       // piece j+1 connecting rows
      }
    }
    hj[nj] = (int64_t)nj * c;
    Stager sg(h, st);
    if ((rc = sg.begin(fit_rows * 16 + (nj + 1) * 8 + (npieces + 1) * 8 + 1024))) return rc;
    if ((rc = sg.put(trows, ht.data(), fit_rows * sizeof(int64_t)))) return rc;
    if ((rc = sg.put(srows, hs.data(), fit_rows * sizeof(int64_t)))) return rc;
    if ((rc = sg.put(joff, hj.data(), (nj + 1) * sizeof(int64_t)))) return rc;
    if ((rc = sg.put(toff, piece_off, (npieces + 1) * sizeof(int64_t)))) return rc;
    if ((rc = sg.end())) return rc;
    if ((rc = launch_procrustes_fit(h, P, trows, P, srows, joff, nj, r, rot, trans, loss, degen, st)))
      return rc;
  } else {
    Stager sg(h, st);
    if ((rc = sg.begin((npieces + 1) * 8))) return rc;
    if ((rc = sg.put(toff, piece_off, (npieces + 1) * sizeof(int64_t)))) return rc;
    if ((rc = sg.end())) return rc;
  }
  // stitch + final re-centring in one pass over P: the column mean comes from
  // per-piece sums of P pushed through each fit (no second pass over out)
  double* sws = rec ? (double*)ws_alloc(h, dc_stitch_ws_bytes(npieces, r, cp.max_m), st) : nullptr;
  if (rec && !sws) return MDSX_CUDA;
  return launch_dc_stitch(h, P, row_idx, toff, npieces, cp.max_m, c, r, rot, trans, out, st,
                          rec ? n : 0, sws);
}

int mdsx_interpolation(mdsx_handle* h, const void* data, int dtype, int64_t ld, int64_t n,
                       int32_t p, const int64_t* sample_idx, int64_t l, int32_t r, double* out,
                       double* estimates, double* gof, mdsx_piece_status* status, double* cond,
                       int32_t* flags, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  const int64_t off[2] = {0, l};
  ClassicalPlan cp;
  int rc = plan_classical(h, p, off, 1, r, cp);
  if (rc) return rc;
  const int64_t csz = mdsx_gower_context_size(l, p, r);
  const size_t need = classical_ws_bytes(cp, p, r) + align_up(l * r * sizeof(double)) +
                      align_up(csz * sizeof(double)) + recenter_ws_bytes(r) +
                      align_up(r * sizeof(double)) + 2048;
  if ((rc = ws_reserve(h, need))) return rc;
  double* base = (double*)ws_alloc(h, l * r * sizeof(double), st);
  if ((rc = run_classical(h, cp, data, dtype, ld, p, sample_idx, r, base, estimates, gof, status, st)))
    return rc;
  if (n <= l) {  // passthrough (algorithms.py:257-258): sample is 0..n-1
    return launch_scatter(h, base, sample_idx, l, r, out, st);
  }
  double* ctx = (double*)ws_alloc(h, csz * sizeof(double), st);
  int32_t* flag = flags;
  double* mean = ctx;
  double* M = mean + p;
  double* v = M + (int64_t)p * r;
  double* S = v + r;
  double* q = S + (int64_t)r * r;
  if ((rc = cuda_check(h, cudaMemsetAsync(flag, 0, 2 * sizeof(int32_t), st), "memset"))) return rc;
  if ((rc = launch_gower_context(h, data, dtype, ld, p, sample_idx, l, base, r, mean, M, v, S, q,
                                 cond, flag, st)))
    return rc;
  // dense rows: bulk-copy stream with fused per-CTA column sums, landmark
  // overwrite with a sum correction, one subtract pass (algorithms.py:264-274)
  double* part = (double*)ws_alloc(h, recenter_ws_bytes(r) + align_up(r * sizeof(double)), st);
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  if (ld == p && r <= 16 && ((size_t)p * es) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(data) & 15) == 0 && h->num_sms * r * sizeof(double) <= recenter_ws_bytes(r)) {
    int nparts = 0;
    // the landmark configuration is centred -> v ~ 0: fp32 norms are exact enough
    const bool n32 = dtype == MDSX_F32 && !getenv("MDSX_GOWER_NORM64");
    if ((rc = launch_gower_bulk(h, data, dtype, n, p, r, mean, M, v, out, part, flag + 1, &nparts,
                                st, n32)))
      return rc;
    const int lparts = (int)((l + 255) / 256);
    if (nparts > 0 && (size_t)(nparts + lparts) * r * sizeof(double) <= recenter_ws_bytes(r)) {
      // landmark overwrite: its per-CTA corrections are extra column-sum partials
      if ((rc = launch_landmark_overwrite(h, base, sample_idx, l, r, out,
                                          part + (size_t)nparts * r, st)))
        return rc;
      return launch_subtract_mean(h, out, n, r, part, nparts + lparts, nullptr, st);
    }
    if (nparts > 0) {             // too many landmarks for the partials buffer: rewrite by scatter
      if ((rc = launch_scatter(h, base, sample_idx, l, r, out, st))) return rc;
      return launch_recenter(h, out, n, r, part, st);
    }
  }
  if ((rc = launch_gower_affine(h, data, dtype, ld, n, p, r, mean, M, v, out, r, flag + 1, st)))
    return rc;
  if ((rc = launch_scatter(h, base, sample_idx, l, r, out, st))) return rc;
  if ((rc = launch_recenter(h, out, n, r, part, st))) return rc;
  return MDSX_OK;
}

}  // extern "C"

// fast_mds finish (algorithms.py:310-311, 341-342, 122-125): the shallowest
// level's in-place apply, the scatter to input order and the re-centring in
// one pass over P (mean from per-job sums pushed through each fit).
extern "C" int mdsx_fast_finish(mdsx_handle* h, const double* P, int32_t r, const int64_t* job_off,
                                int32_t njobs, const double* rot, const double* trans,
                                const int64_t* order, int64_t n, double* out, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (njobs < 1 || r < 1 || r > MDSX_MAX_R) return fail(h, MDSX_PARAM, "bad fast finish shape");
  if (job_off[0] != 0 || job_off[njobs] != n)
    return fail(h, MDSX_PARAM, "fast finish jobs must cover rows 0..n");
  int64_t max_m = 0;
  for (int j = 0; j < njobs; ++j) max_m = std::max<int64_t>(max_m, job_off[j + 1] - job_off[j]);
  const size_t need = align_up((size_t)(njobs + 1) * sizeof(int64_t)) +
                      align_up(dc_stitch_ws_bytes(njobs, r, max_m)) + 4096;
  int rc;
  if ((rc = ws_reserve(h, need))) return rc;
  int64_t* doff = (int64_t*)ws_alloc(h, (size_t)(njobs + 1) * sizeof(int64_t), st);
  double* sws = (double*)ws_alloc(h, dc_stitch_ws_bytes(njobs, r, max_m), st);
  if (!doff || !sws) return MDSX_CUDA;
  if ((rc = upload(h, doff, job_off, (size_t)(njobs + 1) * sizeof(int64_t), st))) return rc;
  return launch_dc_stitch(h, P, order, doff, njobs, max_m, 0, r, rot, trans, out, st, n, sws, 0);
}

extern "C" int mdsx_aligned_correlations(mdsx_handle* h, const double* points, int64_t n,
                                         int32_t r, const void* dominant, int32_t dtype,
                                         int64_t ld, double* corr, double* rotation,
                                         int32_t* zero_var, void* stream) {
  using namespace mdsx;
  if (!h) return MDSX_PARAM;
  if (r < 1 || r > 16) return fail(h, MDSX_UNSUPPORTED, "aligned correlations need 1 <= r <= 16");
  if (n < 2) return fail(h, MDSX_SHAPE, "need at least 2 rows");
  if (dtype != MDSX_F64 && dtype != MDSX_F32) return fail(h, MDSX_PARAM, "bad dtype");
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  const size_t nd = (size_t)corr_ws_doubles(n, r, h->num_sms);
  int rc = ws_reserve(h, align_up(nd * sizeof(double)) + 256);
  if (rc) return rc;
  double* part = (double*)ws_alloc(h, nd * sizeof(double), st);
  if (!part) return MDSX_CUDA;
  return launch_aligned_corr(h, points, n, r, dominant, dtype, ld, part, corr, rotation, zero_var,
                             st);
}

// fast_mds in one call (include/mdsx.h): see k_dcout.cu for the tail.
static int fast_impl(mdsx_handle* h, const void* data, int dtype, int64_t ld, int32_t p,
                     const mdsx_fast_plan* fp, int32_t r, int64_t n_out, int32_t recenter,
                     double* out, double* estimates, double* gof, mdsx_piece_status* status,
                     cudaStream_t st, const ContribGather* shard);

extern "C" int mdsx_fast_mds(mdsx_handle* h, const void* data, int dtype, int64_t ld, int32_t p,
                             const mdsx_fast_plan* fp, int32_t r, int64_t n_out, int32_t recenter,
                             double* out, double* estimates, double* gof, mdsx_piece_status* status,
                             void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  return fast_impl(h, data, dtype, ld, p, fp, r, n_out, recenter, out, estimates, gof, status, st,
                   nullptr);
}

extern "C" int mdsx_fast_mds_sharded(mdsx_handle* h, const void* data, int dtype, int64_t ld,
                                     int32_t p, const mdsx_fast_plan* fp, int32_t r, int64_t n_out,
                                     double* out, double* estimates, double* gof,
                                     mdsx_piece_status* status, int64_t n_total,
                                     int32_t nleaves_total, double* contrib_local,
                                     double* contrib_global, mdsx_gather_fn gather, void* ctx,
                                     void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (!fp || !contrib_local || !contrib_global || !gather || nleaves_total < fp->n_leaves ||
      n_total < n_out)
    return fail(h, MDSX_PARAM, "bad sharded fast arguments");
  const ContribGather ops{contrib_local, contrib_global, nleaves_total, n_total, gather, ctx};
  return fast_impl(h, data, dtype, ld, p, fp, r, n_out, 0, out, estimates, gof, status, st, &ops);
}

static int fast_impl(mdsx_handle* h, const void* data, int dtype, int64_t ld, int32_t p,
                     const mdsx_fast_plan* fp, int32_t r, int64_t n_out, int32_t recenter,
                     double* out, double* estimates, double* gof, mdsx_piece_status* status,
                     cudaStream_t st, const ContribGather* shard) {
  using namespace mdsx;
  if (!fp || fp->npieces < 2 || fp->n_leaves < 1 || fp->n_leaves >= fp->npieces || fp->nlevels < 1)
    return fail(h, MDSX_PARAM, "bad fast plan");
  const int np = fp->npieces, nl = fp->n_leaves, nal = np - nl, nlev = fp->nlevels;
  if (!dc_out_route_ok(data, dtype, ld, p, r, 1))
    return fail(h, MDSX_UNSUPPORTED, "fast route needs p <= 128, r <= 16 and 16-byte aligned rows");
  ClassicalPlan cp;
  int rc = plan_classical(h, p, fp->piece_off, np, r, cp);
  if (rc) return rc;
  for (int j = 0; j < nl; ++j)
    if (cp.pd[j].form != 0) return fail(h, MDSX_UNSUPPORTED, "fast route needs form-0 leaves");
  const int64_t leaf_total = fp->piece_off[nl] - fp->piece_off[0];
  const int64_t al_total = fp->piece_off[np] - fp->piece_off[nl];
  int64_t max_leaf = 0, max_al = 0;
  for (int j = 0; j < np; ++j)
    (j < nl ? max_leaf : max_al) = std::max<int64_t>(j < nl ? max_leaf : max_al, cp.pd[j].m);
  int64_t njobs = 0;
  for (int L = 0; L < nlev; ++L) njobs += fp->level_njobs[L];
  const int64_t ntrk = fp->ntracked;
  const size_t need = classical_ws_bytes(cp, p, r) + align_up(al_total * r * 8) +
                      align_up(points_ws_bytes(nal, max_al, r)) + align_up(nal * sizeof(PieceDesc)) +
                      align_up(ntrk * r * 8) + align_up(njobs * r * r * 8) + align_up(njobs * r * 8) * 2 +
                      align_up(njobs * 4) + align_up((njobs + nlev) * 8) + align_up(nlev * 8) +
                      align_up((size_t)nl * p * r * 8) + 2 * align_up((size_t)nl * r * 8) + 4096 * 4;
  if ((rc = ws_reserve(h, need))) return rc;
  ClassicalOut co;
  if ((rc = run_classical(h, cp, data, dtype, ld, p, fp->row_idx, r, nullptr, estimates, gof, status,
                          st, &co)))
    return rc;
  double* Pal = (double*)ws_alloc(h, al_total * r * 8, st);
  double2* cand = (double2*)ws_alloc(h, points_ws_bytes(nal, max_al, r), st);
  PieceDesc* dpd_al = (PieceDesc*)ws_alloc(h, nal * sizeof(PieceDesc), st);
  double* Ptrk = (double*)ws_alloc(h, std::max<int64_t>(ntrk, 1) * r * 8, st);
  double* rot = (double*)ws_alloc(h, njobs * r * r * 8, st);
  double* trans = (double*)ws_alloc(h, njobs * r * 8, st);
  double* loss = (double*)ws_alloc(h, njobs * 8, st);
  int32_t* degen = (int32_t*)ws_alloc(h, njobs * 4, st);
  int64_t* joff_d = (int64_t*)ws_alloc(h, (njobs + nlev) * 8, st);
  int64_t* jbase_d = (int64_t*)ws_alloc(h, nlev * 8, st);
  double* Uc = (double*)ws_alloc(h, (size_t)nl * p * r * 8, st);
  double* tvec = (double*)ws_alloc(h, (size_t)nl * r * 8, st);
  double* contrib = (double*)ws_alloc(h, (size_t)nl * r * 8, st);
  double* mean = (double*)ws_alloc(h, 64 * 8, st);
  if (!Pal || !cand || !dpd_al || !Ptrk || !rot || !trans || !loss || !degen || !joff_d || !jbase_d ||
      !Uc || !tvec || !contrib || !mean)
    return MDSX_CUDA;
  // alignment sets: full points with the canonical column signs (targets)
  std::vector<PieceDesc> al(cp.pd.begin() + nl, cp.pd.end());
  for (auto& d : al) d.pt_off -= leaf_total;
  std::vector<int64_t> jb(nlev), joff_all;
  {
    int64_t base = 0, ko = 0;
    for (int L = 0; L < nlev; ++L) {
      jb[L] = base;
      const int nj = fp->level_njobs[L];
      for (int t = 0; t <= nj; ++t) joff_all.push_back(fp->job_off[ko + t]);
      ko += nj + 1;
      base += nj;
    }
  }
  Stager sg(h, st);
  if ((rc = sg.begin(nal * sizeof(PieceDesc) + joff_all.size() * 8 + nlev * 8 + 1024))) return rc;
  if ((rc = sg.put(dpd_al, al.data(), nal * sizeof(PieceDesc)))) return rc;
  if ((rc = sg.put(joff_d, joff_all.data(), joff_all.size() * 8))) return rc;
  if ((rc = sg.put(jbase_d, jb.data(), nlev * 8))) return rc;
  if ((rc = sg.end())) return rc;
  if ((rc = launch_points(h, data, dtype, ld, p, fp->row_idx, dpd_al, nal, max_al, r, co.mu, co.U,
                          co.lam, Pal, cand, st, true)))
    return rc;
  // tracked rows in their leaves' frames, then level by level: fit, carry up
  if ((rc = launch_trk_points(h, data, dtype, ld, p, fp->trk_row, fp->trk_leaf, ntrk, co.dpd, r,
                              co.mu, co.U, Ptrk, st)))
    return rc;
  int64_t soff = 0, ko = 0;
  for (int L = 0; L < nlev; ++L) {
    const int nj = fp->level_njobs[L];
    const int64_t nsrc = fp->job_off[ko + nj] - fp->job_off[ko];
    if (nj > 0) {
      if ((rc = launch_procrustes_fit(h, Pal, fp->job_tgt + soff, Ptrk, fp->job_src + soff,
                                      joff_d + ko, nj, r, rot + jb[L] * r * r, trans + jb[L] * r,
                                      loss + jb[L], degen + jb[L], st)))
        return rc;
      if (L + 1 < nlev &&
          (rc = launch_trk_apply(h, Ptrk, fp->trk_job + (int64_t)L * ntrk, ntrk, r,
                                 rot + jb[L] * r * r, trans + jb[L] * r, st)))
        return rc;
    }
    soff += nsrc;
    ko += nj + 1;
  }
  return launch_fast_out(h, data, dtype, ld, p, fp->row_idx, fp->out_idx, co.dpd, nl, max_leaf, nlev,
                         fp->leaf_job, jbase_d, r, co.mu, co.U, rot, trans, Uc, tvec, contrib, mean,
                         recenter ? n_out : 0, out, st, shard);
}
