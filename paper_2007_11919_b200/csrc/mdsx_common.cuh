// Shared device helpers and the handle/workspace runtime of libmdsx.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/mdsx.h"

#define MDSX_MAX_R 32          // largest target dimension r handled in-kernel
#define MDSX_JACOBI_KMAX 112   // largest k for the shared-memory Jacobi solver

// ---------------------------------------------------------------- handle
struct mdsx_handle {
  int device = 0;
  int num_sms = 148;
  int max_smem_optin = 0;
  char* ws = nullptr;          // grow-only device workspace
  size_t ws_size = 0;
  size_t ws_top = 0;           // bump pointer for the current call
  char* pinned = nullptr;      // pinned host staging for small descriptor uploads
  size_t pinned_size = 0;
  cudaEvent_t pinned_free = nullptr;  // recorded after the last upload from `pinned`
  int64_t launches = 0;
  std::string err;
  // optional per-kernel CUDA-event timing (mdsx_timing_enable)
  bool timing = false;
  cudaEvent_t cur_start = nullptr;
  std::vector<cudaEvent_t> event_pool;
  std::vector<std::pair<const char*, std::pair<cudaEvent_t, cudaEvent_t>>> timed;
  std::vector<std::pair<std::string, std::pair<double, int64_t>>> report;
  // executed work credited to a kernel by its launcher (flops), reported
  // as the 4th column of mdsx_timing_report; only kernels whose work depends
  // on run-time iteration counts (block-Krylov products) record it
  std::vector<std::pair<std::string, double>> work;
  // second stream for the piece pipeline (run_classical), created on first use
  cudaStream_t aux = nullptr;
  // piece-pipeline chunk streams (equal priorities: giving the first chunk the
  // greatest priority measured 8% slower on dc2 / fast3)
  cudaStream_t pipe[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_pj[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_anchor = nullptr;   // D&C: anchor signs/targets ready (chunked tail)
  // calls are serialised per handle (the workspace and staging buffer are
  // shared): a call holds `mu`, makes its stream wait for the previous call's
  // last work (`ws_done`) and records `ws_done` on its stream when it returns,
  // so calls from several host threads or on several streams never overwrite
  // each other's descriptors or intermediates while those are in flight
  std::recursive_mutex mu;
  int depth = 0;
  cudaEvent_t ws_done = nullptr;
};

namespace mdsx {

// RAII guard opened by every C-ABI entry point that enqueues device work.
struct CallGuard {
  mdsx_handle* h;
  cudaStream_t st;
  std::unique_lock<std::recursive_mutex> lk;
  CallGuard(mdsx_handle* hh, cudaStream_t s) : h(hh), st(s), lk(hh->mu) {
    if (h->depth++ == 0 && h->ws_done) cudaStreamWaitEvent(st, h->ws_done, 0);
  }
  ~CallGuard() {
    if (--h->depth == 0) {
      if (!h->ws_done) cudaEventCreateWithFlags(&h->ws_done, cudaEventDisableTiming);
      cudaEventRecord(h->ws_done, st);
    }
  }
  CallGuard(const CallGuard&) = delete;
  CallGuard& operator=(const CallGuard&) = delete;
};
#define MDSX_GUARD(h, st)                                  \
  if (!(h)) return MDSX_PARAM;                             \
  ::mdsx::CallGuard mdsx_call_guard_((h), (st))

int fail(mdsx_handle* h, int code, const std::string& msg);
int cuda_check(mdsx_handle* h, cudaError_t e, const char* what);
// Begin a call: resets the bump allocator.  Workspace from a previous call on
// the same stream is safe to reuse (stream order).
void ws_reset(mdsx_handle* h);
// Reserve `bytes` (256-aligned) of device workspace; grows (after a device
// sync) when needed.  Returns nullptr and sets h->err on failure.
void* ws_alloc(mdsx_handle* h, size_t bytes, cudaStream_t st);
// (re)sizes the per-handle workspace for the current call (bump pointer reset)
int ws_reserve(mdsx_handle* h, size_t bytes);

// Sharded D&C / fast MDS: this call's per-piece (per-leaf) contributions to the
// column mean go to `local`; gather(ctx, stream) fills `global` with every
// rank's, in global piece order, on the call's stream; the mean is then taken
// over `total` pieces and n_total rows (distributed.py).
struct ContribGather {
  double* local;
  double* global;
  int32_t total;
  int64_t n_total;
  int (*gather)(void* ctx, void* stream);
  void* ctx;
};
// Upload a small host array via the pinned staging buffer (async on st).
int upload(mdsx_handle* h, void* dst, const void* src, size_t bytes, cudaStream_t st);
inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
cudaEvent_t pooled_event(mdsx_handle* h);
// Call immediately before a kernel launch on stream st.
inline void pre(mdsx_handle* h, cudaStream_t st) {
  if (h->timing) {
    h->cur_start = pooled_event(h);
    cudaEventRecord(h->cur_start, st);
  }
}
// Call immediately after a kernel launch on stream st.
inline int launched(mdsx_handle* h, const char* what, cudaStream_t st) {
  h->launches++;
  if (h->timing && h->cur_start) {
    cudaEvent_t e = pooled_event(h);
    cudaEventRecord(e, st);
    h->timed.push_back({what, {h->cur_start, e}});
    h->cur_start = nullptr;
  }
  return cuda_check(h, cudaGetLastError(), what);
}

// ------------------------------------------------------------ device helpers
template <typename T> __device__ __forceinline__ double ld_val(const T* p) {
  return static_cast<double>(__ldg(p));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Rutishauser/Golub-Van Loan symmetric 2x2 rotation zeroing a_pq.
__device__ __forceinline__ void sym_rotation(double app, double aqq, double apq,
                                             double& c, double& s, double& t) {
  double tau = (aqq - app) / (2.0 * apq);
  double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
  c = 1.0 / sqrt(1.0 + tt * tt);
  s = tt * c;
  t = tt;
}

}  // namespace mdsx

// ---------------------------------------------------------------- descriptors
// One classical-MDS piece.  form 0: A = Xc^T Xc (k = p);  form 1: A = Xc Xc^T (k = m).
struct PieceDesc {
  int64_t row_off;   // offset into row_idx
  int64_t a_off;     // offset (doubles) of the k x k matrix in the A workspace
  int64_t u_off;     // offset (doubles) of the k x r eigenvector block
  int64_t pt_off;    // offset (rows) of the m x r output block
  int32_t m, k, form, id;   // id: global piece index (output slot)
};

// Points epilogue of the Lanczos kernel (form-0 pieces, 16-byte aligned rows,
// r <= 10): after the eigenvectors, the same CTA streams the piece's rows and
// writes its signed points (points_stream.cuh); pending[id] = 0 marks pieces
// done, 1 the ones left to the separate points kernel (Jacobi fallback,
// non-finite input).
struct PtsEpi {
  const void* X;
  int f32;
  int64_t ld;
  int p;
  const int64_t* row_idx;
  const double* mu;
  double* points;
  int* pending;
};

// One batched-GEMM task: C = alpha * op(A) B + beta * D  (row-major, op(A) = A
// (M x K, lda) or A^T with A stored K x M); skipped when *skip != 0.
struct GemmTask {
  const double* A;
  const double* B;
  double* C;
  const double* D;
  const int* skip;
  int M, N, K;
  int lda, ldb, ldc, ldd;
  int transA;
  double alpha, beta;
};

struct GemmBatch {
  int64_t item_off, nitems;
  int narrow;
  int64_t task_off = 0, ntasks = 0;   // host bookkeeping (work accounting)
};

// Host launchers implemented in the kernel translation units.
namespace mdsx {
int launch_piece_means(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                       const int64_t* row_idx, const PieceDesc* pd, int npieces,
                       double* mu, mdsx_piece_status* status, cudaStream_t st);
int launch_gram(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                const int64_t* row_idx, const PieceDesc* pd, const double* mu,
                const int4* tiles, int ntiles, double* A, cudaStream_t st);
int launch_jacobi(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r, double* A,
                  double* U, double* lam, double* estimates, double* gof,
                  mdsx_piece_status* status, int qform_trivial, cudaStream_t st);
size_t points_ws_bytes(int npieces, int64_t max_m, int r);
int launch_points(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                  const int64_t* row_idx, const PieceDesc* pd, int npieces, int64_t max_m, int r,
                  const double* mu, const double* U, const double* lam, double* points,
                  double2* cand, cudaStream_t st, bool all_form0 = false,
                  const int* pending = nullptr);
GemmBatch append_bgemm(std::vector<GemmTask>& tasks, std::vector<int4>& items,
                       const std::vector<GemmTask>& batch);
int launch_bgemm(mdsx_handle* h, const GemmTask* dev_tasks, const int4* dev_items,
                 const GemmBatch& b, cudaStream_t st);
}  // namespace mdsx
