// Batched fp64 GEMM for the block-Krylov eigensolver of large pieces:
//   C_t = alpha * op(A_t) * B_t + beta * D_t      (op(A) = A or A^T)
// over a host-built list of (task, row-tile, col-tile) work items.  fp64 FMA
// in registers, 16 x 16 thread grid, operand panels staged in shared memory;
// fixed reduction order (deterministic).
#include "mdsx_common.cuh"

#include <vector>

namespace {

constexpr int BK = 16;
constexpr int GT_THREADS = 256;

template <int BM, int BN>
__global__ void __launch_bounds__(GT_THREADS)
bgemm_kernel(const GemmTask* __restrict__ tasks, const int4* __restrict__ items) {
  constexpr int TM = BM / 16, TN = BN / 16;
  __shared__ double sa[BK][BM + 1];
  __shared__ double sb[BK][BN + 1];
  const int4 it = items[blockIdx.x];
  const GemmTask t = tasks[it.x];
  if (t.skip && *t.skip) return;
  const int m0 = it.y * BM, n0 = it.z * BN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[TM][TN];
#pragma unroll
  for (int u = 0; u < TM; ++u)
#pragma unroll
    for (int v = 0; v < TN; ++v) acc[u][v] = 0.0;
  for (int k0 = 0; k0 < t.K; k0 += BK) {
    for (int e = threadIdx.x; e < BK * BM; e += GT_THREADS) {
      int kk, mm;
      if (t.transA) { kk = e / BM; mm = e % BM; }     // stored K x M: contiguous in m
      else { mm = e / BK; kk = e % BK; }              // stored M x K: contiguous in k
      const int gm = m0 + mm, gk = k0 + kk;
      double v = 0.0;
      if (gm < t.M && gk < t.K)
        v = t.transA ? t.A[(int64_t)gk * t.lda + gm] : t.A[(int64_t)gm * t.lda + gk];
      sa[kk][mm] = v;
    }
    for (int e = threadIdx.x; e < BK * BN; e += GT_THREADS) {
      const int kk = e / BN, nn = e % BN;
      const int gk = k0 + kk, gn = n0 + nn;
      sb[kk][nn] = (gk < t.K && gn < t.N) ? t.B[(int64_t)gk * t.ldb + gn] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double a[TM], b[TN];
#pragma unroll
      for (int u = 0; u < TM; ++u) a[u] = sa[kk][ty + 16 * u];
#pragma unroll
      for (int v = 0; v < TN; ++v) b[v] = sb[kk][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < TM; ++u)
#pragma unroll
        for (int v = 0; v < TN; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < TM; ++u)
#pragma unroll
    for (int v = 0; v < TN; ++v) {
      const int gm = m0 + ty + 16 * u, gn = n0 + tx + 16 * v;
      if (gm < t.M && gn < t.N) {
        const double dv = t.beta == 0.0 ? 0.0 : t.beta * t.D[(int64_t)gm * t.ldd + gn];
        t.C[(int64_t)gm * t.ldc + gn] = fma(t.alpha, acc[u][v], dv);
      }
    }
}

}  // namespace

namespace mdsx {

// Append one batched GEMM (one task per item of `batch`) to the global task /
// work-item lists; returns the launch record.  All tasks of a batch share the
// tile shape (narrow = N <= 16).
GemmBatch append_bgemm(std::vector<GemmTask>& tasks, std::vector<int4>& items,
                       const std::vector<GemmTask>& batch) {
  GemmBatch b{(int64_t)items.size(), 0, 0};
  if (batch.empty()) return b;
  b.narrow = batch[0].N <= 16 ? 1 : 0;
  const int BM = b.narrow ? 128 : 64, BN = b.narrow ? 16 : 64;
  for (const auto& t : batch) {
    const int id = (int)tasks.size();
    tasks.push_back(t);
    const int tm = (t.M + BM - 1) / BM, tn = (t.N + BN - 1) / BN;
    for (int a = 0; a < tm; ++a)
      for (int c = 0; c < tn; ++c) items.push_back(make_int4(id, a, c, 0));
  }
  b.nitems = (int64_t)items.size() - b.item_off;
  return b;
}

int launch_bgemm(mdsx_handle* h, const GemmTask* dev_tasks, const int4* dev_items,
                 const GemmBatch& b, cudaStream_t st) {
  if (b.nitems == 0) return MDSX_OK;
  mdsx::pre(h, st);
  if (b.narrow)
    bgemm_kernel<128, 16><<<(unsigned)b.nitems, GT_THREADS, 0, st>>>(dev_tasks, dev_items + b.item_off);
  else
    bgemm_kernel<64, 64><<<(unsigned)b.nitems, GT_THREADS, 0, st>>>(dev_tasks, dev_items + b.item_off);
  return launched(h, "bgemm_kernel", st);
}

}  // namespace mdsx
