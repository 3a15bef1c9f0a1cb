// Batched fp64 GEMM for the block-Krylov eigensolver of large pieces:
//   C_t = alpha * op(A_t) * B_t + beta * D_t      (op(A) = A or A^T)
// over a host-built list of (task, row-tile, col-tile) work items.  fp64 FMA
// in registers, 16 x 16 thread grid, operand panels staged in shared memory;
// fixed reduction order (deterministic).
#include "mdsx_common.cuh"

#include <cstdlib>
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


__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Same contract on the fp64 tensor pipe (DMMA m8n8k4): the CTA tile BM x BN is
// split over 8 warps in a (BM/WM) x (BN/WN) grid, each warp holding MI x NI
// 8x8 accumulator blocks; K staged BK at a time with register prefetch of the
// next panel; shared-memory pitches == 4 (mod 16) doubles make the fragment
// loads conflict-free.
template <int BM, int BN, int WM, int WN>
__global__ void __launch_bounds__(GT_THREADS)
bgemm_dmma_kernel(const GemmTask* __restrict__ tasks, const int4* __restrict__ items) {
  constexpr int MI = WM / 8, NI = WN / 8;
  constexpr int WGN = BN / WN;                       // warps along n
  constexpr int PA = BM + 4, PB = BN + 4;
  constexpr int EA = BK * BM / GT_THREADS, EB = (BK * BN + GT_THREADS - 1) / GT_THREADS;
  __shared__ __align__(16) double sa[BK][PA];
  __shared__ __align__(16) double sb[BK][PB];
  const int4 it = items[blockIdx.x];
  const GemmTask t = tasks[it.x];
  if (t.skip && *t.skip) return;
  const int m0 = it.y * BM, n0 = it.z * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = (warp / WGN) * WM, wn = (warp % WGN) * WN;
  double acc[MI][NI][2];
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double pa[EA], pb[EB];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int q = 0; q < EA; ++q) {
      const int e = tid + q * GT_THREADS;
      int kk, mm;
      if (t.transA) { kk = e / BM; mm = e % BM; }
      else { mm = e / BK; kk = e % BK; }
      const int gm = m0 + mm, gk = k0 + kk;
      pa[q] = (gm < t.M && gk < t.K)
                  ? (t.transA ? t.A[(int64_t)gk * t.lda + gm] : t.A[(int64_t)gm * t.lda + gk])
                  : 0.0;
    }
#pragma unroll
    for (int q = 0; q < EB; ++q) {
      const int e = tid + q * GT_THREADS;
      const int kk = e / BN, nn = e % BN;
      const int gk = k0 + kk, gn = n0 + nn;
      pb[q] = (e < BK * BN && gk < t.K && gn < t.N) ? t.B[(int64_t)gk * t.ldb + gn] : 0.0;
    }
  };
  auto stash = [&]() {
#pragma unroll
    for (int q = 0; q < EA; ++q) {
      const int e = tid + q * GT_THREADS;
      int kk, mm;
      if (t.transA) { kk = e / BM; mm = e % BM; }
      else { mm = e / BK; kk = e % BK; }
      sa[kk][mm] = pa[q];
    }
#pragma unroll
    for (int q = 0; q < EB; ++q) {
      const int e = tid + q * GT_THREADS;
      if (e < BK * BN) sb[e / BN][e % BN] = pb[q];
    }
  };
  fetch(0);
  for (int k0 = 0; k0 < t.K; k0 += BK) {
    stash();
    __syncthreads();
    if (k0 + BK < t.K) fetch(k0 + BK);              // next panel in flight during the DMMAs
#pragma unroll
    for (int ks = 0; ks < BK / 4; ++ks) {
      double af[MI], bf[NI];
#pragma unroll
      for (int i = 0; i < MI; ++i) af[i] = sa[4 * ks + tig][wm + 8 * i + gid];
#pragma unroll
      for (int j = 0; j < NI; ++j) bf[j] = sb[4 * ks + tig][wn + 8 * j + gid];
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NI; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < MI; ++i)
#pragma unroll
    for (int j = 0; j < NI; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int gm = m0 + wm + 8 * i + gid, gn = n0 + wn + 8 * j + 2 * tig + v;
        if (gm < t.M && gn < t.N) {
          const double dv = t.beta == 0.0 ? 0.0 : t.beta * t.D[(int64_t)gm * t.ldd + gn];
          t.C[(int64_t)gm * t.ldc + gn] = fma(t.alpha, acc[i][j][v], dv);
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
  b.task_off = (int64_t)tasks.size();
  b.ntasks = (int64_t)batch.size();
  if (batch.empty()) return b;
  b.narrow = batch[0].N <= 16 ? 1 : 0;
  if (b.narrow) {
    // few large-M tasks (e.g. the single landmark piece of interpolation):
    // 32-row tiles so the product spreads over 4x more CTAs
    int64_t tiles128 = 0;
    for (const auto& t : batch) tiles128 += (t.M + 127) / 128;
    if (tiles128 < 64 && !getenv("MDSX_BGEMM_NO_SMALL")) b.narrow = 2;
  }
  const int BM = b.narrow == 2 ? 32 : b.narrow ? 128 : 64, BN = b.narrow ? 16 : 64;
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
  if (getenv("MDSX_BGEMM_FMA")) {                 // the CUDA-core variant, for comparison
    if (b.narrow == 2)
      bgemm_kernel<32, 16><<<(unsigned)b.nitems, GT_THREADS, 0, st>>>(dev_tasks, dev_items + b.item_off);
    else if (b.narrow)
      bgemm_kernel<128, 16><<<(unsigned)b.nitems, GT_THREADS, 0, st>>>(dev_tasks, dev_items + b.item_off);
    else
      bgemm_kernel<64, 64><<<(unsigned)b.nitems, GT_THREADS, 0, st>>>(dev_tasks, dev_items + b.item_off);
    return launched(h, "bgemm_kernel", st);
  }
  if (b.narrow == 2)
    bgemm_dmma_kernel<32, 16, 8, 8><<<(unsigned)b.nitems, GT_THREADS, 0, st>>>(dev_tasks, dev_items + b.item_off);
  else if (b.narrow)
    bgemm_dmma_kernel<128, 16, 16, 16><<<(unsigned)b.nitems, GT_THREADS, 0, st>>>(dev_tasks, dev_items + b.item_off);
  else
    bgemm_dmma_kernel<64, 64, 32, 16><<<(unsigned)b.nitems, GT_THREADS, 0, st>>>(dev_tasks, dev_items + b.item_off);
  return launched(h, "bgemm_dmma_kernel", st);
}

}  // namespace mdsx
