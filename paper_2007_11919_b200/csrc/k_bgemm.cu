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


// The narrow products of the block-Krylov cycle (C = alpha A B + beta D with
// N <= 16, A not transposed: Z = A Q, Q -= Q P, Y = Q S) stream A once and are
// HBM-bound (4 flop per byte of A), so the panels come through a 4-stage
// cp.async ring: per stage 128 rows x 16 columns of A (row-major, 16-byte
// copies, zero fill past M / K) and the 16 x 16 panel of B; one barrier per
// stage; 8 warps, each 16 rows x 16 columns (2 x 2 DMMA blocks).  Pitches of
// 20 doubles keep both fragment loads conflict-free.  Needs 16-byte aligned
// rows of B (even ldb); rows of A that are only 8-byte aligned (odd lda) are
// copied 8 bytes at a time.
// TA (op(A) = A^T, A stored K x M: the projections P = Q^T Z): the A panel is
// 16 k-rows x 128 m-columns, k-major as stored (pitch 132), so these long-K,
// few-tile products also keep three panels in flight instead of one.
constexpr int ST_BM = 128, ST_BN = 16, ST_KC = 16, ST_P = 20, ST_NS = 4, ST_PT = ST_BM + 4;

__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}

__device__ __forceinline__ void cp_async8_zfill(void* dst, const void* src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}

template <bool TA>
__global__ void __launch_bounds__(GT_THREADS, 2)
bgemm_stream_kernel(const GemmTask* __restrict__ tasks, const int4* __restrict__ items) {
  extern __shared__ __align__(16) double st_smem[];
  constexpr int SA = TA ? ST_KC * ST_PT : ST_BM * ST_P;   // doubles per A stage
  double* sA = st_smem;                                   // ST_NS x SA
  double* sB = sA + (size_t)ST_NS * SA;                   // ST_NS x ST_KC x ST_P
  const int4 it = items[blockIdx.x];
  const GemmTask t = tasks[it.x];
  if (t.skip && *t.skip) return;
  const int m0 = it.y * ST_BM, n0 = it.z * ST_BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = warp * 16;
  const int nch = (t.K + ST_KC - 1) / ST_KC;
  const bool a16 = TA || ((t.lda & 1) == 0 && (reinterpret_cast<uintptr_t>(t.A) & 15) == 0);
  auto issue = [&](int c) {
    if (c < nch) {
      const int s = c % ST_NS, k0 = c * ST_KC;
#pragma unroll
      for (int u = 0; u < ST_BM * 8 / GT_THREADS; ++u) {
        const int e = tid + GT_THREADS * u;
        if (TA) {
          const int kk = e >> 6, gm = m0 + 2 * (e & 63), gk = k0 + kk;
          const int nval = gk < t.K ? min(max(t.M - gm, 0), 2) : 0;
          const double* src = nval > 0 ? t.A + (int64_t)gk * t.lda + gm : t.A;
          cp_async16_zfill(sA + (size_t)s * SA + kk * ST_PT + 2 * (e & 63), src, 8 * nval);
        } else if (a16) {
          const int row = e >> 3, kf = k0 + 2 * (e & 7);
          const int gm = m0 + row;
          const int nval = gm < t.M ? min(max(t.K - kf, 0), 2) : 0;
          const double* src = nval > 0 ? t.A + (int64_t)gm * t.lda + kf : t.A;
          cp_async16_zfill(sA + (size_t)s * SA + row * ST_P + 2 * (e & 7), src, 8 * nval);
        } else {
          // rows of A only 8-byte aligned (odd lda): two 8-byte copies per segment
          const int row = e >> 3, gm = m0 + row;
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int kf = k0 + 2 * (e & 7) + h2;
            const bool live = gm < t.M && kf < t.K;
            const double* src = live ? t.A + (int64_t)gm * t.lda + kf : t.A;
            cp_async8_zfill(sA + (size_t)s * SA + row * ST_P + 2 * (e & 7) + h2, src, live ? 8 : 0);
          }
        }
      }
      if (tid < ST_KC * 8) {
        const int kk = tid >> 3, gn = n0 + 2 * (tid & 7);
        const int gk = k0 + kk;
        const int nval = gk < t.K ? min(max(t.N - gn, 0), 2) : 0;
        const double* src = nval > 0 ? t.B + (int64_t)gk * t.ldb + gn : t.B;
        cp_async16_zfill(sB + ((size_t)s * ST_KC + kk) * ST_P + 2 * (tid & 7), src, 8 * nval);
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int c = 0; c < ST_NS - 1; ++c) issue(c);
  for (int c = 0; c < nch; ++c) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(ST_NS - 2));
    __syncthreads();                 // panel c landed for everyone; stage (c - 1) % NS is free
    issue(c + ST_NS - 1);
    const double* a_s = sA + (size_t)(c % ST_NS) * SA +
                        (TA ? tig * ST_PT + wm + gid : (wm + gid) * ST_P + tig);
    const double* b_s = sB + ((size_t)(c % ST_NS) * ST_KC + tig) * ST_P + gid;
    const int nks = min(ST_KC / 4, (t.K - c * ST_KC + 3) >> 2);
#pragma unroll
    for (int ks = 0; ks < ST_KC / 4; ++ks) {
      if (ks >= nks) break;
      double af[2], bf[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = TA ? a_s[4 * ks * ST_PT + 8 * i] : a_s[8 * i * ST_P + 4 * ks];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = b_s[(size_t)4 * ks * ST_P + 8 * j];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int gm = m0 + wm + 8 * i + gid, gn = n0 + 8 * j + 2 * tig + v;
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
  if (b.narrow != 2 && !getenv("MDSX_BGEMM_NO_STREAM")) {
    // streamed panels (rows of A and B on 16-byte boundaries): the narrow
    // products, and every A^T B product (the Rayleigh-Ritz matrix H = Q^T Z is
    // tiled 128 x 16 too: its K loop is as long and as latency-bound)
    bool ok = true;
    for (const auto& t : batch) {
      ok = ok && t.transA == batch[0].transA && (t.ldb & 1) == 0 &&
           (reinterpret_cast<uintptr_t>(t.B) & 15) == 0;
      // A^T panels need 16-byte rows of A; A panels fall back to 8-byte copies in the kernel
      if (t.transA) ok = ok && (t.lda & 1) == 0 && (reinterpret_cast<uintptr_t>(t.A) & 15) == 0;
    }
    if (ok && batch[0].transA) b.narrow = 4;
    else if (ok && b.narrow == 1) b.narrow = 3;
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
    else if (b.narrow)     // 1, 3 or 4
      bgemm_kernel<128, 16><<<(unsigned)b.nitems, GT_THREADS, 0, st>>>(dev_tasks, dev_items + b.item_off);
    else
      bgemm_kernel<64, 64><<<(unsigned)b.nitems, GT_THREADS, 0, st>>>(dev_tasks, dev_items + b.item_off);
    return launched(h, "bgemm_kernel", st);
  }
  if (b.narrow == 3) {
    const size_t smem = (size_t)ST_NS * (ST_BM + ST_KC) * ST_P * sizeof(double);
    cudaFuncSetAttribute(bgemm_stream_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bgemm_stream_kernel<false><<<(unsigned)b.nitems, GT_THREADS, smem, st>>>(dev_tasks, dev_items + b.item_off);
    return launched(h, "bgemm_stream_kernel", st);
  }
  if (b.narrow == 4) {
    const size_t smem = (size_t)ST_NS * ST_KC * (ST_PT + ST_P) * sizeof(double);
    cudaFuncSetAttribute(bgemm_stream_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    bgemm_stream_kernel<true><<<(unsigned)b.nitems, GT_THREADS, smem, st>>>(dev_tasks, dev_items + b.item_off);
    return launched(h, "bgemm_stream_kernel", st);
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
