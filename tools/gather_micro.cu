// Random-row gather bandwidth on one B200: rows of an n x p fp64 matrix read
// in a random permutation (the D&C / fast MDS piece access pattern), three
// ways, against a sequential read of the same bytes.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gather_micro tools/gather_micro.cu && /tmp/gather_micro
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
#include "../paper_2007_11919_b200/csrc/bulk.cuh"

// one warp per row, coalesced 16-byte loads, 8 rows in flight per warp
__global__ void gather_warp(const double* __restrict__ X, int p, const int64_t* __restrict__ idx,
                            int64_t n, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  const int q = p / 2;
  for (int64_t r0 = w * 8; r0 < n; r0 += nw * 8) {
    double2 v[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t r = r0 + u;
      const double2* row = reinterpret_cast<const double2*>(X + (r < n ? idx[r] : 0) * p);
      v[u][0] = lane < q ? __ldg(row + lane) : make_double2(0, 0);
      v[u][1] = lane + 32 < q ? __ldg(row + lane + 32) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u][0].x + v[u][0].y + v[u][1].x + v[u][1].y;
  }
  if (acc == 12345.678) out[0] = acc;
}

// sequential: same loads, identity index
__global__ void seq_warp(const double* __restrict__ X, int p, int64_t n, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc = 0.0;
  const int q = p / 2;
  for (int64_t r0 = w * 8; r0 < n; r0 += nw * 8) {
    double2 v[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t r = r0 + u < n ? r0 + u : 0;
      const double2* row = reinterpret_cast<const double2*>(X + r * p);
      v[u][0] = lane < q ? __ldg(row + lane) : make_double2(0, 0);
      v[u][1] = lane + 32 < q ? __ldg(row + lane + 32) : make_double2(0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u][0].x + v[u][0].y + v[u][1].x + v[u][1].y;
  }
  if (acc == 12345.678) out[0] = acc;
}


// TMA ring: a producer warp issues one cp.async.bulk per row (lane = row) into
// NS stages of 32 rows; consumer warps only release stages (data-movement rate)
template <int NS, int NC>
__global__ void gather_tma(const double* __restrict__ X, int p, const int64_t* __restrict__ idx,
                           int64_t n, int64_t rows_per_cta, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + NS;
  double* stage = reinterpret_cast<double*>(sm + 256);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r_begin = blockIdx.x * rows_per_cta;
  const int64_t r_end = min(n, r_begin + rows_per_cta);
  const int nch = (int)((r_end - r_begin + 31) / 32);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) { bulk::bar_init(&full[s], 1); bulk::bar_init(&empty[s], NC); }
    bulk::bar_fence();
  }
  __syncthreads();
  double acc = 0.0;
  if (warp == NC) {
    for (int c = 0; c < nch; ++c) {
      const int s = c % NS;
      if (c >= NS) bulk::wait(&empty[s], (unsigned)((c / NS - 1) & 1));
      const int64_t r0 = r_begin + 32 * c;
      const int nr = (int)min((int64_t)32, r_end - r0);
      const int64_t gi = lane < nr ? idx[r0 + lane] : 0;
      if (lane == 0) bulk::arrive_expect(&full[s], (unsigned)(nr * p * 8));
      __syncwarp();
      if (lane < nr) bulk::copy(stage + (size_t)s * 32 * p + lane * p, X + gi * p, p * 8, &full[s]);
    }
  } else {
    for (int c = 0; c < nch; ++c) {
      const int s = c % NS;
      bulk::wait(&full[s], (unsigned)((c / NS) & 1));
      acc += stage[(size_t)s * 32 * p + lane];
      __syncwarp();
      if (lane == 0) bulk::arrive(&empty[s]);
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const int64_t n = 1000000;
  const int p = 100;
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* X;
  int64_t* idx;
  double* out;
  cudaMalloc(&X, n * p * sizeof(double));
  cudaMalloc(&idx, n * sizeof(int64_t));
  cudaMalloc(&out, 64);
  cudaMemset(X, 0, n * p * sizeof(double));
  std::vector<int64_t> h(n);
  for (int64_t i = 0; i < n; ++i) h[i] = i;
  std::shuffle(h.begin(), h.end(), std::mt19937_64(1));
  cudaMemcpy(idx, h.data(), n * 8, cudaMemcpyHostToDevice);
  std::vector<int64_t> hs(h);                    // sorted within 1000-row pieces
  for (int64_t i = 0; i < n; i += 1000) std::sort(hs.begin() + i, hs.begin() + std::min(n, i + 1000));
  int64_t* idx_s;
  cudaMalloc(&idx_s, n * 8);
  cudaMemcpy(idx_s, hs.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)n * p * 8;
  for (int wpb : {8, 16, 32}) {
    for (int bps : {2, 4, 8}) {
      const int blocks = sms * bps, thr = 32 * wpb;
      float ms[3];
      for (int k = 0; k < 3; ++k) {
        for (int rep = 0; rep < 2; ++rep) {
          cudaEventRecord(e0);
          if (k == 0) gather_warp<<<blocks, thr>>>(X, p, idx, n, out);
          else if (k == 1) gather_warp<<<blocks, thr>>>(X, p, idx_s, n, out);
          else seq_warp<<<blocks, thr>>>(X, p, n, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms[k], e0, e1);
        }
      }
      printf("warps/CTA %2d CTAs/SM %d: random %.0f GB/s  sorted-in-piece %.0f GB/s  sequential %.0f GB/s\n",
             wpb, bps, bytes / ms[0] / 1e6, bytes / ms[1] / 1e6, bytes / ms[2] / 1e6);
    }
  }
  auto tma = [&](auto kern, int ns, int cps) {
    const size_t smem = 256 + (size_t)ns * 32 * p * 8;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int blocks = sms * cps;
    const int64_t rpc = (n + blocks - 1) / blocks;
    float ms = 0;
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      kern<<<blocks, 32 * 5, smem>>>(X, p, idx, n, rpc, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
    }
    printf("TMA ring NS=%d CTAs/SM=%d: %.0f GB/s (%s)\n", ns, cps, bytes / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  tma(gather_tma<2, 4>, 2, 2);
  tma(gather_tma<4, 4>, 4, 2);
  tma(gather_tma<2, 4>, 2, 4);
  tma(gather_tma<3, 4>, 3, 3);
  tma(gather_tma<8, 4>, 8, 1);
  tma(gather_tma<2, 4>, 2, 8);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
