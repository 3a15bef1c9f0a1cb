// Host->device transfer of n x p fp64 rows in a random row order (the D&C plan
// order) on one B200: (a) a zero-copy gather kernel reading page-locked host
// rows over PCIe, (b) a sequential cudaMemcpyAsync of the same bytes.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/zc tools/zc_micro.cu && /tmp/zc
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__global__ void zc_gather(const double* __restrict__ src, int p, const int64_t* __restrict__ order,
                          int64_t n, double* __restrict__ dst, int rows_per_warp) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int q = p / 2;
  for (int64_t r0 = w * rows_per_warp; r0 < n; r0 += nw * rows_per_warp) {
    double2 v[8][2];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (u < rows_per_warp && r0 + u < n) {
        const double2* row = reinterpret_cast<const double2*>(src + order[r0 + u] * p);
        v[u][0] = lane < q ? row[lane] : make_double2(0, 0);
        v[u][1] = lane + 32 < q ? row[lane + 32] : make_double2(0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (u < rows_per_warp && r0 + u < n) {
        double2* d = reinterpret_cast<double2*>(dst + (r0 + u) * p);
        if (lane < q) d[lane] = v[u][0];
        if (lane + 32 < q) d[lane + 32] = v[u][1];
      }
    }
  }
}

int main() {
  const int64_t n = 1000000;
  const int p = 100;
  const size_t bytes = (size_t)n * p * 8;
  double *h, *d;
  int64_t* ord;
  cudaHostAlloc(&h, bytes, cudaHostAllocDefault);
  cudaMalloc(&d, bytes);
  cudaMalloc(&ord, n * 8);
  for (size_t i = 0; i < (size_t)n * p; ++i) h[i] = (double)i;
  std::vector<int64_t> o(n);
  for (int64_t i = 0; i < n; ++i) o[i] = i;
  std::shuffle(o.begin(), o.end(), std::mt19937_64(1));
  cudaMemcpy(ord, o.data(), n * 8, cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  printf("sequential cudaMemcpyAsync (pinned): %.2f ms  %.1f GB/s\n", ms, bytes / ms / 1e6);
  for (int blocksm : {1, 2, 4, 8})
    for (int rpw : {1, 4, 8}) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        zc_gather<<<sms * blocksm, 256>>>(h, p, ord, n, d, rpw);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
      }
      std::vector<double> chk(p);
      cudaMemcpy(chk.data(), d + 12345 * p, p * 8, cudaMemcpyDeviceToHost);
      const bool ok = chk[3] == (double)(o[12345] * p + 3);
      printf("zero-copy gather CTAs/SM %d rows/warp %d: %.2f ms  %.1f GB/s %s\n", blocksm, rpw, ms,
             bytes / ms / 1e6, ok ? "ok" : "WRONG");
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
