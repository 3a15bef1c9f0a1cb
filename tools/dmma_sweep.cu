// DMMA m8n8k4 throughput on one B200 as a function of warps per scheduler and
// independent accumulators per warp (ILP), and with fresh operands loaded from
// shared memory each step (the Gram kernel's pattern).  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_sweep tools/dmma_sweep.cu && /tmp/dmma_sweep
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dmma_ilp(double* out, int iters) {
  double acc[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i][0] = acc[i][1] = 0.0;
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// NB fragments loaded from smem per k-step, NB*(NB+1)/2/Q DMMAs per warp (Gram pattern)
template <int NB, int NP>
__global__ void dmma_lds(double* out, int iters) {
  __shared__ double st[32 * 108];
  for (int i = threadIdx.x; i < 32 * 108; i += blockDim.x) st[i] = i * 1e-6;
  __syncthreads();
  const int lane = threadIdx.x & 31, gid = lane >> 2, tig = lane & 3;
  double acc[NP][2];
#pragma unroll
  for (int i = 0; i < NP; ++i) acc[i][0] = acc[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
    const double* src = st + ((it & 7) * 4 + tig) * 108 + gid;
    double f[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) f[b] = src[8 * b];
#pragma unroll
    for (int u = 0; u < NP; ++u)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[u][0]), "+d"(acc[u][1]) : "d"(f[u % NB]), "d"(f[(u * 7) % NB]));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NP; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static double run(void (*k)(double*, int), int blocks, int threads, int iters, int dmma_per_iter,
                  double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<blocks, threads>>>(out, iters / 10);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 256 * dmma_per_iter * (double)iters * blocks * (threads / 32);
  return fl / ms / 1e9;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, sizeof(double) * sms * 64 * 1024);
  const int it = 4000;
  printf("warps/SMSP  ILP=1   ILP=2   ILP=4   ILP=8   ILP=16  ILP=23 (TFLOP/s)\n");
  for (int w = 1; w <= 8; w *= 2) {
    const int thr = 128 * w;
    printf("%9d  %6.2f  %6.2f  %6.2f  %6.2f  %6.2f  %6.2f\n", w,
           run(dmma_ilp<1>, sms, thr, it * 8, 1, out), run(dmma_ilp<2>, sms, thr, it * 4, 2, out),
           run(dmma_ilp<4>, sms, thr, it * 2, 4, out), run(dmma_ilp<8>, sms, thr, it, 8, out),
           run(dmma_ilp<16>, sms, thr, it / 2, 16, out), run(dmma_ilp<23>, sms, thr, it / 2, 23, out));
  }
  printf("Gram pattern (13 LDS + 23 DMMA per warp-step):\n");
  for (int w = 1; w <= 4; w *= 2)
    printf("  warps/SMSP %d: %6.2f TFLOP/s\n", w, run(dmma_lds<13, 23>, sms, 128 * w, it, 23, out));
  printf("  (8 LDS + 12 DMMA) warps/SMSP 2: %6.2f  4: %6.2f\n", run(dmma_lds<8, 12>, sms, 256, it, 12, out),
         run(dmma_lds<8, 12>, sms, 512, it, 12, out));
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
