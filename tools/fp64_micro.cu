// Microbenchmark: FP64 FMA (CUDA cores), DMMA m8n8k4 (fp64 tensor) and
// F2F.F64.F32 conversion throughput on one B200.  Build + run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_micro tools/fp64_micro.cu && /tmp/fp64_micro
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[4][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
  double s = 0;
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void mixed_kernel(double* out, int iters) {
  double acc[4][2] = {};
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double f[8];
  for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(a), "d"(b));
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = fma(f[i], b, 1e-9);
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  for (int i = 0; i < 8; ++i) s += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dfma2_kernel(double* out, int iters) {
  double b = 1.0 + threadIdx.x * 1e-4;
  double f[8];
  for (int i = 0; i < 8; ++i) f[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) f[i] = fma(f[i], b, 1e-9);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += f[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void f2f_kernel(double* out, const float* in, int iters) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = in[i] + threadIdx.x;
  double s[8] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      s[i] += (double)x[i];
      x[i] = __int_as_float(__float_as_int(x[i]) ^ 1);
    }
  double t = 0;
  for (int i = 0; i < 8; ++i) t += s[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  float* in; cudaMalloc(&in, 64); cudaMemset(in, 0, 64);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0);
    dfma_kernel<<<sms * 4, 512>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)sms * 4 * 512;
    printf("DFMA: %.2f TFLOP/s %.3f ms (%.1f FMA/clk/SM at 1965 MHz)\n", fl / ms / 1e9, ms,
           fl / 2 / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0);
    dmma_kernel<<<sms * 4, 512>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 4 * iters * (double)sms * 4 * 512 / 32;
    printf("DMMA: %.2f TFLOP/s  %.3f ms\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0);
    mixed_kernel<<<sms * 4, 512>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("mixed 4 DMMA + 8 DFMA per iter: %.3f ms (DMMA-only %.3f-equivalent work)\n", ms, 0.0);
    cudaEventRecord(e0);
    dfma2_kernel<<<sms * 4, 512>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    printf("dfma2 (8 DFMA/iter, register b): %.3f ms\n", ms);
    cudaEventRecord(e0);
    f2f_kernel<<<sms * 4, 512>>>(out, in, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
    double cv = 8.0 * iters * (double)sms * 4 * 512;
    printf("F2F+DADD: %.1f conv/clk/SM\n", cv / (ms * 1e-3) / sms / 1.965e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
