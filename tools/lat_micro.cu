// Dependent-chain latencies on one thread (clock64): DFMA, DADD, F2F f64<->f32,
// MUFU.RCP + Newton (fast_rcp), DDIV, DSQRT, LDS.64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lat tools/lat_micro.cu && /tmp/lat
#include <cstdio>
__device__ __forceinline__ double fast_rcp(double d) {
  double r = (double)__frcp_rn((float)d);
  r = r * fma(-d, r, 2.0);
  r = r * fma(-d, r, 2.0);
  return r;
}
__global__ void lat(double* out, long long* t, double seed) {
  __shared__ double sm[64];
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
  __syncthreads();
  const int N = 1000;
  double x = seed;
  long long t0 = clock64();
  for (int i = 0; i < N; ++i) x = fma(x, 1.0000001, 1e-9);
  long long t1 = clock64();
  for (int i = 0; i < N; ++i) x = fast_rcp(x + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < N; ++i) x = 1.0 / (x + 1.0);
  long long t3 = clock64();
  for (int i = 0; i < N; ++i) x = sqrt(x + 1.0);
  long long t4 = clock64();
  int idx = 0;
  for (int i = 0; i < N; ++i) { x += sm[idx]; idx = ((int)x) & 31; }
  long long t5 = clock64();
  for (int i = 0; i < N; ++i) x = (double)(float)x + 1e-3;
  long long t6 = clock64();
  out[threadIdx.x] = x;
  t[0] = (t1 - t0) / N; t[1] = (t2 - t1) / N; t[2] = (t3 - t2) / N; t[3] = (t4 - t3) / N;
  t[4] = (t5 - t4) / N; t[5] = (t6 - t5) / N;
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 1024); cudaMallocManaged(&t, 64);
  lat<<<1, 1>>>(o, t, 0.5); cudaDeviceSynchronize();
  lat<<<1, 1>>>(o, t, 0.5); cudaDeviceSynchronize();
  printf("clk per dependent op: DFMA %lld | fast_rcp(+DADD) %lld | DDIV(+DADD) %lld | DSQRT(+DADD) %lld | LDS+DADD+cvt %lld | F2F d->f->d + DADD %lld\n",
         t[0], t[1], t[2], t[3], t[4], t[5]);
  return 0;
}
