// Column compaction for wide inputs.  A column that is zero in every row of
// the data matrix (the always-blank border pixels of image data: 280 of 784 in
// config 5) contributes exactly zero to every piece's centred Gram, to the
// eigenvector entries, the piece means, the points X~U and the Gower terms, so
// the algorithms run unchanged -- and produce the same configuration -- on the
// matrix of the active columns (algorithms.py:115-119 sees the full matrix;
// the arithmetic differs only in the order of exact-zero terms).  One pass
// finds the active columns (mdsx_active_columns), a second gathers them into
// a dense row-major copy (mdsx_gather_columns); the k x k Gram, the Krylov
// products and their traffic then shrink by (active / p)^2.
#include "mdsx_common.cuh"

#include <algorithm>
#include <vector>

namespace {

// Dense rows (ld == p): the matrix is a flat array of 16-byte vectors and the
// grid-stride step is a multiple of the vectors per row, so every thread
// visits one fixed column group and keeps its flags in registers; four loads
// in flight per thread.
template <typename T>
__global__ void __launch_bounds__(256)
nonzero_cols_flat_kernel(const T* __restrict__ X, int64_t nvec, int vpr, int64_t step,
                         int* __restrict__ flags) {
  using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
  constexpr int VW = 16 / sizeof(T);
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t0 >= step) return;
  const V* xv = reinterpret_cast<const V*>(X);
  bool nz[VW];
#pragma unroll
  for (int u = 0; u < VW; ++u) nz[u] = false;
  for (int64_t v0 = t0; v0 < nvec; v0 += 4 * step) {
    V w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) w[q] = v0 + q * step < nvec ? xv[v0 + q * step] : V{};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const T* e = reinterpret_cast<const T*>(&w[q]);
#pragma unroll
      for (int u = 0; u < VW; ++u) nz[u] |= !(e[u] == T(0));   // NaN counts as active
    }
  }
  const int g = (int)(t0 % vpr);
#pragma unroll
  for (int u = 0; u < VW; ++u)
    if (nz[u]) atomicOr(flags + g * VW + u, 1);
}

// general rows: a warp per row, lanes over the columns
template <typename T>
__global__ void __launch_bounds__(256)
nonzero_cols_kernel(const T* __restrict__ X, int64_t ld, int64_t n, int p, int* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w; i < n; i += nw)
    for (int c = lane; c < p; c += 32)
      if (!(X[i * ld + c] == T(0))) atomicOr(flags + c, 1);
}

// out[i][j] = X[i][cols[j]] (j < pa), 0 for pa <= j < ldo: the column list in
// shared memory, 4 rows per CTA iteration, threads over the columns
template <typename T>
__global__ void __launch_bounds__(256)
gather_cols_kernel(const T* __restrict__ X, int64_t ld, int64_t n, const int32_t* __restrict__ cols,
                   int pa, int ldo, T* __restrict__ out) {
  extern __shared__ int scols[];
  for (int j = threadIdx.x; j < ldo; j += blockDim.x) scols[j] = j < pa ? cols[j] : -1;
  __syncthreads();
  for (int64_t i0 = (int64_t)blockIdx.x * 4; i0 < n; i0 += (int64_t)gridDim.x * 4)
    for (int j = threadIdx.x; j < ldo; j += blockDim.x) {
      const int c = scols[j];
      T v[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) v[q] = (c >= 0 && i0 + q < n) ? X[(i0 + q) * ld + c] : T(0);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (i0 + q < n) out[(i0 + q) * ldo + j] = v[q];
    }
}

}  // namespace

using namespace mdsx;

extern "C" int mdsx_active_columns(mdsx_handle* h, const void* data, int dtype, int64_t ld,
                                   int64_t n, int32_t p, int32_t* cols, int32_t* count,
                                   void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (!data || !cols || !count || n < 1 || p < 1 || ld < p)
    return fail(h, MDSX_PARAM, "bad active-column arguments");
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  const bool flat = ld == p && (p * es) % 16 == 0 && (reinterpret_cast<uintptr_t>(data) & 15) == 0;
  int rc = ws_reserve(h, (size_t)p * sizeof(int) + 256);
  if (rc) return rc;
  int* flags = (int*)ws_alloc(h, (size_t)p * sizeof(int), st);
  if (!flags) return MDSX_CUDA;
  if ((rc = cuda_check(h, cudaMemsetAsync(flags, 0, (size_t)p * sizeof(int), st), "memset"))) return rc;
  mdsx::pre(h, st);
  if (flat) {
    const int vpr = (int)(p * es / 16);
    const int64_t nvec = n * vpr;
    // step: a multiple of vpr near 2048 threads per SM
    const int64_t want = (int64_t)h->num_sms * 2048;
    const int64_t step = std::max<int64_t>(vpr, (want / vpr) * vpr);
    const int blocks = (int)((step + 255) / 256);
    if (dtype == MDSX_F32)
      nonzero_cols_flat_kernel<float><<<blocks, 256, 0, st>>>((const float*)data, nvec, vpr, step, flags);
    else
      nonzero_cols_flat_kernel<double><<<blocks, 256, 0, st>>>((const double*)data, nvec, vpr, step, flags);
  } else {
    const int blocks = (int)std::min<int64_t>((n + 7) / 8, (int64_t)h->num_sms * 8);
    if (dtype == MDSX_F32)
      nonzero_cols_kernel<float><<<blocks, 256, 0, st>>>((const float*)data, ld, n, p, flags);
    else
      nonzero_cols_kernel<double><<<blocks, 256, 0, st>>>((const double*)data, ld, n, p, flags);
  }
  if ((rc = launched(h, "nonzero_cols_kernel", st))) return rc;
  std::vector<int> hf(p);
  if ((rc = cuda_check(h, cudaMemcpyAsync(hf.data(), flags, (size_t)p * sizeof(int),
                                          cudaMemcpyDeviceToHost, st), "active columns d2h")))
    return rc;
  if ((rc = cuda_check(h, cudaStreamSynchronize(st), "active columns sync"))) return rc;
  int c = 0;
  for (int j = 0; j < p; ++j)
    if (hf[j]) cols[c++] = j;
  *count = c;
  return MDSX_OK;
}

extern "C" int mdsx_gather_columns(mdsx_handle* h, const void* data, int dtype, int64_t ld,
                                   int64_t n, const int32_t* cols, int32_t pa, int64_t ldo,
                                   void* out, void* stream) {
  cudaStream_t st = as_stream(stream);
  MDSX_GUARD(h, st);
  if (!data || !cols || !out || n < 0 || pa < 0 || ldo < pa)
    return fail(h, MDSX_PARAM, "bad gather-columns arguments");
  if (n == 0 || ldo == 0) return MDSX_OK;
  if (ldo > 1 << 20) return fail(h, MDSX_PARAM, "gather columns: ldo too large");
  const int blocks = (int)std::min<int64_t>((n + 3) / 4, (int64_t)h->num_sms * 8);
  const size_t sm = (size_t)ldo * sizeof(int);
  mdsx::pre(h, st);
  if (dtype == MDSX_F32)
    gather_cols_kernel<float><<<blocks, 256, sm, st>>>((const float*)data, ld, n, cols, pa, (int)ldo, (float*)out);
  else
    gather_cols_kernel<double><<<blocks, 256, sm, st>>>((const double*)data, ld, n, cols, pa, (int)ldo, (double*)out);
  return launched(h, "gather_cols_kernel", st);
}
