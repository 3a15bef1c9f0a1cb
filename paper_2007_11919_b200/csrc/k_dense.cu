// Function-level dense seams: K1 distance matrices (linalg.py:61-104), K2
// double centering (linalg.py:107-121) and the squared-distance validity
// checks (linalg.py:41-58).  These materialise m x m matrices and exist for
// the public primitives and for classical_mds(delta); the partition
// algorithms never call them (they go through k_classical.cu).
#include "mdsx_common.cuh"

#include <algorithm>

namespace {

constexpr int DT = 32;  // distance tile

template <typename T>
__global__ void rownorm_kernel(const T* __restrict__ X, int64_t ld, int64_t m, int p,
                               double* __restrict__ nrm) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int a = 0; a < p; ++a) {
    const double v = mdsx::ld_val(X + i * ld + a);
    s = fma(v, v, s);
  }
  nrm[i] = s;
}

// out_ij = max(na_i + nb_j - 2 a_i.b_j, 0); self: exact-zero diagonal.
// For self distances d_ij and d_ji are computed from identical products and
// sums (commutative), so the matrix is exactly symmetric and the reference's
// 0.5 (d + d^T) step is the identity.
template <typename T>
__global__ void __launch_bounds__(DT * 8)
sqdist_kernel(const T* __restrict__ A, int64_t lda, int64_t ma, const T* __restrict__ B,
              int64_t ldb, int64_t mb, int p, const double* __restrict__ na,
              const double* __restrict__ nb, double* __restrict__ out, int64_t ldo, int self) {
  __shared__ double sa[DT][DT + 1];
  __shared__ double sb[DT][DT + 1];
  const int tx = threadIdx.x % DT, ty = threadIdx.x / DT;  // 32 x 8
  const int64_t i0 = (int64_t)blockIdx.y * DT, j0 = (int64_t)blockIdx.x * DT;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int k0 = 0; k0 < p; k0 += DT) {
    for (int e = threadIdx.x; e < DT * DT; e += DT * 8) {
      const int rr = e / DT, kk = e % DT;
      const int64_t ia = i0 + rr, jb = j0 + rr;
      sa[rr][kk] = (ia < ma && k0 + kk < p) ? mdsx::ld_val(A + ia * lda + k0 + kk) : 0.0;
      sb[rr][kk] = (jb < mb && k0 + kk < p) ? mdsx::ld_val(B + jb * ldb + k0 + kk) : 0.0;
    }
    __syncthreads();
    for (int kk = 0; kk < DT; ++kk) {
      const double b = sb[tx][kk];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] = fma(sa[ty + 8 * u][kk], b, acc[u]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = i0 + ty + 8 * u, j = j0 + tx;
    if (i < ma && j < mb) {
      double d;
      if (self) d = (i == j) ? 0.0 : fmax((na[i] + nb[j]) - 2.0 * acc[u], 0.0);
      else d = fmax((-2.0 * acc[u] + na[i]) + nb[j], 0.0);
      out[i * ldo + j] = d;
    }
  }
}

__global__ void rowmean_kernel(const double* __restrict__ D, int64_t m, double* __restrict__ mu) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s = 0.0;
  for (int64_t j = 0; j < m; ++j) s += D[i * m + j];
  mu[i] = s / (double)m;
}

__global__ void grandmean_kernel(const double* __restrict__ mu, int64_t m, double* __restrict__ g) {
  __shared__ double red[256];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += 256) s += mu[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) g[0] = red[0] / (double)m;
}

// q_ij = -1/2 (d_ij - mu_i - mu_j + g), then 0.5 (q + q^T) (linalg.py:116-121)
__global__ void dcenter_kernel(const double* __restrict__ D, int64_t m, const double* __restrict__ mu,
                               const double* __restrict__ g, double* __restrict__ Q) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= m * m) return;
  const int64_t i = e / m, j = e % m;
  const double gm = g[0];
  const double qij = -0.5 * (((D[i * m + j] - mu[i]) - mu[j]) + gm);
  const double qji = -0.5 * (((D[j * m + i] - mu[j]) - mu[i]) + gm);
  Q[e] = 0.5 * (qij + qji);
}

// validity of a squared-distance matrix (linalg.py:41-58): flags bit0 non-finite,
// bit1 asymmetric, bit2 nonzero diagonal, bit3 negative.  Two passes: scale, checks.
__global__ void absmax_kernel(const double* __restrict__ D, int64_t total,
                              unsigned long long* __restrict__ mx, int32_t* __restrict__ flags) {
  double loc = 0.0;
  bool bad = false;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const double v = D[e];
    if (!isfinite(v)) bad = true;
    else loc = fmax(loc, fabs(v));
  }
  atomicMax(mx, (unsigned long long)__double_as_longlong(loc));  // non-negative doubles order as ints
  if (bad) atomicOr(flags, 1);
}

__global__ void delta_check_kernel(const double* __restrict__ D, int64_t m,
                                   const unsigned long long* __restrict__ mx,
                                   int32_t* __restrict__ flags) {
  const double scale = __longlong_as_double((long long)mx[0]);
  const double tol = 1e-9 * fmax(scale, 1.0);
  int f = 0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m * m;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / m, j = e % m;
    const double v = D[e];
    if (fabs(v - D[j * m + i]) > tol) f |= 2;
    if (i == j && fabs(v) > tol) f |= 4;
    if (v < -tol) f |= 8;
  }
  if (f) atomicOr(flags, f);
}

}  // namespace

namespace mdsx {

int launch_sqdist(mdsx_handle* h, const void* A, int64_t lda, int64_t ma, const void* B,
                  int64_t ldb, int64_t mb, int dtype, int p, double* na, double* nb, double* out,
                  int64_t ldo, int self, cudaStream_t st) {
  if (ma == 0 || mb == 0) return MDSX_OK;
  auto go = [&](auto tag) {
    using T = decltype(tag);
    mdsx::pre(h, st);
    rownorm_kernel<T><<<(unsigned)((ma + 255) / 256), 256, 0, st>>>((const T*)A, lda, ma, p, na);
    int rc = launched(h, "rownorm_kernel", st);
    if (rc) return rc;
    if (!self) {
      mdsx::pre(h, st);
      rownorm_kernel<T><<<(unsigned)((mb + 255) / 256), 256, 0, st>>>((const T*)B, ldb, mb, p, nb);
      rc = launched(h, "rownorm_kernel", st);
      if (rc) return rc;
    }
    dim3 grid((unsigned)((mb + DT - 1) / DT), (unsigned)((ma + DT - 1) / DT));
    mdsx::pre(h, st);
    sqdist_kernel<T><<<grid, DT * 8, 0, st>>>((const T*)A, lda, ma, (const T*)B, ldb, mb, p, na,
                                                self ? na : nb, out, ldo, self);
    return launched(h, "sqdist_kernel", st);
  };
  return dtype == MDSX_F64 ? go(double{}) : go(float{});
}

int launch_double_center(mdsx_handle* h, const double* D, int64_t m, double* mu, double* g,
                         double* Q, cudaStream_t st) {
  mdsx::pre(h, st);
  rowmean_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(D, m, mu);
  int rc = launched(h, "rowmean_kernel", st);
  if (rc) return rc;
  mdsx::pre(h, st);
  grandmean_kernel<<<1, 256, 0, st>>>(mu, m, g);
  rc = launched(h, "grandmean_kernel", st);
  if (rc) return rc;
  mdsx::pre(h, st);
  dcenter_kernel<<<(unsigned)((m * m + 255) / 256), 256, 0, st>>>(D, m, mu, g, Q);
  return launched(h, "dcenter_kernel", st);
}

int launch_delta_check(mdsx_handle* h, const double* D, int64_t m, unsigned long long* mx,
                       int32_t* flags, cudaStream_t st) {
  const int blocks = (int)std::min<int64_t>((m * m + 255) / 256, (int64_t)h->num_sms * 4);
  mdsx::pre(h, st);
  absmax_kernel<<<blocks, 256, 0, st>>>(D, m * m, mx, flags);
  int rc = launched(h, "absmax_kernel", st);
  if (rc) return rc;
  mdsx::pre(h, st);
  delta_check_kernel<<<blocks, 256, 0, st>>>(D, m, mx, flags);
  return launched(h, "delta_check_kernel", st);
}

}  // namespace mdsx
