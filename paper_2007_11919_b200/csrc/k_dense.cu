// Function-level dense seams: K1 distance matrices (linalg.py:61-104), K2
// double centering (linalg.py:107-121) and the squared-distance validity
// checks (linalg.py:41-58).  These materialise m x m matrices and exist for
// the public primitives and for classical_mds(delta); the partition
// algorithms never call them (they go through k_classical.cu).
#include "mdsx_common.cuh"

#include <algorithm>
#include <vector>

namespace {

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

// K1 on the fp64 tensor pipe: the cross term A B^T of a 64 x 64 output tile by
// DMMA m8n8k4 (8 warps as 2 x 4, each 32 x 16 = 4 x 2 blocks), rows staged
// 16 features at a time in shared memory with pitches == 4 (mod 16) doubles
// (conflict-free fragments).  Self distances: only tiles on and below the
// diagonal are computed and mirrored, so D is exactly symmetric (the
// reference's (D + D^T)/2 is the identity) with half the work.
constexpr int QT = 64, QK = 16, QP = QT + 4;

template <typename T>
__global__ void __launch_bounds__(256)
sqdist_dmma_kernel(const T* __restrict__ A, int64_t lda, int64_t ma, const T* __restrict__ B,
                   int64_t ldb, int64_t mb, int p, const double* __restrict__ na,
                   const double* __restrict__ nb, double* __restrict__ out, int64_t ldo, int self,
                   const int2* __restrict__ tiles) {
  __shared__ __align__(16) double sa[QK][QP];
  __shared__ __align__(16) double sb[QK][QP];
  const int2 tl = tiles ? tiles[blockIdx.x] : make_int2(blockIdx.y, blockIdx.x);
  const int64_t i0 = (int64_t)tl.x * QT, j0 = (int64_t)tl.y * QT;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = (warp >> 2) * 32, wn = (warp & 3) * 16;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int k0 = 0; k0 < p; k0 += QK) {
    // 64 rows x 16 features of each operand: thread -> (row, 4 features)
    {
      const int rr = tid >> 2, kq = (tid & 3) * 4;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = kq + u;
        const int64_t ia = i0 + rr, jb = j0 + rr;
        sa[kk][rr] = (ia < ma && k0 + kk < p) ? mdsx::ld_val(A + ia * lda + k0 + kk) : 0.0;
        sb[kk][rr] = (jb < mb && k0 + kk < p) ? mdsx::ld_val(B + jb * ldb + k0 + kk) : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < QK / 4; ++ks) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = sa[4 * ks + tig][wm + 8 * i + gid];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = sb[4 * ks + tig][wn + 8 * j + gid];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(af[i]), "d"(bf[j]));
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int64_t gi = i0 + wm + 8 * i + gid, gj = j0 + wn + 8 * j + 2 * tig + v;
        if (gi >= ma || gj >= mb) continue;
        if (self) {
          if (gj > gi) continue;                       // lower triangle, mirrored
          const double d = gi == gj ? 0.0 : fmax((na[gi] + nb[gj]) - 2.0 * acc[i][j][v], 0.0);
          out[gi * ldo + gj] = d;
          out[gj * ldo + gi] = d;
        } else {
          out[gi * ldo + gj] = fmax((-2.0 * acc[i][j][v] + na[gi]) + nb[gj], 0.0);
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
    const int64_t ta = (ma + QT - 1) / QT, tb = (mb + QT - 1) / QT;
    if (self) {                        // lower-triangle tile list (ti >= tj)
      std::vector<int2> tl;
      for (int64_t a = 0; a < ta; ++a)
        for (int64_t b = 0; b <= a; ++b) tl.push_back(make_int2((int)a, (int)b));
      int2* dt = (int2*)ws_alloc(h, tl.size() * sizeof(int2), st);
      if (!dt) return (int)MDSX_CUDA;
      if ((rc = upload(h, dt, tl.data(), tl.size() * sizeof(int2), st))) return rc;
      mdsx::pre(h, st);
      sqdist_dmma_kernel<T><<<(unsigned)tl.size(), 256, 0, st>>>(
          (const T*)A, lda, ma, (const T*)B, ldb, mb, p, na, na, out, ldo, 1, dt);
    } else {
      dim3 grid((unsigned)tb, (unsigned)ta);
      mdsx::pre(h, st);
      sqdist_dmma_kernel<T><<<grid, 256, 0, st>>>((const T*)A, lda, ma, (const T*)B, ldb, mb, p,
                                                  na, nb, out, ldo, 0, nullptr);
    }
    return launched(h, "sqdist_dmma_kernel", st);
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
