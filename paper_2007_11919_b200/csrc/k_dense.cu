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

// K1, pipelined: a 128 x 64 output tile per CTA (8 warps as 4 x 2, each 32 x 32
// = 4 x 4 DMMA blocks: 16 DMMA per 8 fragment loads), the operand rows staged
// ROW-MAJOR, 128 bytes of features per row and stage, by 16-byte cp.async
// (zero fill past p and past the last row) into a 3-stage ring, one barrier
// per stage.  Row pitches of 20 doubles / 36 floats make the m8n8k4 fragment
// loads conflict-free without a transposing store.  Needs 16-byte aligned rows.
template <typename T> struct SqCfg;
template <> struct SqCfg<double> { static constexpr int KC = 16, P = 20; };
template <> struct SqCfg<float> { static constexpr int KC = 32, P = 36; };
constexpr int SQ_TM = 128, SQ_TN = 64, SQ_NS = 3;

__device__ __forceinline__ void cp_async16_zfill(void* dst, const void* src, int bytes) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}

template <typename T>
__global__ void __launch_bounds__(256, 2)
sqdist_tile_kernel(const T* __restrict__ A, int64_t lda, int64_t ma, const T* __restrict__ B,
                   int64_t ldb, int64_t mb, int p, const double* __restrict__ na,
                   const double* __restrict__ nb, double* __restrict__ out, int64_t ldo, int self,
                   const int2* __restrict__ tiles) {
  extern __shared__ __align__(16) unsigned char sq_smem[];
  constexpr int KC = SqCfg<T>::KC, P = SqCfg<T>::P, EPS = 16 / (int)sizeof(T);
  T* sA = reinterpret_cast<T*>(sq_smem);                 // SQ_NS x SQ_TM x P
  T* sB = sA + (size_t)SQ_NS * SQ_TM * P;                // SQ_NS x SQ_TN x P
  const int2 tl = tiles ? tiles[blockIdx.x] : make_int2(blockIdx.y, blockIdx.x);
  const int64_t i0 = (int64_t)tl.x * SQ_TM, j0 = (int64_t)tl.y * SQ_TN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  const int nchunks = (p + KC - 1) / KC;

  auto issue = [&](int c) {
    if (c < nchunks) {
      const int s = c % SQ_NS, k0 = c * KC;
#pragma unroll
      for (int u = 0; u < (SQ_TM + SQ_TN) * 8 / 256; ++u) {
        const int e = tid + 256 * u;
        const int row = e >> 3, seg = e & 7;
        const bool isA = row < SQ_TM;                       // warp-uniform (32 copies = 4 rows)
        const int rr = isA ? row : row - SQ_TM;
        const int64_t g = (isA ? i0 : j0) + rr;
        const bool live = g < (isA ? ma : mb);
        const int kf = k0 + seg * EPS;
        const int nval = live ? min(max(p - kf, 0), EPS) : 0;
        const T* src = nval > 0 ? (isA ? A + g * lda : B + g * ldb) + kf : A;
        T* dst = (isA ? sA + ((size_t)s * SQ_TM + rr) * P : sB + ((size_t)s * SQ_TN + rr) * P) +
                 seg * EPS;
        cp_async16_zfill(dst, src, nval * (int)sizeof(T));
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
#pragma unroll
  for (int c = 0; c < SQ_NS - 1; ++c) issue(c);
  for (int c = 0; c < nchunks; ++c) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(SQ_NS - 2));
    __syncthreads();                  // chunk c landed for everyone; stage (c - 1) % NS is free
    issue(c + SQ_NS - 1);
    const T* a_s = sA + ((size_t)(c % SQ_NS) * SQ_TM + wm + gid) * P + tig;
    const T* b_s = sB + ((size_t)(c % SQ_NS) * SQ_TN + wn + gid) * P + tig;
    const int nks = min(KC / 4, (p - c * KC + 3) >> 2);     // the last chunk stops at p
#pragma unroll
    for (int ks = 0; ks < KC / 4; ++ks) {
      if (ks >= nks) break;
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = (double)a_s[(size_t)8 * i * P + 4 * ks];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = (double)b_s[(size_t)8 * j * P + 4 * ks];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(af[i]), "d"(bf[j]));
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gi = i0 + wm + 8 * i + gid;
    if (gi >= ma) continue;
    const double nai = na[gi];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gj = j0 + wn + 8 * j + 2 * tig;
      if (self) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          if (gj + v >= mb || gj + v > gi) continue;       // lower triangle, mirrored
          const double d = gi == gj + v ? 0.0 : fmax((nai + nb[gj + v]) - 2.0 * acc[i][j][v], 0.0);
          out[gi * ldo + gj + v] = d;
          out[(gj + v) * ldo + gi] = d;
        }
      } else {
#pragma unroll
        for (int v = 0; v < 2; ++v)
          if (gj + v < mb) out[gi * ldo + gj + v] = fmax((-2.0 * acc[i][j][v] + nai) + nb[gj + v], 0.0);
      }
    }
  }
}

// Row means of a row-major m x m matrix: a warp per row, lanes stride the
// columns (coalesced; 16-byte loads when m is even, eight loads in flight per
// lane), per-lane running sums and a butterfly in fixed order (deterministic).
__global__ void __launch_bounds__(256)
rowmean_warp_kernel(const double* __restrict__ D, int64_t m, double* __restrict__ mu) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (i >= m) return;
  const double* row = D + i * m;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if ((m & 1) == 0 && (reinterpret_cast<uintptr_t>(D) & 15) == 0) {
    const double2* r2 = reinterpret_cast<const double2*>(row);
    const int64_t h = m >> 1;
    int64_t j = lane;
    for (; j + 224 < h; j += 256) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = r2[j + 32 * u];
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        s0 += v[u].x;
        s1 += v[u].y;
        s2 += v[u + 1].x;
        s3 += v[u + 1].y;
      }
    }
    for (; j < h; j += 32) {
      const double2 v = r2[j];
      s0 += v.x;
      s1 += v.y;
    }
  } else {
    int64_t j = lane;
    for (; j + 96 < m; j += 128) {
      s0 += row[j];
      s1 += row[j + 32];
      s2 += row[j + 64];
      s3 += row[j + 96];
    }
    for (; j < m; j += 32) s0 += row[j];
  }
  double s = (s0 + s1) + (s2 + s3);
  s = mdsx::warp_sum(s);
  if (lane == 0) mu[i] = s / (double)m;
}

// K2 by 64 x 64 tile pairs: the CTA of tile (I, J), I <= J, reads D_IJ and D_JI
// once (coalesced, D_JI transposed through shared memory), forms
// q = 0.5 (q_ij + q_ji) with q_ij = -1/2 (((d_ij - mu_i) - mu_j) + g) and writes
// Q_IJ and its transpose Q_JI (both coalesced): one read and one write of the
// matrix, exactly symmetric output, the arithmetic of linalg.py:116-121.
// Thread (tx = column, ty) takes rows ty, ty + 4, ...; all its loads are issued
// before the first use.  Shared rows are padded to 65 (conflict-free transposes).
constexpr int DC_T = 64, DC_P = DC_T + 1;

__global__ void __launch_bounds__(256, 2)
dcenter_tile_kernel(const double* __restrict__ D, int64_t m, const double* __restrict__ mu,
                    const double* __restrict__ g, double* __restrict__ Q, int nt) {
  extern __shared__ double dc_smem[];
  double* tji = dc_smem;                     // DC_T x DC_P
  double* tq = dc_smem + DC_T * DC_P;
  __shared__ double mu_i[DC_T];
  // linear CTA index -> (I, J), I <= J, row I has nt - I tiles
  int I = 0, rem = blockIdx.x;
  while (rem >= nt - I) { rem -= nt - I; ++I; }
  const int J = I + rem;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;
  const int64_t i0 = (int64_t)I * DC_T, j0 = (int64_t)J * DC_T;
  const double gm = g[0];
  const bool cj = j0 + tx < m, ci = i0 + tx < m;
  double dij[16], dji[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int a = ty + 4 * u;
    dij[u] = (i0 + a < m && cj) ? D[(i0 + a) * m + j0 + tx] : 0.0;
    dji[u] = (j0 + a < m && ci) ? D[(j0 + a) * m + i0 + tx] : 0.0;     // row a of D_JI
  }
  if (threadIdx.x < DC_T) mu_i[threadIdx.x] = i0 + threadIdx.x < m ? mu[i0 + threadIdx.x] : 0.0;
  const double muj = cj ? mu[j0 + tx] : 0.0;
#pragma unroll
  for (int u = 0; u < 16; ++u) tji[(ty + 4 * u) * DC_P + tx] = dji[u];
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int a = ty + 4 * u;
    const double mui = mu_i[a];
    const double qij = -0.5 * (((dij[u] - mui) - muj) + gm);
    const double qji = -0.5 * (((tji[tx * DC_P + a] - muj) - mui) + gm);
    const double q = 0.5 * (qij + qji);
    if (i0 + a < m && cj) Q[(i0 + a) * m + j0 + tx] = q;
    tq[a * DC_P + tx] = q;
  }
  if (I == J) return;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int b2 = ty + 4 * u;                        // row of Q_JI = column of Q_IJ
    if (j0 + b2 < m && ci) Q[(j0 + b2) * m + i0 + tx] = tq[tx * DC_P + b2];
  }
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
    const size_t es = sizeof(T);
    const bool tiled = ((size_t)lda * es) % 16 == 0 && ((size_t)ldb * es) % 16 == 0 &&
                       (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                       (reinterpret_cast<uintptr_t>(B) & 15) == 0 && !getenv("MDSX_SQDIST_SYNC");
    const int TM = tiled ? SQ_TM : QT, TN = tiled ? SQ_TN : QT;
    const int64_t ta = (ma + TM - 1) / TM, tb = (mb + TN - 1) / TN;
    const size_t smem = (size_t)SQ_NS * (SQ_TM + SQ_TN) * SqCfg<T>::P * es;
    if (tiled)
      cudaFuncSetAttribute(sqdist_tile_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
    if (self) {                        // tiles that touch the lower triangle
      std::vector<int2> tl;
      for (int64_t a = 0; a < ta; ++a)
        for (int64_t b = 0; b < tb && b * TN <= a * TM + TM - 1; ++b)
          tl.push_back(make_int2((int)a, (int)b));
      int2* dt = (int2*)ws_alloc(h, tl.size() * sizeof(int2), st);
      if (!dt) return (int)MDSX_CUDA;
      if ((rc = upload(h, dt, tl.data(), tl.size() * sizeof(int2), st))) return rc;
      mdsx::pre(h, st);
      if (tiled)
        sqdist_tile_kernel<T><<<(unsigned)tl.size(), 256, smem, st>>>(
            (const T*)A, lda, ma, (const T*)B, ldb, mb, p, na, na, out, ldo, 1, dt);
      else
        sqdist_dmma_kernel<T><<<(unsigned)tl.size(), 256, 0, st>>>(
            (const T*)A, lda, ma, (const T*)B, ldb, mb, p, na, na, out, ldo, 1, dt);
    } else {
      dim3 grid((unsigned)tb, (unsigned)ta);
      mdsx::pre(h, st);
      if (tiled)
        sqdist_tile_kernel<T><<<grid, 256, smem, st>>>((const T*)A, lda, ma, (const T*)B, ldb, mb,
                                                       p, na, nb, out, ldo, 0, nullptr);
      else
        sqdist_dmma_kernel<T><<<grid, 256, 0, st>>>((const T*)A, lda, ma, (const T*)B, ldb, mb, p,
                                                    na, nb, out, ldo, 0, nullptr);
    }
    return launched(h, tiled ? "sqdist_tile_kernel" : "sqdist_dmma_kernel", st);
  };
  return dtype == MDSX_F64 ? go(double{}) : go(float{});
}

int launch_double_center(mdsx_handle* h, const double* D, int64_t m, double* mu, double* g,
                         double* Q, cudaStream_t st) {
  mdsx::pre(h, st);
  rowmean_warp_kernel<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(D, m, mu);
  int rc = launched(h, "rowmean_warp_kernel", st);
  if (rc) return rc;
  mdsx::pre(h, st);
  grandmean_kernel<<<1, 256, 0, st>>>(mu, m, g);
  rc = launched(h, "grandmean_kernel", st);
  if (rc) return rc;
  const int64_t nt = (m + DC_T - 1) / DC_T;
  const size_t smem = 2 * (size_t)DC_T * DC_P * sizeof(double);
  cudaFuncSetAttribute(dcenter_tile_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mdsx::pre(h, st);
  if (nt * (nt + 1) / 2 < (int64_t)1 << 31 && !getenv("MDSX_DCENTER_FLAT")) {
    dcenter_tile_kernel<<<(unsigned)(nt * (nt + 1) / 2), 256, smem, st>>>(D, m, mu, g, Q, (int)nt);
    return launched(h, "dcenter_tile_kernel", st);
  }
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
