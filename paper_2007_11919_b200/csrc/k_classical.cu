// Batched classical MDS of plan pieces (classical.py:88-160, linalg.py:61-169).
//
// B200 formulation: double centering of the squared-distance matrix equals
// the Gram matrix of column-centred rows (linalg.py:107-121 <-> S/95), so each
// piece is centred once (K2: column means, fixed-order reductions) and its
// Gram is built on the fp64 pipe (K1) in whichever orientation is smaller:
//   form 0  A = Xc^T Xc  (k = p <  m)  -> points = Xc U_r
//   form 1  A = Xc Xc^T  (k = m <= p)  -> points = V_r sqrt(lambda_r)
// The k x k eigenproblem (K3) is solved by a parallel-order cyclic Jacobi
// method entirely in shared memory (one CTA per piece, k <= 112), which
// returns the full spectrum, so G1/G2 use the complete denominators exactly
// as classical.py:75-85.  The sign rule of linalg.py:139-146 is applied to
// the output columns.
#include "mdsx_common.cuh"

#include <algorithm>

namespace {

constexpr int GT = 64;   // Gram output tile
constexpr int GK = 16;   // reduction step
constexpr int JAC_THREADS = 512;
constexpr int JAC_MAX_SWEEPS = 40;

// ----------------------------------------------------------------- K2 means
template <typename T>
__global__ void __launch_bounds__(256)
piece_means_kernel(const T* __restrict__ X, int64_t ld, int p, const int64_t* __restrict__ row_idx,
                   const PieceDesc* __restrict__ pd, double* __restrict__ mu_all,
                   mdsx_piece_status* __restrict__ status) {
  __shared__ double part[256];
  __shared__ int nonfinite;
  if (threadIdx.x == 0) nonfinite = 0;
  __syncthreads();
  const PieceDesc d = pd[blockIdx.x];
  const int64_t* ridx = row_idx + d.row_off;
  double* mu = mu_all + (int64_t)blockIdx.x * p;
  const int tid = threadIdx.x;
  if (p <= 256) {
    const int G = 256 / p;            // row groups
    const int col = tid % p, grp = tid / p;
    double s = 0.0;
    bool bad = false;
    if (grp < G)
      for (int i = grp; i < d.m; i += G) {
        const double v = mdsx::ld_val(X + ridx[i] * ld + col);
        bad |= !isfinite(v);
        s += v;
      }
    if (bad) nonfinite = 1;
    part[tid] = s;
    __syncthreads();
    if (tid < p) {
      double t = 0.0;
      for (int g = 0; g < G; ++g) t += part[g * p + tid];
      mu[tid] = t / d.m;
    }
  } else {
    for (int col = tid; col < p; col += 256) {
      double s = 0.0;
      bool bad = false;
      for (int i = 0; i < d.m; ++i) {
        const double v = mdsx::ld_val(X + ridx[i] * ld + col);
        bad |= !isfinite(v);
        s += v;
      }
      if (bad) nonfinite = 1;
      mu[col] = s / d.m;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0)
    status[blockIdx.x] = mdsx_piece_status{nonfinite ? MDSX_INVALID_INPUT : MDSX_OK, 0, 0.0};
}

// ------------------------------------------------------------------ K1 Gram
// One CTA per (piece, ti, tj) lower-triangle 64x64 tile; fp64 FMA, 4x4 per
// thread, reduction order fixed -> bitwise deterministic and exactly
// symmetric (diagonal tiles compute both halves with identical products).
template <typename T>
__global__ void __launch_bounds__(256)
gram_kernel(const T* __restrict__ X, int64_t ld, int p, const int64_t* __restrict__ row_idx,
            const PieceDesc* __restrict__ pd, const double* __restrict__ mu_all,
            const int4* __restrict__ tiles, double* __restrict__ A) {
  __shared__ double sa[GK][GT + 1];
  __shared__ double sb[GK][GT + 1];
  const int4 tl = tiles[blockIdx.x];
  const PieceDesc d = pd[tl.x];
  const int ti = tl.y, tj = tl.z, k = d.k;
  const double* mu = mu_all + (int64_t)tl.x * p;
  const int64_t* ridx = row_idx + d.row_off;
  const int K = d.form == 0 ? d.m : p;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;

  for (int k0 = 0; k0 < K; k0 += GK) {
    if (d.form == 0) {
      for (int e = threadIdx.x; e < GK * GT; e += 256) {
        const int t = e / GT, a = e % GT, tt = k0 + t;
        const int ai = ti * GT + a, aj = tj * GT + a;
        double va = 0.0, vb = 0.0;
        if (tt < K) {
          const T* row = X + ridx[tt] * ld;
          if (ai < k) va = mdsx::ld_val(row + ai) - mu[ai];
          if (aj < k) vb = mdsx::ld_val(row + aj) - mu[aj];
        }
        sa[t][a] = va;
        sb[t][a] = vb;
      }
    } else {
      for (int e = threadIdx.x; e < GK * GT; e += 256) {
        const int t = e % GK, i = e / GK, tt = k0 + t;
        const int ri = ti * GT + i, rj = tj * GT + i;
        double va = 0.0, vb = 0.0;
        if (tt < K) {
          const double m = mu[tt];
          if (ri < k) va = mdsx::ld_val(X + ridx[ri] * ld + tt) - m;
          if (rj < k) vb = mdsx::ld_val(X + ridx[rj] * ld + tt) - m;
        }
        sa[t][i] = va;
        sb[t][i] = vb;
      }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < GK; ++t) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = sa[t][ty + 16 * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) b[v] = sb[t][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
  double* out = A + d.a_off;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int x = ti * GT + ty + 16 * u, y = tj * GT + tx + 16 * v;
      if (x < k && y < k) {
        out[(int64_t)x * k + y] = acc[u][v];
        if (ti != tj) out[(int64_t)y * k + x] = acc[u][v];
      }
    }
}

// ------------------------------------------------------------- K3 Jacobi
// Parallel cyclic Jacobi (round-robin pairing) on a k x k symmetric matrix in
// shared memory.  Each round rotates kk/2 disjoint pairs; the two-sided
// update is done as independent 2x2 block tasks (one writer per block).
__global__ void __launch_bounds__(JAC_THREADS)
jacobi_kernel(const PieceDesc* __restrict__ pd, int r, const double* __restrict__ Aall,
              double* __restrict__ Uout, double* __restrict__ lam_out,
              double* __restrict__ estimates, double* __restrict__ gof,
              mdsx_piece_status* __restrict__ status, int qform_trivial) {
  extern __shared__ double sm[];
  __shared__ double cs[MDSX_JACOBI_KMAX / 2], sn[MDSX_JACOBI_KMAX / 2], tn[MDSX_JACOBI_KMAX / 2];
  __shared__ int pp[MDSX_JACOBI_KMAX / 2], qq[MDSX_JACOBI_KMAX / 2];
  __shared__ int nrot;
  __shared__ double red[JAC_THREADS];
  __shared__ int order[MDSX_JACOBI_KMAX];
  __shared__ double lam[MDSX_JACOBI_KMAX];
  __shared__ int trivial;

  const PieceDesc d = pd[blockIdx.x];
  const int k = d.k, kk = k + (k & 1), P = kk / 2;
  const int tid = threadIdx.x, nt = blockDim.x;
  double* A = sm;
  double* U = sm + kk * kk;
  const double* Ag = Aall + d.a_off;

  double fro = 0.0;
  for (int e = tid; e < kk * kk; e += nt) {
    const int i = e / kk, j = e % kk;
    const double v = (i < k && j < k) ? Ag[(int64_t)i * k + j] : 0.0;
    A[e] = v;
    U[e] = (i == j) ? 1.0 : 0.0;
    fro += v * v;
  }
  red[tid] = fro;
  __syncthreads();
  for (int s = nt / 2; s > 0; s >>= 1) {
    if (tid < s) red[tid] += red[tid + s];
    __syncthreads();
  }
  const double floor_abs = 1e-17 * sqrt(red[0]);
  const double eps = 2.220446049250313e-16;

  int sweep = 0;
  bool converged = (k <= 1);
  for (; sweep < JAC_MAX_SWEEPS && !converged; ++sweep) {
    __syncthreads();
    if (tid == 0) nrot = 0;
    __syncthreads();
    for (int rnd = 0; rnd < kk - 1; ++rnd) {
      if (tid < P) {
        const int x = (tid == 0) ? 0 : 1 + (rnd + tid - 1) % (kk - 1);
        const int y = 1 + (rnd - tid + kk - 2) % (kk - 1);
        const int p_ = min(x, y), q_ = max(x, y);
        const double app = A[p_ * kk + p_], aqq = A[q_ * kk + q_], apq = A[p_ * kk + q_];
        double c = 1.0, s = 0.0, t = 0.0;
        if (fabs(apq) > fmax(eps * sqrt(fabs(app) * fabs(aqq)), floor_abs)) {
          mdsx::sym_rotation(app, aqq, apq, c, s, t);
          atomicAdd(&nrot, 1);
        }
        cs[tid] = c; sn[tid] = s; tn[tid] = t; pp[tid] = p_; qq[tid] = q_;
      }
      __syncthreads();
      for (int L = tid; L < P * P; L += nt) {
        const int i = L / P, i2 = L % P;
        if (i2 > i) continue;
        const int p = pp[i], q = qq[i];
        if (i == i2) {
          const double t = tn[i];
          if (t != 0.0) {
            const double apq = A[p * kk + q];
            A[p * kk + p] -= t * apq;
            A[q * kk + q] += t * apq;
            A[p * kk + q] = 0.0;
            A[q * kk + p] = 0.0;
          }
          continue;
        }
        const int p2 = pp[i2], q2 = qq[i2];
        const double c = cs[i], s = sn[i], c2 = cs[i2], s2 = sn[i2];
        const double a1 = A[p * kk + p2], a2 = A[p * kk + q2];
        const double a3 = A[q * kk + p2], a4 = A[q * kk + q2];
        const double b1 = c2 * a1 - s2 * a2, b2 = s2 * a1 + c2 * a2;
        const double b3 = c2 * a3 - s2 * a4, b4 = s2 * a3 + c2 * a4;
        const double n1 = c * b1 - s * b3, n3 = s * b1 + c * b3;
        const double n2 = c * b2 - s * b4, n4 = s * b2 + c * b4;
        A[p * kk + p2] = n1; A[p2 * kk + p] = n1;
        A[p * kk + q2] = n2; A[q2 * kk + p] = n2;
        A[q * kk + p2] = n3; A[p2 * kk + q] = n3;
        A[q * kk + q2] = n4; A[q2 * kk + q] = n4;
      }
      for (int L = tid; L < kk * P; L += nt) {
        const int row = L / P, i = L % P;
        const double s = sn[i];
        if (s == 0.0) continue;
        const double c = cs[i];
        const int p = pp[i], q = qq[i];
        const double up = U[row * kk + p], uq = U[row * kk + q];
        U[row * kk + p] = c * up - s * uq;
        U[row * kk + q] = s * up + c * uq;
      }
      __syncthreads();
    }
    converged = (nrot == 0);
  }
  __syncthreads();

  // ---- spectrum post-processing (classical.py:88-106, 137-150)
  if (tid == 0) trivial = -1;
  __syncthreads();
  if (qform_trivial && d.form == 1) {
    // eigenvector with the largest |V^T 1| carries the structural zero
    if (tid < k) {
      double s = 0.0;
      for (int i = 0; i < k; ++i) s += U[i * kk + tid];
      red[tid] = fabs(s);
    }
    __syncthreads();
    if (tid == 0) {
      int best = 0;
      for (int j = 1; j < k; ++j)
        if (red[j] > red[best]) best = j;
      trivial = best;
    }
    __syncthreads();
  }
  const int triv = trivial;
  if (tid < k && tid != triv) {
    const double lj = A[tid * kk + tid];
    int rank = 0;
    for (int i = 0; i < k; ++i) {
      if (i == triv || i == tid) continue;
      const double li = A[i * kk + i];
      if (li > lj || (li == lj && i < tid)) ++rank;
    }
    order[rank] = tid;
  }
  __syncthreads();
  if (tid == 0) {
    const int nv = k - (triv >= 0 ? 1 : 0);
    double mx = 0.0;
    for (int i = 0; i < nv; ++i) mx = fmax(mx, fabs(A[order[i] * kk + order[i]]));
    const double tol = 1e-8 * mx;
    double sum_abs = 0.0, sum_pos = 0.0, kept = 0.0;
    for (int i = 0; i < nv; ++i) {
      double v = A[order[i] * kk + order[i]];
      if (fabs(v) <= tol) v = 0.0;
      lam[i] = v;
      sum_abs += fabs(v);
      sum_pos += fmax(v, 0.0);
      if (i < r) kept += v;
    }
    mdsx_piece_status st{MDSX_OK, 0, 0.0};
    if (status[blockIdx.x].code != MDSX_OK) st.code = status[blockIdx.x].code;
    else if (!converged) st.code = MDSX_NUMERICAL;
    for (int i = 0; i < r && st.code == MDSX_OK; ++i) {
      const double v = i < nv ? lam[i] : 0.0;
      if (v <= 0.0) { st.code = MDSX_DEGENERATE; st.index = i + 1; st.value = v; }
    }
    if (st.code == MDSX_OK && sum_abs == 0.0) st.code = MDSX_DEGENERATE;
    status[blockIdx.x] = st;
    double* g = gof + 2 * (int64_t)blockIdx.x;
    g[0] = st.code == MDSX_OK ? kept / sum_abs : 0.0;
    g[1] = st.code == MDSX_OK ? kept / sum_pos : 0.0;
    for (int i = 0; i < r; ++i) {
      const double v = i < nv ? lam[i] : 0.0;
      estimates[(int64_t)blockIdx.x * r + i] = v / d.m;
      lam_out[(int64_t)blockIdx.x * r + i] = v;
    }
  }
  __syncthreads();
  const int nv = k - (triv >= 0 ? 1 : 0);
  for (int e = tid; e < k * r; e += nt) {
    const int a = e / r, c = e % r;
    Uout[d.u_off + e] = c < nv ? U[a * kk + order[c]] : 0.0;
  }
}

// ------------------------------------------------------------ points + signs
template <typename T, int RM>
__global__ void __launch_bounds__(256)
points_kernel(const T* __restrict__ X, int64_t ld, int p, const int64_t* __restrict__ row_idx,
              const PieceDesc* __restrict__ pd, int r, const double* __restrict__ mu_all,
              const double* __restrict__ Uall, const double* __restrict__ lam_all,
              double* __restrict__ points) {
  extern __shared__ double sm[];
  __shared__ double bval[256];
  __shared__ int bidx[256];
  __shared__ double sgn[RM];
  const PieceDesc d = pd[blockIdx.x];
  const int tid = threadIdx.x;
  const int64_t* ridx = row_idx + d.row_off;
  double* out = points + d.pt_off * r;
  const double* Ug = Uall + d.u_off;
  double* sU = sm;                 // p x r (form 0)
  double* smu = sm + (int64_t)p * r;
  if (d.form == 0) {
    for (int e = tid; e < p * r; e += 256) sU[e] = Ug[e];
    for (int e = tid; e < p; e += 256) smu[e] = mu_all[(int64_t)blockIdx.x * p + e];
  }
  __syncthreads();
  double sl[RM];
#pragma unroll
  for (int c = 0; c < RM; ++c) sl[c] = (c < r) ? sqrt(lam_all[(int64_t)blockIdx.x * r + c]) : 0.0;

  double best[RM];
  int bi[RM];
#pragma unroll
  for (int c = 0; c < RM; ++c) { best[c] = -1.0; bi[c] = 0x7fffffff; }
  for (int i = tid; i < d.m; i += 256) {
    double acc[RM];
#pragma unroll
    for (int c = 0; c < RM; ++c) acc[c] = 0.0;
    if (d.form == 0) {
      const T* row = X + ridx[i] * ld;
      for (int a = 0; a < p; ++a) {
        const double y = mdsx::ld_val(row + a) - smu[a];
#pragma unroll
        for (int c = 0; c < RM; ++c)
          if (c < r) acc[c] = fma(y, sU[a * r + c], acc[c]);
      }
    } else {
#pragma unroll
      for (int c = 0; c < RM; ++c)
        if (c < r) acc[c] = Ug[(int64_t)i * r + c] * sl[c];
    }
#pragma unroll
    for (int c = 0; c < RM; ++c)
      if (c < r) {
        out[(int64_t)i * r + c] = acc[c];
        const double a = fabs(acc[c]);
        if (a > best[c]) { best[c] = a; bi[c] = i; }   // rows visited ascending
      }
  }
  // block argmax per column: largest |.|, lowest index on ties
  for (int c = 0; c < r; ++c) {
    bval[tid] = best[c];
    bidx[tid] = bi[c];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (tid < s) {
        const double v2 = bval[tid + s];
        const int i2 = bidx[tid + s];
        if (v2 > bval[tid] || (v2 == bval[tid] && i2 < bidx[tid])) { bval[tid] = v2; bidx[tid] = i2; }
      }
      __syncthreads();
    }
    if (tid == 0) {
      const int lead = bidx[0];
      double s = 1.0;
      if (lead < d.m) {
        const double v = out[(int64_t)lead * r + c];
        s = v < 0.0 ? -1.0 : 1.0;
      }
      sgn[c] = s;
    }
    __syncthreads();
  }
  for (int i = tid; i < d.m; i += 256)
    for (int c = 0; c < r; ++c)
      if (sgn[c] < 0.0) out[(int64_t)i * r + c] = -out[(int64_t)i * r + c];
}

template <typename T>
int points_dispatch(mdsx_handle* h, const T* X, int64_t ld, int p, const int64_t* row_idx,
                    const PieceDesc* pd, int npieces, int r, const double* mu, const double* U,
                    const double* lam, double* points, cudaStream_t st) {
  const size_t smem = ((size_t)p * r + p) * sizeof(double);
  auto go = [&](auto kern) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<npieces, 256, smem, st>>>(X, ld, p, row_idx, pd, r, mu, U, lam, points);
    return mdsx::launched(h, "points_kernel");
  };
  if (r <= 4) return go(points_kernel<T, 4>);
  if (r <= 8) return go(points_kernel<T, 8>);
  if (r <= 16) return go(points_kernel<T, 16>);
  return go(points_kernel<T, 32>);
}

}  // namespace

namespace mdsx {

int launch_piece_means(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                       const int64_t* row_idx, const PieceDesc* pd, int npieces, double* mu,
                       mdsx_piece_status* status, cudaStream_t st) {
  if (dtype == MDSX_F64)
    piece_means_kernel<double><<<npieces, 256, 0, st>>>((const double*)data, ld, p, row_idx, pd, mu,
                                                        status);
  else
    piece_means_kernel<float><<<npieces, 256, 0, st>>>((const float*)data, ld, p, row_idx, pd, mu,
                                                       status);
  return launched(h, "piece_means_kernel");
}

int launch_gram(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                const int64_t* row_idx, const PieceDesc* pd, const double* mu, const int4* tiles,
                int ntiles, double* A, cudaStream_t st) {
  if (ntiles == 0) return MDSX_OK;
  if (dtype == MDSX_F64)
    gram_kernel<double><<<ntiles, 256, 0, st>>>((const double*)data, ld, p, row_idx, pd, mu, tiles, A);
  else
    gram_kernel<float><<<ntiles, 256, 0, st>>>((const float*)data, ld, p, row_idx, pd, mu, tiles, A);
  return launched(h, "gram_kernel");
}

int launch_jacobi(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r, double* A,
                  double* U, double* lam, double* estimates, double* gof,
                  mdsx_piece_status* status, int qform_trivial, cudaStream_t st) {
  const int kk = kmax + (kmax & 1);
  const size_t smem = (size_t)2 * kk * kk * sizeof(double);
  cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  jacobi_kernel<<<npieces, JAC_THREADS, smem, st>>>(pd, r, A, U, lam, estimates, gof, status,
                                                     qform_trivial);
  return launched(h, "jacobi_kernel");
}

int launch_points(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                  const int64_t* row_idx, const PieceDesc* pd, int npieces, int r,
                  const double* mu, const double* U, const double* lam, double* points,
                  cudaStream_t st) {
  if (dtype == MDSX_F64)
    return points_dispatch(h, (const double*)data, ld, p, row_idx, pd, npieces, r, mu, U, lam,
                           points, st);
  return points_dispatch(h, (const float*)data, ld, p, row_idx, pd, npieces, r, mu, U, lam,
                         points, st);
}

}  // namespace mdsx
