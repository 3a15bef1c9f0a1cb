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

#include <cstdlib>
#include "piece_solvers.cuh"

#include <algorithm>

namespace {

constexpr int GT = 64;   // Gram output tile
constexpr int GK = 16;   // reduction step

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
  double* mu = mu_all + (int64_t)d.id * p;
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
    status[d.id] = mdsx_piece_status{nonfinite ? MDSX_INVALID_INPUT : MDSX_OK, 0, 0.0};
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
  const double* mu = mu_all + (int64_t)d.id * p;
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


// ---- form 1 on the fp64 tensor pipe: 64 x 64 tiles of Q = Y Y^T (Y = the
// piece's rows centred by the piece means), K = features in chunks of 32
// staged by cp.async into a 3-deep ring (each thread copies fixed rows, so the
// row indices are read once), converted and centred at fragment-load time.
// 8 warps as 2 x 4, 32 x 16 outputs each (m8n8k4, 4 A + 2 B fragments per
// 8 DMMA).  Pitch 36 elements: conflict-free fragment loads (fp32 and fp64).
constexpr int RA_FC = 32;                 // features per chunk
constexpr int RA_NS = 3;
constexpr int RA_P = 36;

__device__ __forceinline__ void dmma_r(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <typename T>
__global__ void __launch_bounds__(256)
gram_rows_async_kernel(const T* __restrict__ X, int64_t ld, int p,
                       const int64_t* __restrict__ row_idx, const PieceDesc* __restrict__ pd,
                       const double* __restrict__ mu_all, const int4* __restrict__ tiles,
                       double* __restrict__ A) {
  constexpr int SLICE = GT * RA_P;
  extern __shared__ __align__(16) unsigned char ra_smem[];
  T* ring = reinterpret_cast<T*>(ra_smem);            // RA_NS x 2 slices
  const int4 tl = tiles[blockIdx.x];
  const PieceDesc d = pd[tl.x];
  const int ti = tl.y, tj = tl.z, k = d.k;
  const bool diag = ti == tj;
  const double* mu = mu_all + (int64_t)d.id * p;
  const int64_t* ridx = row_idx + d.row_off;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 2, wc = warp & 3;            // warp sub-tile: rows 32*wr.., cols 16*wc..
  const int nchunks = (p + RA_FC - 1) / RA_FC;
  // copy duty: thread t handles row (t >> 1) of the tile pair (0..63: block ti,
  // 64..127: block tj) and every other 16-byte piece of it, starting at (t & 1)
  const int crow = tid >> 1, cpart = tid & 1;          // 128 rows x 2 halves
  const bool second = crow >= GT;
  const int lrow = second ? crow - GT : crow;
  const int grow = (second ? tj : ti) * GT + lrow;     // row within the piece
  const bool active = (!second || !diag) && grow < k;
  const char* src = active ? reinterpret_cast<const char*>(X + ridx[grow] * ld) : nullptr;
  constexpr int PCS = RA_FC * (int)sizeof(T) / 16;     // 16-byte pieces per row per chunk
  auto issue = [&](int c) {
    if (c < nchunks && active) {
      T* dst = ring + (size_t)(c % RA_NS) * 2 * SLICE + (second ? SLICE : 0) + (size_t)lrow * RA_P;
      const int f0 = c * RA_FC;
      const int nf = min(RA_FC, p - f0);
      const int nbytes = nf * (int)sizeof(T);
      for (int q = cpart; q < PCS; q += 2) {
        if (16 * q < nbytes) {
          const unsigned sa_ = (unsigned)__cvta_generic_to_shared(reinterpret_cast<char*>(dst) + 16 * q);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa_),
                       "l"(src + (size_t)f0 * sizeof(T) + 16 * q));
        }
      }
      // the last chunk: zeros complete its last group of four features (mean 0 there)
      if (cpart == 0)
        for (int f = nf; f < ((nf + 3) & ~3); ++f) dst[f] = T(0);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
#pragma unroll
  for (int c = 0; c < RA_NS - 1; ++c) issue(c);
  // no row predicates: a row past k of the tile only reaches output rows /
  // columns the epilogue drops
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(RA_NS - 2));
    __syncthreads();                 // chunk c landed for everyone; stage (c - 1) % NS is free
    issue(c + RA_NS - 1);
    const T* sta = ring + (size_t)(c % RA_NS) * 2 * SLICE;
    const T* stb = diag ? sta : sta + SLICE;
    const int f0 = c * RA_FC;
    const int nks = (min(RA_FC, p - f0) + 3) >> 2;
    double mr[RA_FC / 4];                                // this lane's chunk means, loaded together
#pragma unroll
    for (int ks = 0; ks < RA_FC / 4; ++ks) mr[ks] = f0 + 4 * ks + tig < p ? mu[f0 + 4 * ks + tig] : 0.0;
    const T* pa = sta + (wr * 32 + gid) * RA_P + tig;
    const T* pb = stb + (wc * 16 + gid) * RA_P + tig;
#pragma unroll
    for (int ks = 0; ks < RA_FC / 4; ++ks) {
      if (ks >= nks) break;
      const double m = mr[ks];
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = (double)pa[i * 8 * RA_P + 4 * ks] - m;
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = (double)pb[j * 8 * RA_P + 4 * ks] - m;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_r(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  double* out = A + d.a_off;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int x = ti * GT + wr * 32 + i * 8 + gid, y = tj * GT + wc * 16 + j * 8 + 2 * tig + v;
        if (x < k && y < k) {
          out[(int64_t)x * k + y] = acc[i][j][v];
          if (!diag) out[(int64_t)y * k + x] = acc[i][j][v];
        }
      }
}

// ------------------------------------------------------------- K3 Jacobi
// Re-solve, with the full Jacobi method, the pieces the Lanczos kernel flagged
// (status NUMERICAL with value -2: Krylov basis capacity exhausted).
__global__ void __launch_bounds__(mdsx::JAC_THREADS)
jacobi_fallback_kernel(const PieceDesc* __restrict__ pd, int r, const double* __restrict__ Aall,
                       double* __restrict__ Uout, double* __restrict__ lam_out,
                       double* __restrict__ estimates, double* __restrict__ gof,
                       mdsx_piece_status* __restrict__ status) {
  extern __shared__ double sm[];
  __shared__ mdsx::PieceScratch ps;
  const PieceDesc d = pd[blockIdx.x];
  const mdsx_piece_status s0 = status[d.id];
  if (!(s0.code == MDSX_NUMERICAL && s0.value == -2.0)) return;
  __syncthreads();
  if (threadIdx.x == 0) status[d.id] = mdsx_piece_status{MDSX_OK, 0, 0.0};
  __syncthreads();
  mdsx::full_jacobi_piece(d, r, Aall, Uout, lam_out, estimates, gof, status, 1, sm, ps);
}

__global__ void __launch_bounds__(mdsx::JAC_THREADS)
jacobi_kernel(const PieceDesc* __restrict__ pd, int r, const double* __restrict__ Aall,
              double* __restrict__ Uout, double* __restrict__ lam_out,
              double* __restrict__ estimates, double* __restrict__ gof,
              mdsx_piece_status* __restrict__ status, int qform_trivial) {
  extern __shared__ double sm[];
  __shared__ mdsx::PieceScratch ps;
  mdsx::full_jacobi_piece(pd[blockIdx.x], r, Aall, Uout, lam_out, estimates, gof, status,
                          qform_trivial, sm, ps);
}

}  // namespace

namespace mdsx {

int launch_jacobi_fallback(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r,
                           double* A, double* U, double* lam, double* estimates, double* gof,
                           mdsx_piece_status* status, cudaStream_t st) {
  if (npieces == 0) return MDSX_OK;
  const int kk = kmax + (kmax & 1);
  const size_t smem = (size_t)2 * kk * kk * sizeof(double);
  cudaFuncSetAttribute(jacobi_fallback_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)smem);
  mdsx::pre(h, st);
  jacobi_fallback_kernel<<<npieces, mdsx::JAC_THREADS, smem, st>>>(pd, r, A, U, lam, estimates,
                                                                   gof, status);
  return launched(h, "jacobi_fallback_kernel", st);
}

int launch_piece_means(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                       const int64_t* row_idx, const PieceDesc* pd, int npieces, double* mu,
                       mdsx_piece_status* status, cudaStream_t st) {
  mdsx::pre(h, st);
  if (dtype == MDSX_F64)
    piece_means_kernel<double><<<npieces, 256, 0, st>>>((const double*)data, ld, p, row_idx, pd, mu,
                                                        status);
  else
    piece_means_kernel<float><<<npieces, 256, 0, st>>>((const float*)data, ld, p, row_idx, pd, mu,
                                                       status);
  return launched(h, "piece_means_kernel", st);
}

int launch_gram(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                const int64_t* row_idx, const PieceDesc* pd, const double* mu, const int4* tiles,
                int ntiles, double* A, cudaStream_t st) {
  if (ntiles == 0) return MDSX_OK;
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  if (((size_t)p * es) % 16 == 0 && ((size_t)ld * es) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(data) & 15) == 0 && !getenv("MDSX_GRAM_ROWS_FMA")) {
    auto go = [&](auto tag) {
      using T = decltype(tag);
      const size_t smem = (size_t)RA_NS * 2 * GT * RA_P * sizeof(T);
      cudaFuncSetAttribute(gram_rows_async_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      mdsx::pre(h, st);
      gram_rows_async_kernel<T><<<ntiles, 256, smem, st>>>((const T*)data, ld, p, row_idx, pd, mu,
                                                           tiles, A);
      return launched(h, "gram_rows_async_kernel", st);
    };
    return dtype == MDSX_F64 ? go(double{}) : go(float{});
  }
  mdsx::pre(h, st);
  if (dtype == MDSX_F64)
    gram_kernel<double><<<ntiles, 256, 0, st>>>((const double*)data, ld, p, row_idx, pd, mu, tiles, A);
  else
    gram_kernel<float><<<ntiles, 256, 0, st>>>((const float*)data, ld, p, row_idx, pd, mu, tiles, A);
  return launched(h, "gram_kernel", st);
}

int launch_jacobi(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r, double* A,
                  double* U, double* lam, double* estimates, double* gof,
                  mdsx_piece_status* status, int qform_trivial, cudaStream_t st) {
  const int kk = kmax + (kmax & 1);
  const size_t smem = (size_t)2 * kk * kk * sizeof(double);
  cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mdsx::pre(h, st);
  jacobi_kernel<<<npieces, mdsx::JAC_THREADS, smem, st>>>(pd, r, A, U, lam, estimates, gof, status,
                                                     qform_trivial);
  return launched(h, "jacobi_kernel", st);
}

}  // namespace mdsx
