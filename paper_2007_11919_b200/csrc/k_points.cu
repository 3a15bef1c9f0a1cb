// Piece configurations X = Xc U_r (form 0) or V_r sqrt(lambda_r) (form 1)
// and the canonical column signs of linalg.py:139-146 (largest |entry|
// positive, lowest index on ties).
//
// points_kernel: grid (row chunk of CH rows, piece).  Row tiles of the
// gathered data are staged in shared memory with coalesced loads (each row is
// a contiguous p-vector), centred, and multiplied by U (p x r, smem); every
// CTA also emits its per-column argmax candidate (|value|, row).
// sign_kernel: one CTA per piece reduces the candidates in fixed order and
// flips the piece's columns.
#include "mdsx_common.cuh"

#include <algorithm>

namespace {

constexpr int CH = 256;       // rows per CTA
constexpr int PT = 256;       // threads

// Thread (row i, column group g) computes the 4 columns [4g, 4g+4) of row i:
// x loads from the row tile, U loads are warp-broadcasts, no predication.
template <typename T>
__global__ void __launch_bounds__(PT)
points_kernel(const T* __restrict__ X, int64_t ld, int p, const int64_t* __restrict__ row_idx,
              const PieceDesc* __restrict__ pd, int r, const double* __restrict__ mu_all,
              const double* __restrict__ Uall, const double* __restrict__ lam_all,
              double* __restrict__ points, double2* __restrict__ cand, int maxch, int tr) {
  extern __shared__ double sm[];
  __shared__ double bval[PT];
  __shared__ int bidx[PT];
  const PieceDesc d = pd[blockIdx.y];
  const int chunk = blockIdx.x;
  const int r0 = chunk * CH;
  if (r0 >= d.m) return;
  const int rows = min(CH, d.m - r0);
  const int tid = threadIdx.x;
  const int64_t* ridx = row_idx + d.row_off + r0;
  double* out = points + (d.pt_off + r0) * r;
  const double* Ug = Uall + d.u_off;
  const int G = (r + 3) / 4;                   // column groups of 4
  const int rp = 4 * G;                        // padded r
  const int i_loc = tid % tr, g = tid / tr;
  const bool worker = g < G;

  double best[4];
  int bi[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) { best[j] = -1.0; bi[j] = 0x7fffffff; }

  if (d.form == 1) {
    for (int i = tid; i < rows; i += PT)
      for (int c = 0; c < r; ++c) {
        const double v = Ug[(int64_t)(r0 + i) * r + c] * sqrt(lam_all[(int64_t)d.id * r + c]);
        out[(int64_t)i * r + c] = v;
      }
  } else {
    const int pp = p + 1;                        // padded tile row (conflict-free)
    double* sU = sm;                             // p x rp
    double* smu = sU + (size_t)p * rp;           // p
    double* tile = smu + p;                      // tr x pp
    for (int e = tid; e < p * rp; e += PT) {
      const int a = e / rp, c = e % rp;
      sU[e] = c < r ? Ug[(int64_t)a * r + c] : 0.0;
    }
    for (int e = tid; e < p; e += PT) smu[e] = mu_all[(int64_t)d.id * p + e];
    for (int t0 = 0; t0 < rows; t0 += tr) {
      const int nr = min(tr, rows - t0);
      __syncthreads();
      for (int i = tid / 32; i < nr; i += PT / 32) {   // warp per row: coalesced
        const T* src = X + ridx[t0 + i] * ld;
        for (int a = tid % 32; a < p; a += 32) tile[i * pp + a] = mdsx::ld_val(src + a) - smu[a];
      }
      __syncthreads();
      if (worker && i_loc < nr) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const double* xr = tile + i_loc * pp;
        const double* ug = sU + 4 * g;
        for (int a = 0; a < p; ++a) {
          const double x = xr[a];
          const double2 u01 = *reinterpret_cast<const double2*>(ug + a * rp);
          const double2 u23 = *reinterpret_cast<const double2*>(ug + a * rp + 2);
          acc[0] = fma(x, u01.x, acc[0]);
          acc[1] = fma(x, u01.y, acc[1]);
          acc[2] = fma(x, u23.x, acc[2]);
          acc[3] = fma(x, u23.y, acc[3]);
        }
        const int i = t0 + i_loc;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = 4 * g + j;
          if (c < r) {
            out[(int64_t)i * r + c] = acc[j];
            if (fabs(acc[j]) > best[j]) { best[j] = fabs(acc[j]); bi[j] = r0 + i; }
          }
        }
      }
    }
  }
  // per-CTA candidates per column (ties -> lowest row), fixed-order tree
  for (int c = 0; c < r; ++c) {
    __syncthreads();
    double v = -1.0;
    int ix = 0x7fffffff;
    if (d.form == 1) {
      for (int i = tid; i < rows; i += PT) {
        const double a = fabs(out[(int64_t)i * r + c]);
        if (a > v) { v = a; ix = r0 + i; }
      }
    } else if (worker && c / 4 == g) {
      v = best[c % 4];
      ix = bi[c % 4];
    }
    bval[tid] = v;
    bidx[tid] = ix;
    __syncthreads();
    for (int s = PT / 2; s > 0; s >>= 1) {
      if (tid < s) {
        const double v2 = bval[tid + s];
        const int i2 = bidx[tid + s];
        if (v2 > bval[tid] || (v2 == bval[tid] && i2 < bidx[tid])) { bval[tid] = v2; bidx[tid] = i2; }
      }
      __syncthreads();
    }
    if (tid == 0) cand[((size_t)d.id * maxch + chunk) * r + c] = make_double2(bval[0], (double)bidx[0]);
  }
}

__global__ void __launch_bounds__(PT)
sign_kernel(const PieceDesc* __restrict__ pd, int r, const double2* __restrict__ cand, int maxch,
            double* __restrict__ points) {
  __shared__ double sgn[MDSX_MAX_R];
  const PieceDesc d = pd[blockIdx.x];
  const int nch = (d.m + CH - 1) / CH;
  double* out = points + d.pt_off * r;
  if (threadIdx.x < r) {
    const int c = threadIdx.x;
    double bv = -1.0;
    int bi = 0x7fffffff;
    for (int ch = 0; ch < nch; ++ch) {
      const double2 e = cand[((size_t)d.id * maxch + ch) * r + c];
      const int i = (int)e.y;
      if (e.x > bv || (e.x == bv && i < bi)) { bv = e.x; bi = i; }
    }
    double s = 1.0;
    if (bi < d.m && out[(int64_t)bi * r + c] < 0.0) s = -1.0;
    sgn[c] = s;
  }
  __syncthreads();
  for (int64_t e = threadIdx.x; e < (int64_t)d.m * r; e += PT) {
    const int c = (int)(e % r);
    if (sgn[c] < 0.0) out[e] = -out[e];
  }
}

}  // namespace

namespace mdsx {

size_t points_ws_bytes(int npieces, int64_t max_m, int r) {
  const int64_t maxch = (max_m + CH - 1) / CH;
  return (size_t)npieces * maxch * r * sizeof(double2);
}

int launch_points(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                  const int64_t* row_idx, const PieceDesc* pd, int npieces, int64_t max_m, int r,
                  const double* mu, const double* U, const double* lam, double* points,
                  double2* cand, cudaStream_t st) {
  const int maxch = (int)((max_m + CH - 1) / CH);
  const int G = (r + 3) / 4, rp = 4 * G;
  // rows per tile: one per thread group, limited by the ~200 KB smem budget
  int tr = PT / G;
  const size_t fixed = ((size_t)p * rp + p) * sizeof(double);
  while (tr > 8 && fixed + (size_t)tr * (p + 1) * sizeof(double) > 200 * 1024) tr >>= 1;
  const size_t smem = fixed + (size_t)tr * (p + 1) * sizeof(double);
  dim3 grid((unsigned)maxch, (unsigned)npieces);
  int rc;
  if (dtype == MDSX_F32) {
    cudaFuncSetAttribute(points_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mdsx::pre(h, st);
    points_kernel<float><<<grid, PT, smem, st>>>((const float*)data, ld, p, row_idx, pd, r, mu, U,
                                                 lam, points, cand, maxch, tr);
  } else {
    cudaFuncSetAttribute(points_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mdsx::pre(h, st);
    points_kernel<double><<<grid, PT, smem, st>>>((const double*)data, ld, p, row_idx, pd, r, mu,
                                                  U, lam, points, cand, maxch, tr);
  }
  if ((rc = launched(h, "points_kernel", st))) return rc;
  mdsx::pre(h, st);
  sign_kernel<<<npieces, PT, 0, st>>>(pd, r, cand, maxch, points);
  return launched(h, "sign_kernel", st);
}

}  // namespace mdsx
