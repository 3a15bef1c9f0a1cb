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
#include "points_stream.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

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
    // form 0: double-buffered 32-row tiles; every thread owns EPT tile elements
    // (loads issued for tile t+1 before the FMAs on tile t)
    const int pp = p + 1;                        // padded tile row (conflict-free)
    double* sU = sm;                             // p x rp
    double* smu = sU + (size_t)p * rp;           // p
    double* tiles = smu + p;                     // 2 x tr x pp
    for (int e = tid; e < p * rp; e += PT) {
      const int a = e / rp, c = e % rp;
      sU[e] = c < r ? Ug[(int64_t)a * r + c] : 0.0;
    }
    for (int e = tid; e < p; e += PT) smu[e] = mu_all[(int64_t)d.id * p + e];
    __syncthreads();
    // row offsets of this CTA's rows, staged once (no dependent index loads per element)
    __shared__ int64_t rbase[CH];
    for (int i = tid; i < rows; i += PT) rbase[i] = ridx[i] * ld;
    const int ntiles = (rows + tr - 1) / tr;
    const int rpw = tr / (PT / 32);              // rows per warp per tile (tr is a multiple of 8)
    const int lane = tid & 31, wq = tid >> 5;
    constexpr int EPT = 16;                      // 4 rows x 4 columns (128-column block) per lane
    double pre[EPT];
    auto fetch = [&](int t, int pass) {
      const int t0 = t * tr, nr = min(tr, rows - t0);
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int j = q >> 2, a = pass * 128 + lane + 32 * (q & 3);
        const int rr = wq * rpw + j;
        // raw values only: consuming them here would stall on the loads
        pre[q] = (j < rpw && rr < nr && a < p) ? mdsx::ld_val(X + rbase[t0 + rr] + a) : 0.0;
      }
    };
    auto store = [&](int b, int pass) {
      double* tb = tiles + (size_t)b * tr * pp;
#pragma unroll
      for (int q = 0; q < EPT; ++q) {
        const int j = q >> 2, a = pass * 128 + lane + 32 * (q & 3);
        if (j < rpw && a < p) tb[(wq * rpw + j) * pp + a] = pre[q] - smu[a];
      }
    };
    __syncthreads();
    const int passes = (p + 127) / 128;
    for (int pass = 0; pass < passes; ++pass) { fetch(0, pass); store(0, pass); }
    __syncthreads();
    for (int t = 0; t < ntiles; ++t) {
      const int b = t & 1;
      const bool more = t + 1 < ntiles;
      if (more) fetch(t + 1, 0);                 // first pass in flight during the FMAs
      const int t0 = t * tr, nr = min(tr, rows - t0);
      if (worker && i_loc < nr) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        const double* xr = tiles + (size_t)b * tr * pp + i_loc * pp;
        const double* ug = sU + 4 * g;
#pragma unroll 4
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
      if (more) {
        store(b ^ 1, 0);
        for (int pass = 1; pass < passes; ++pass) { fetch(t + 1, pass); store(b ^ 1, pass); }
      }
      __syncthreads();
    }
  }
  // per-CTA candidates per column (ties -> lowest row): warp shuffles, then
  // one fixed-order pass over the 8 warp results
  __shared__ double wv_s[PT / 32][MDSX_MAX_R];
  __shared__ int wi_s[PT / 32][MDSX_MAX_R];
  const int lane = tid & 31, warp = tid >> 5;
  for (int c = 0; c < r; ++c) {
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
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, ix, o);
      if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
    }
    if (lane == 0) { wv_s[warp][c] = v; wi_s[warp][c] = ix; }
  }
  __syncthreads();
  if (tid < r) {
    double v = -1.0;
    int ix = 0x7fffffff;
    for (int w = 0; w < PT / 32; ++w) {
      const double v2 = wv_s[w][tid];
      const int i2 = wi_s[w][tid];
      if (v2 > v || (v2 == v && i2 < ix)) { v = v2; ix = i2; }
    }
    cand[((size_t)d.id * maxch + chunk) * r + tid] = make_double2(v, (double)ix);
  }
}


// ---- form 0, 16-byte aligned rows (points_stream.cuh).  Grid (chunks, pieces):
// chunks == 1 -> one CTA per piece, signs applied in the CTA; otherwise each
// CTA takes CH rows and leaves its column candidates for sign_kernel (few
// pieces: spread one piece over several SMs).  `pending` (optional): only
// pieces with pending[id] != 0 -- the ones whose points the fused Lanczos
// epilogue did not produce.
template <typename T, int RM>
__global__ void __launch_bounds__(mdsx::PS_T, 2)
points_piece_kernel(const T* __restrict__ X, int64_t ld, int p, const int64_t* __restrict__ row_idx,
                    const PieceDesc* __restrict__ pd, int r, const double* __restrict__ mu_all,
                    const double* __restrict__ Uall, double* __restrict__ points,
                    const int* __restrict__ pending, double2* __restrict__ cand, int maxch) {
  extern __shared__ __align__(16) unsigned char pr_smem[];
  const PieceDesc d = pd[blockIdx.y];
  if (pending && !pending[d.id]) return;
  const bool chunked = gridDim.x > 1;
  const int r0 = chunked ? blockIdx.x * CH : 0;
  if (r0 >= d.m) return;
  const int rows = chunked ? min(CH, d.m - r0) : d.m;
  mdsx::PieceStream<T, RM> ps(pr_smem, X, ld, row_idx + d.row_off + r0, p, rows);
  ps.prologue();
  mdsx::ps_load_records<RM>(pr_smem, Uall + d.u_off, mu_all + (int64_t)d.id * p, p, r);
  __syncthreads();
  ps.run(pr_smem, r, points + (d.pt_off + r0) * r,
         chunked ? cand + ((size_t)d.id * maxch + blockIdx.x) * r : nullptr, r0);
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

// Signs for the chunked points_piece_kernel: candidates hold the SIGNED value
// of each chunk's largest |entry| (x) and its row (y); grid (chunks, pieces),
// every CTA reduces the piece's candidates (fixed order, lowest row on ties)
// and flips its own chunk's rows.
__global__ void __launch_bounds__(PT)
sign_chunk_kernel(const PieceDesc* __restrict__ pd, int r, const double2* __restrict__ cand,
                  int maxch, double* __restrict__ points) {
  __shared__ double sgn[MDSX_MAX_R];
  const PieceDesc d = pd[blockIdx.y];
  const int r0 = blockIdx.x * CH;
  if (r0 >= d.m) return;
  const int nch = (d.m + CH - 1) / CH;
  if (threadIdx.x < r) {
    const int c = threadIdx.x;
    double bv = -1.0, bs = 1.0;
    int bi = 0x7fffffff;
    for (int ch = 0; ch < nch; ++ch) {
      const double2 e = cand[((size_t)d.id * maxch + ch) * r + c];
      const int i = (int)e.y;
      const double a = fabs(e.x);
      if (a > bv || (a == bv && i < bi)) { bv = a; bi = i; bs = e.x < 0.0 ? -1.0 : 1.0; }
    }
    sgn[c] = bs;
  }
  __syncthreads();
  double* out = points + (d.pt_off + r0) * r;
  const int rows = min(CH, d.m - r0);
  for (int e = threadIdx.x; e < rows * r; e += PT) {
    const int c = e % r;
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
                  double2* cand, cudaStream_t st, bool all_form0, const int* pending) {
  const int maxch = (int)((max_m + CH - 1) / CH);
  const int G = (r + 3) / 4, rp = 4 * G;
  // tile rows: 32 (one per lane) unless the double buffer would not fit
  int tr = 32;
  const size_t fixed = ((size_t)p * rp + p) * sizeof(double);
  while (tr > 8 && fixed + 2 * (size_t)tr * (p + 1) * sizeof(double) > 200 * 1024) tr >>= 1;
  if (tr * G > PT) tr = PT / G;
  const size_t smem = fixed + 2 * (size_t)tr * (p + 1) * sizeof(double);
  dim3 grid((unsigned)maxch, (unsigned)npieces);
  int rc;
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  // form-0 pieces with 16-byte aligned rows: per-thread cp.async row streams
  // (a piece batch is all form 0 here whenever p < every m; form-1 pieces and
  // unaligned data use the tiled kernel)
  const bool rows_ok = data != nullptr && r <= 16 && ((size_t)p * es) % 16 == 0 &&
                       ((size_t)ld * es) % 16 == 0 && (reinterpret_cast<uintptr_t>(data) & 15) == 0 &&
                       !getenv("MDSX_POINTS_TILED");
  if (rows_ok && all_form0) {
    // few pieces (e.g. the landmark set of interpolation): CH-row chunks over
    // several CTAs + sign_kernel; many pieces: one CTA per piece
    const int chunks = (npieces < 2 * h->num_sms && !pending) ? maxch : 1;
    const int RM = r <= 4 ? 4 : r <= 8 ? 8 : r <= 10 ? 10 : r <= 12 ? 12 : 16;
    auto go = [&](auto tag, auto rm) {
      using T = decltype(tag);
      constexpr int RMc = decltype(rm)::value;
      const size_t smem2 = mdsx::ps_smem_bytes<RMc>(p);
      auto kern = points_piece_kernel<T, RMc>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
      mdsx::pre(h, st);
      kern<<<dim3(chunks, npieces), mdsx::PS_T, smem2, st>>>((const T*)data, ld, p, row_idx, pd, r,
                                                             mu, U, points, pending, cand, maxch);
      return launched(h, "points_piece_kernel", st);
    };
    auto by_rm = [&](auto tag) {
      switch (RM) {
        case 4: return go(tag, std::integral_constant<int, 4>{});
        case 8: return go(tag, std::integral_constant<int, 8>{});
        case 10: return go(tag, std::integral_constant<int, 10>{});
        case 12: return go(tag, std::integral_constant<int, 12>{});
        default: return go(tag, std::integral_constant<int, 16>{});
      }
    };
    int rc2 = dtype == MDSX_F32 ? by_rm(float{}) : by_rm(double{});
    if (rc2 || chunks == 1) return rc2;
    mdsx::pre(h, st);
    sign_chunk_kernel<<<dim3(chunks, npieces), PT, 0, st>>>(pd, r, cand, maxch, points);
    return launched(h, "sign_chunk_kernel", st);
  }
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
