// Divide-and-conquer tail without per-piece point matrices
// (algorithms.py:146-166): the configuration of piece j is P_j = (X_j - mu_j) U_j
// (k = p feature space, U_j the top-r eigenvectors of the centred Gram), and
// the output rows are P_j T_j + t_j - mean.  Only three things need points:
//   * the anchor (piece 1, all rows): the canonical column signs
//     (linalg.py:139-146) of the frame every other piece is aligned to, and
//     its first c rows as the Procrustes target;
//   * every other piece's first c (connecting) rows: the Procrustes source.
//     A piece's own column signs never matter: they are absorbed by its fit
//     (P S T' = P T for T' = S T);
//   * the column mean of the output, which follows from the connecting rows:
//     sum_own (x - mu_j) = -sum_conn (x - mu_j) because the centred rows of a
//     piece sum to zero, so mean = (1/n) sum_j [-(sum_i<c P_j[i]) T_j + n_own_j t_j].
// Everything else is ONE pass over the rows (dc_out_kernel): out[row] =
// (x - mu_j) U'_j + t_j - mean with U'_j = U_j T_j, on the fp64 tensor pipe
// (DMMA m8n8k4: 8 rows x 8 columns per fragment, U' held in registers).
#include "mdsx_common.cuh"
#include "bulk.cuh"

#include <algorithm>
#include <type_traits>

namespace {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int RMX = 16;            // r handled here

// Points of rows [first, first + count) of pieces pbase + blockIdx.x (count <= 0:
// every row from `first`), unsigned U: one warp per row, lanes over features,
// r warp sums.  Row i of piece j goes to dst[(j - pbase) * dst_stride + i - first].
template <typename T>
__global__ void __launch_bounds__(128)
dc_rows_kernel(const T* __restrict__ X, int64_t ld, int p, const int64_t* __restrict__ row_idx,
               const PieceDesc* __restrict__ pd, int pbase, int r, int first, int count,
               const double* __restrict__ mu_all, const double* __restrict__ Uall,
               double* __restrict__ dst, int64_t dst_stride) {
  const PieceDesc d = pd[pbase + blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* U = Uall + d.u_off;
  const double* mu = mu_all + (int64_t)d.id * p;
  const int last = count > 0 ? min(d.m, first + count) : d.m;
  for (int i = first + blockIdx.y * 4 + warp; i < last; i += 4 * gridDim.y) {
    const T* row = X + row_idx[d.row_off + i] * ld;
    double acc[RMX];
#pragma unroll
    for (int q = 0; q < RMX; ++q) acc[q] = 0.0;
    for (int a = lane; a < p; a += 32) {
      const double y = (double)row[a] - mu[a];
#pragma unroll
      for (int q = 0; q < RMX; ++q)
        if (q < r) acc[q] = fma(y, U[a * r + q], acc[q]);
    }
    double* o = dst + (int64_t)blockIdx.x * dst_stride + (int64_t)(i - first) * r;
#pragma unroll
    for (int q = 0; q < RMX; ++q) {
      if (q >= r) break;
      const double v = mdsx::warp_sum(acc[q]);
      if (lane == 0) o[q] = v;
    }
  }
}

// Canonical column signs of the anchor's points Pa (m x r): largest |value|
// positive, lowest row on ties (linalg.py:139-146); U_0 flipped in place, the
// signed first c rows -> tgt.
__global__ void __launch_bounds__(256)
dc_sign_kernel(const double* __restrict__ Pa, const PieceDesc* __restrict__ pd, int r, int c,
               double* __restrict__ Uall, double* __restrict__ tgt, int p) {
  __shared__ double bv[256];
  __shared__ int bi[256];
  __shared__ double sgn[RMX];
  const PieceDesc d = pd[0];
  const int G = 256 / r;
  const int q = threadIdx.x % r, g = threadIdx.x / r;
  double v = 0.0;
  int ix = 0x7fffffff;
  if (g < G)
    for (int i = g; i < d.m; i += G) {                 // rows ascending per thread
      const double x = Pa[(int64_t)i * r + q];
      if (ix == 0x7fffffff || fabs(x) > fabs(v)) { v = x; ix = i; }
    }
  bv[threadIdx.x] = v;
  bi[threadIdx.x] = g < G ? ix : 0x7fffffff;
  __syncthreads();
  if (threadIdx.x < r) {
    double bvv = 0.0;
    int bix = 0x7fffffff;
    for (int u = 0; u < G; ++u) {
      const double v2 = bv[u * r + threadIdx.x];
      const int i2 = bi[u * r + threadIdx.x];
      if (i2 != 0x7fffffff &&
          (bix == 0x7fffffff || fabs(v2) > fabs(bvv) || (fabs(v2) == fabs(bvv) && i2 < bix))) {
        bvv = v2;
        bix = i2;
      }
    }
    sgn[threadIdx.x] = bvv < 0.0 ? -1.0 : 1.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < c * r; e += 256) tgt[e] = Pa[e] * sgn[e % r];
  double* U = Uall + d.u_off;
  for (int e = threadIdx.x; e < p * r; e += 256) U[e] *= sgn[e % r];
}

// U'_j = U_j T_j, tvec_j = t_j (piece 0: U_0, already signed, t = 0) and the
// column-mean contribution -(sum_i<c P_j[i]) T_j + (m_j - c) t_j.
__global__ void __launch_bounds__(128)
dc_compose_kernel(const PieceDesc* __restrict__ pd, int pbase, int p, int r, int c,
                  const double* __restrict__ Uall, const double* __restrict__ rot,
                  const double* __restrict__ trans, const double* __restrict__ src,
                  double* __restrict__ Uc, double* __restrict__ tvec, double* __restrict__ contrib,
                  const int32_t* __restrict__ pending) {
  const int j = pbase + blockIdx.x;
  if (pending != nullptr && j > 0 && pending[j] == 0) return;   // composed by dc_fit_kernel
  const PieceDesc d = pd[j];
  const double* U = Uall + d.u_off;
  double* O = Uc + (int64_t)j * p * r;
  __shared__ double Ts[RMX * RMX], cs[RMX];
  if (j == 0) {
    for (int e = threadIdx.x; e < p * r; e += blockDim.x) O[e] = U[e];
    if (threadIdx.x < r) {
      contrib[threadIdx.x] = 0.0;
      tvec[threadIdx.x] = 0.0;
    }
    return;
  }
  const double* Tj = rot + (int64_t)(j - 1) * r * r;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) Ts[e] = Tj[e];
  if (threadIdx.x < r) {
    double s = 0.0;
    for (int i = 0; i < c; ++i) s += src[((int64_t)j * c + i) * r + threadIdx.x];
    cs[threadIdx.x] = s;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < p * r; e += blockDim.x) {
    const int a = e / r, q = e - a * r;
    double v = 0.0;
    for (int b = 0; b < r; ++b) v = fma(U[a * r + b], Ts[b * r + q], v);
    O[e] = v;
  }
  if (threadIdx.x < r) {
    const int q = threadIdx.x;
    double v = 0.0;
    for (int b = 0; b < r; ++b) v = fma(cs[b], Ts[b * r + q], v);
    const double t = trans[(int64_t)(j - 1) * r + q];
    tvec[(int64_t)j * r + q] = t;
    contrib[(int64_t)j * r + q] = (double)(d.m - c) * t - v;
  }
}

// mean = sum_j contrib_j / n in a fixed order (thread (q, g) sums pieces
// g, g + G, ...; the G partials of a column are then added in order)
__global__ void __launch_bounds__(256)
dc_mean2_kernel(const double* __restrict__ contrib, int npieces, int r, double inv_n,
                double* __restrict__ mean) {
  __shared__ double part[256];
  const int G = 256 / r;
  const int q = threadIdx.x % r, g = threadIdx.x / r;
  double s = 0.0;
  if (g < G)
    for (int j = g; j < npieces; j += G) s += contrib[(int64_t)j * r + q];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x < r) {
    double t = 0.0;
    for (int u = 0; u < G; ++u) t += part[u * r + threadIdx.x];
    mean[threadIdx.x] = t * inv_n;
  }
}

// The output pass: out[oidx[row]] = (x - mu_j) Uc_j + tvec_j - mean for the
// rows [first_j, m_j) of piece j (first_j = 0 for piece 0 or when c0 == 0,
// else c0).  Grid (row ranges of up to PO_ROWS rows, pieces).  Rows reach
// shared memory through the same warp-specialised ring as the Gram: a
// producer warp gathers PO_KC rows per stage, one cp.async.bulk per row (row
// index loaded two stages ahead), on the stage's `full` mbarrier; each of the
// 4 compute warps takes one 8-row tile of a stage on the fp64 tensor pipe
// (m8n8k4, the K range split over two accumulator sets) and releases the
// stage on its `empty` mbarrier.  U' fragments live in registers for the whole
// CTA, the piece mean in shared memory; the stage pitch P (== 4 mod 16
// doubles) makes the fragment loads conflict-free and the padding columns
// [p, P) are zero.
constexpr int PO_THREADS = 128;   // compute warps
constexpr int PO_CTA = PO_THREADS + 32;
constexpr int PO_KC = 32;         // rows per stage (one per producer lane, 4 tiles of 8)
constexpr int PO_NS = 4;          // stages
constexpr int PO_ROWS = 1024;     // rows per CTA
constexpr int PO_HDR = 2048;      // mbarriers + piece mean

template <typename T, int K4, int NT>
__global__ void __launch_bounds__(PO_CTA, 2)
piece_out_kernel(const T* __restrict__ X, int64_t ld, int p, int P, const int64_t* __restrict__ row_idx,
                 const int64_t* __restrict__ out_idx, const PieceDesc* __restrict__ pd, int r, int c0,
                 const double* __restrict__ mu_all, const double* __restrict__ Uc,
                 const double* __restrict__ tvec, const double* __restrict__ mean,
                 double* __restrict__ out) {
  extern __shared__ __align__(128) unsigned char do_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(do_smem);
  uint64_t* empty = full + PO_NS;
  double* smu = reinterpret_cast<double*>(do_smem + 128);           // 4 K4 <= 128
  T* stage = reinterpret_cast<T*>(do_smem + PO_HDR);
  const int j = blockIdx.y;                       // local piece (Uc, tvec are offset)
  const PieceDesc d = pd[j];
  const int first = d.id == 0 ? 0 : c0;
  const int r0 = first + blockIdx.x * PO_ROWS;
  if (r0 >= d.m) return;
  const int nrows = min(PO_ROWS, d.m - r0);
  const int nch = (nrows + PO_KC - 1) / PO_KC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t* ridx = row_idx + d.row_off + r0;
  const int64_t* oidx = (out_idx ? out_idx : row_idx) + d.row_off + r0;
  const size_t stage_elems = (size_t)PO_KC * P;
  for (int e = tid; e < 4 * K4; e += PO_CTA) smu[e] = e < p ? mu_all[(int64_t)d.id * p + e] : 0.0;
  for (int e = tid; P > p && e < PO_NS * PO_KC * (P - p); e += PO_CTA)
    stage[(size_t)(e / (P - p)) * P + p + e % (P - p)] = T(0);
  if (tid == 0) {
    for (int s = 0; s < PO_NS; ++s) {
      bulk::bar_init(&full[s], 1);
      bulk::bar_init(&empty[s], PO_THREADS / 32);
    }
    bulk::bar_fence();
  }
  __syncthreads();

  if (warp == PO_THREADS / 32) {                  // ---- producer
    const unsigned row_bytes = (unsigned)((size_t)p * sizeof(T));
    int64_t nidx = lane < nrows ? ridx[lane] : 0;
    int64_t nidx2 = PO_KC + lane < nrows ? ridx[PO_KC + lane] : 0;
    for (int c = 0; c < nch; ++c) {
      const int s = c % PO_NS;
      const int b0 = c * PO_KC, nr = min(PO_KC, nrows - b0);
      const int64_t idx = nidx;
      nidx = nidx2;
      if (b0 + 2 * PO_KC + lane < nrows) nidx2 = ridx[b0 + 2 * PO_KC + lane];
      if (c >= PO_NS) bulk::wait(&empty[s], (unsigned)((c / PO_NS - 1) & 1));
      if (lane == 0) bulk::arrive_expect(&full[s], (unsigned)nr * row_bytes);
      __syncwarp();
      if (lane < nr)
        bulk::copy(stage + (size_t)s * stage_elems + (size_t)lane * P, X + idx * ld, row_bytes, &full[s]);
    }
    return;
  }

  // ---- compute warps
  const double* U = Uc + (int64_t)j * p * r;
  double bf[K4][NT];
#pragma unroll
  for (int k4 = 0; k4 < K4; ++k4) {
    const int a = 4 * k4 + tig;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int q = 8 * n + gid;
      bf[k4][n] = (a < p && q < r) ? U[a * r + q] : 0.0;
    }
  }
  double add[NT][2];
#pragma unroll
  for (int n = 0; n < NT; ++n)
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int q = 8 * n + 2 * tig + v;
      add[n][v] = q < r ? tvec[(int64_t)j * r + q] - mean[q] : 0.0;
    }
  for (int c = 0; c < nch; ++c) {
    const int s = c % PO_NS;
    const int b0 = c * PO_KC, nr = min(PO_KC, nrows - b0);
    const int tr = 8 * warp;                       // this warp's tile: stage rows tr .. tr+7
    const int row = b0 + tr + gid;
    // output row index loaded before the wait: its latency hides under the DMMAs
    const int64_t orow = tr + gid < nr ? oidx[row] : 0;
    bulk::wait(&full[s], (unsigned)((c / PO_NS) & 1));
    double acc[NT][4][2];                          // K range split over four accumulator sets
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int hh = 0; hh < 4; ++hh) acc[n][hh][0] = acc[n][hh][1] = 0.0;
    if (tr < nr) {
      const T* x0 = stage + (size_t)s * stage_elems + (size_t)(tr + gid) * P + tig;
#pragma unroll
      for (int k4 = 0; k4 < K4; ++k4) {
        const double xa = (double)x0[4 * k4] - smu[4 * k4 + tig];
#pragma unroll
        for (int n = 0; n < NT; ++n) dmma(acc[n][k4 & 3][0], acc[n][k4 & 3][1], xa, bf[k4][n]);
      }
    }
    __syncwarp();
    if (lane == 0) bulk::arrive(&empty[s]);
    // lane (gid, tig) holds out[row gid of the tile][8n + 2tig + v]
    if (tr + gid < nr) {
      double* o = out + orow * r;
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int q = 8 * n + 2 * tig;
        const double v0 = (acc[n][0][0] + acc[n][1][0]) + (acc[n][2][0] + acc[n][3][0]) + add[n][0];
        const double v1 = (acc[n][0][1] + acc[n][1][1]) + (acc[n][2][1] + acc[n][3][1]) + add[n][1];
        if (q + 1 < r && !(r & 1)) {             // 16-byte aligned pair (row stride r doubles, r even)
          *reinterpret_cast<double2*>(o + q) = make_double2(v0, v1);
        } else if (q + 1 < r) {
          o[q] = v0;
          o[q + 1] = v1;
        } else if (q < r) {
          o[q] = v0;
        }
      }
    }
  }
}

static int dco_pitch(int p, size_t es) {
  int P = p;
  if (es == 8) { while (P % 16 != 4) ++P; }
  else { while (P % 32 != 8) ++P; }
  return P;
}

}  // namespace

namespace mdsx {

bool dc_out_route_ok(const void* data, int dtype, int64_t ld, int p, int r, int c) {
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  return data != nullptr && p <= 128 && r <= RMX && c >= 1 &&
         ((size_t)p * es) % 16 == 0 && ((size_t)ld * es) % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(data) & 15) == 0;
}

size_t dc_out_ws_doubles(int npieces, int p, int r, int c, int64_t m0) {
  return (size_t)npieces * c * r + (size_t)npieces * p * r + 2 * (size_t)npieces * r +
         (size_t)m0 * r + 64;
}

int launch_rows_points(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                       const int64_t* row_idx, const PieceDesc* pd, int pbase, int npieces, int r,
                       int first, int count, int64_t rows_hint, const double* mu, const double* U,
                       double* dst, int64_t dst_stride, cudaStream_t st) {
  if (npieces <= 0) return MDSX_OK;
  const int gy = (int)std::max<int64_t>(1, std::min<int64_t>(64, (rows_hint + 31) / 32));
  mdsx::pre(h, st);
  if (dtype == MDSX_F32)
    dc_rows_kernel<float><<<dim3(npieces, gy), 128, 0, st>>>((const float*)data, ld, p, row_idx, pd,
                                                            pbase, r, first, count, mu, U, dst, dst_stride);
  else
    dc_rows_kernel<double><<<dim3(npieces, gy), 128, 0, st>>>((const double*)data, ld, p, row_idx, pd,
                                                             pbase, r, first, count, mu, U, dst, dst_stride);
  return launched(h, "rows_points_kernel", st);
}

// Anchor: points of piece 0, canonical signs (U_0 flipped, signed targets in
// Pc rows 0..c).
int launch_dc_points(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                     const int64_t* row_idx, const PieceDesc* pd, int npieces, int r, int c,
                     int64_t m0, const double* mu, double* U, double* Pc, double* Pa,
                     cudaStream_t st) {
  (void)npieces;
  int rc;
  if ((rc = launch_rows_points(h, data, dtype, ld, p, row_idx, pd, 0, 1, r, 0, 0, m0, mu, U, Pa, 0, st)))
    return rc;
  mdsx::pre(h, st);
  dc_sign_kernel<<<1, 256, 0, st>>>(Pa, pd, r, c, U, Pc, p);
  return launched(h, "dc_sign_kernel", st);
}

// Connecting rows (first c) of pieces pbase .. pbase+count-1 -> Pc[j * c ..].
int launch_dc_conn(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                   const int64_t* row_idx, const PieceDesc* pd, int pbase, int count, int r, int c,
                   const double* mu, const double* U, double* Pc, cudaStream_t st) {
  return launch_rows_points(h, data, dtype, ld, p, row_idx, pd, pbase, count, r, 0, c, c, mu, U,
                            Pc + (int64_t)pbase * c * r, (int64_t)c * r, st);
}

int launch_dc_compose(mdsx_handle* h, const PieceDesc* pd, int pbase, int count, int p, int r, int c,
                      const double* U, const double* rot, const double* trans, const double* Pc,
                      double* Uc, double* tvec, double* contrib, cudaStream_t st,
                      const int32_t* pending) {
  if (count <= 0) return MDSX_OK;
  mdsx::pre(h, st);
  dc_compose_kernel<<<count, 128, 0, st>>>(pd, pbase, p, r, c, U, rot, trans, Pc, Uc, tvec, contrib,
                                           pending);
  return launched(h, "dc_compose_kernel", st);
}

int launch_piece_out(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                     const int64_t* row_idx, const int64_t* out_idx, const PieceDesc* pd,
                     int npieces, int64_t max_m, int r, int c0, const double* mu, const double* Uc,
                     const double* tvec, const double* mean, double* out, cudaStream_t st) {
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  const dim3 grid((unsigned)((max_m + PO_ROWS - 1) / PO_ROWS), (unsigned)npieces);
  auto go = [&](auto tag, auto k4, auto nt) {
    using Tt = decltype(tag);
    constexpr int K4 = decltype(k4)::value;
    constexpr int NT = decltype(nt)::value;
    const int P = dco_pitch(std::max(p, 4 * K4), es);      // fragment loads stay inside the row
    const size_t smem = PO_HDR + (size_t)PO_NS * PO_KC * P * es;
    auto kern = piece_out_kernel<Tt, K4, NT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mdsx::pre(h, st);
    kern<<<grid, PO_CTA, smem, st>>>((const Tt*)data, ld, p, P, row_idx, out_idx, pd, r, c0, mu, Uc,
                                     tvec, mean, out);
    return launched(h, "piece_out_kernel", st);
  };
  auto by_k = [&](auto tag, auto nt) {
    const int k4 = (p + 3) / 4;
    if (k4 <= 8) return go(tag, std::integral_constant<int, 8>{}, nt);
    if (k4 <= 16) return go(tag, std::integral_constant<int, 16>{}, nt);
    if (k4 == 25) return go(tag, std::integral_constant<int, 25>{}, nt);
    if (k4 <= 26) return go(tag, std::integral_constant<int, 26>{}, nt);
    return go(tag, std::integral_constant<int, 32>{}, nt);
  };
  auto by_nt = [&](auto tag) {
    return r <= 8 ? by_k(tag, std::integral_constant<int, 1>{}) : by_k(tag, std::integral_constant<int, 2>{});
  };
  return dtype == MDSX_F32 ? by_nt(float{}) : by_nt(double{});
}

int launch_shift_rows(mdsx_handle* h, double* X, const int64_t* idx, int64_t n, int r,
                      const double* shift, cudaStream_t st);

// Column mean of the D&C output from the per-piece contributions (fixed order).
int launch_dc_mean(mdsx_handle* h, const double* contrib, int npieces, int r, int64_t n,
                   double* mean, cudaStream_t st) {
  mdsx::pre(h, st);
  dc_mean2_kernel<<<1, 256, 0, st>>>(contrib, npieces, r, 1.0 / (double)n, mean);
  return launched(h, "dc_mean_kernel", st);
}

// Final re-centring of the D&C output: mean from the per-piece contributions
// (fixed order), one shift pass over the n x r output.
int launch_dc_recentre(mdsx_handle* h, const double* contrib, int npieces, int r, int64_t n,
                       double* mean, double* out, cudaStream_t st) {
  mdsx::pre(h, st);
  dc_mean2_kernel<<<1, 256, 0, st>>>(contrib, npieces, r, 1.0 / (double)n, mean);
  int rc = launched(h, "dc_mean_kernel", st);
  if (rc) return rc;
  return launch_shift_rows(h, out, nullptr, n, r, mean, st);
}

}  // namespace mdsx

// ---------------------------------------------------------------------------
// fast_mds tail (algorithms.py:285-348) without leaf point matrices.  A leaf's
// rows reach the output through the composition of its alignment and every
// ancestor's: out = (x - mu_leaf) U_leaf T_tot + t_tot - mean.  Points are
// only formed for the TRACKED rows (every row some node's alignment samples),
// which are carried up the tree level by level (fit, then apply to the
// tracked rows of that level's subtrees), and for the alignment sets (the
// Procrustes targets).  The mean needs no pass over the rows: the centred
// rows of a leaf sum to zero, so mean = sum_leaves m_leaf t_tot / n.
namespace {

// points of tracked rows (leaf id per row, rows grouped by leaf): a CTA takes
// 16 consecutive tracked rows, stages them centred in shared memory (coalesced
// row reads) together with U of the first and the last row's leaf (the window
// spans one or two leaves unless leaves track fewer than 16 rows; rows of a
// leaf in between read U from L1/L2), and a thread per (row, column) output
// runs the p-long dot product
constexpr int TK_ROWS = 16;

template <typename T>
__global__ void __launch_bounds__(128)
trk_points_kernel(const T* __restrict__ X, int64_t ld, int p, const int64_t* __restrict__ trk_row,
                  const int32_t* __restrict__ trk_leaf, int64_t ntrk, const PieceDesc* __restrict__ pd,
                  int r, const double* __restrict__ mu_all, const double* __restrict__ Uall,
                  double* __restrict__ P) {
  extern __shared__ double tk_sm[];
  double* xs = tk_sm;                                   // TK_ROWS x (p + 1)
  double* us = tk_sm + TK_ROWS * (p + 1);               // 2 x p x r
  const int pp = p + 1;
  const int64_t i0 = (int64_t)blockIdx.x * TK_ROWS;
  const int nr = (int)min((int64_t)TK_ROWS, ntrk - i0);
  const int l0 = trk_leaf[i0], l1 = trk_leaf[i0 + nr - 1];
  const double* U0 = Uall + pd[l0].u_off;
  const double* U1 = Uall + pd[l1].u_off;
  __shared__ int64_t srow[TK_ROWS], smu[TK_ROWS];
  __shared__ int sleaf[TK_ROWS];
  if (threadIdx.x < nr) {                              // per-row metadata, loaded once
    const int lf = trk_leaf[i0 + threadIdx.x];
    sleaf[threadIdx.x] = lf;
    srow[threadIdx.x] = trk_row[i0 + threadIdx.x] * ld;
    smu[threadIdx.x] = (int64_t)pd[lf].id * p;
  }
  // loads batched 8 per thread before their stores (one latency per batch,
  // not per element)
  for (int e0 = threadIdx.x; e0 < p * r; e0 += 8 * blockDim.x) {
    double v0[8], v1[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      v0[u] = e < p * r ? U0[e] : 0.0;
      v1[u] = e < p * r ? U1[e] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < p * r) {
        us[e] = v0[u];
        us[p * r + e] = v1[u];
      }
    }
  }
  __syncthreads();
  for (int e0 = threadIdx.x; e0 < nr * p; e0 += 8 * blockDim.x) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < nr * p) {
        const int t = e / p, a = e - t * p;
        v[u] = (double)X[srow[t] + a] - mu_all[smu[t] + a];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e < nr * p) {
        const int t = e / p, a = e - t * p;
        xs[t * pp + a] = v[u];
      }
    }
  }
  __syncthreads();
  for (int o = threadIdx.x; o < nr * r; o += blockDim.x) {
    const int t = o / r, q = o - t * r;
    const int lf = sleaf[t];
    const double* U = lf == l0 ? us : lf == l1 ? us + p * r : Uall + pd[lf].u_off;
    const double* xr = xs + t * pp;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int a = 0;
    for (; a + 3 < p; a += 4) {
      s0 = fma(xr[a], U[a * r + q], s0);
      s1 = fma(xr[a + 1], U[(a + 1) * r + q], s1);
      s2 = fma(xr[a + 2], U[(a + 2) * r + q], s2);
      s3 = fma(xr[a + 3], U[(a + 3) * r + q], s3);
    }
    for (; a < p; ++a) s0 = fma(xr[a], U[a * r + q], s0);
    P[(i0 + t) * r + q] = (s0 + s1) + (s2 + s3);
  }
}

// tracked rows of this level's subtrees: P <- P T_job + t_job (thread per row)
__global__ void trk_apply_kernel(double* __restrict__ P, const int32_t* __restrict__ job, int64_t ntrk,
                                 int r, const double* __restrict__ rot, const double* __restrict__ trans) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntrk) return;
  const int jb = job[i];
  if (jb < 0) return;
  double x[RMX];
#pragma unroll
  for (int q = 0; q < RMX; ++q) x[q] = q < r ? P[i * r + q] : 0.0;
  const double* T = rot + (int64_t)jb * r * r;
  for (int q = 0; q < r; ++q) {
    double v = trans[(int64_t)jb * r + q];
#pragma unroll
    for (int b = 0; b < RMX; ++b)
      if (b < r) v = fma(x[b], T[b * r + q], v);
    P[i * r + q] = v;
  }
}

// per leaf: T_tot, t_tot over the levels (deepest first), U' = U T_tot,
// contrib = m_leaf t_tot
__global__ void __launch_bounds__(128)
fast_compose_kernel(const PieceDesc* __restrict__ pd, int nlev, int nleaves, int p, int r,
                    const int32_t* __restrict__ leaf_job, const int64_t* __restrict__ lev_jbase,
                    const double* __restrict__ rot, const double* __restrict__ trans,
                    const double* __restrict__ Uall, double* __restrict__ Uc,
                    double* __restrict__ tvec, double* __restrict__ contrib) {
  const int j = blockIdx.x;
  const PieceDesc d = pd[j];
  __shared__ double Tt[RMX * RMX], tt[RMX], Tn[RMX * RMX], tn[RMX];
  const int tid = threadIdx.x;
  for (int e = tid; e < r * r; e += blockDim.x) Tt[e] = (e / r == e % r) ? 1.0 : 0.0;
  if (tid < r) tt[tid] = 0.0;
  __syncthreads();
  for (int L = 0; L < nlev; ++L) {
    const int jb = leaf_job[(int64_t)L * nleaves + j];
    if (jb < 0) continue;                               // uniform over the CTA
    const double* T = rot + (lev_jbase[L] + jb) * r * r;
    const double* t = trans + (lev_jbase[L] + jb) * r;
    for (int e = tid; e < r * r; e += blockDim.x) {
      const int a = e / r, q = e % r;
      double v = 0.0;
      for (int b = 0; b < r; ++b) v = fma(Tt[a * r + b], T[b * r + q], v);
      Tn[e] = v;
    }
    if (tid < r) {
      double v = t[tid];
      for (int b = 0; b < r; ++b) v = fma(tt[b], T[b * r + tid], v);
      tn[tid] = v;
    }
    __syncthreads();
    for (int e = tid; e < r * r; e += blockDim.x) Tt[e] = Tn[e];
    if (tid < r) tt[tid] = tn[tid];
    __syncthreads();
  }
  const double* U = Uall + d.u_off;
  double* O = Uc + (int64_t)j * p * r;
  for (int e = tid; e < p * r; e += blockDim.x) {
    const int a = e / r, q = e - a * r;
    double v = 0.0;
    for (int b = 0; b < r; ++b) v = fma(U[a * r + b], Tt[b * r + q], v);
    O[e] = v;
  }
  if (tid < r) {
    tvec[(int64_t)j * r + tid] = tt[tid];
    contrib[(int64_t)j * r + tid] = (double)d.m * tt[tid];
  }
}

}  // namespace

namespace mdsx {

int launch_trk_points(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                      const int64_t* trk_row, const int32_t* trk_leaf, int64_t ntrk,
                      const PieceDesc* pd, int r, const double* mu, const double* U, double* P,
                      cudaStream_t st) {
  if (ntrk == 0) return MDSX_OK;
  if (p > 128) return fail(h, MDSX_UNSUPPORTED, "tracked points: p > 128");
  const unsigned blocks = (unsigned)((ntrk + TK_ROWS - 1) / TK_ROWS);
  const size_t sm = ((size_t)TK_ROWS * (p + 1) + 2 * (size_t)p * r) * sizeof(double);
  mdsx::pre(h, st);
  if (dtype == MDSX_F32)
    trk_points_kernel<float><<<blocks, 128, sm, st>>>((const float*)data, ld, p, trk_row, trk_leaf, ntrk,
                                                     pd, r, mu, U, P);
  else
    trk_points_kernel<double><<<blocks, 128, sm, st>>>((const double*)data, ld, p, trk_row, trk_leaf, ntrk,
                                                      pd, r, mu, U, P);
  return launched(h, "rows_points_kernel", st);
}

int launch_trk_apply(mdsx_handle* h, double* P, const int32_t* job, int64_t ntrk, int r,
                     const double* rot, const double* trans, cudaStream_t st) {
  if (ntrk == 0) return MDSX_OK;
  mdsx::pre(h, st);
  trk_apply_kernel<<<(unsigned)((ntrk + 127) / 128), 128, 0, st>>>(P, job, ntrk, r, rot, trans);
  return launched(h, "trk_apply_kernel", st);
}

int launch_fast_out(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                    const int64_t* row_idx, const int64_t* out_idx, const PieceDesc* pd, int nleaves,
                    int64_t max_m, int nlev, const int32_t* leaf_job, const int64_t* lev_jbase,
                    int r, const double* mu, const double* U, const double* rot, const double* trans,
                    double* Uc, double* tvec, double* contrib, double* mean, int64_t n_recenter,
                    double* out, cudaStream_t st, const ContribGather* shard) {
  int rc;
  mdsx::pre(h, st);
  fast_compose_kernel<<<nleaves, 128, 0, st>>>(pd, nlev, nleaves, p, r, leaf_job, lev_jbase, rot,
                                               trans, U, Uc, tvec, shard ? shard->local : contrib);
  if ((rc = launched(h, "fast_compose_kernel", st))) return rc;
  if (shard) {          // every rank's leaf contributions, global leaf order
    if (shard->gather(shard->ctx, st) != 0) return fail(h, MDSX_CUDA, "contribution gather failed");
    mdsx::pre(h, st);
    dc_mean2_kernel<<<1, 256, 0, st>>>(shard->global, shard->total, r, 1.0 / (double)shard->n_total,
                                       mean);
    if ((rc = launched(h, "dc_mean_kernel", st))) return rc;
  } else if (n_recenter > 0) {
    mdsx::pre(h, st);
    dc_mean2_kernel<<<1, 256, 0, st>>>(contrib, nleaves, r, 1.0 / (double)n_recenter, mean);
    if ((rc = launched(h, "dc_mean_kernel", st))) return rc;
  } else if ((rc = cuda_check(h, cudaMemsetAsync(mean, 0, r * sizeof(double), st), "memset"))) {
    return rc;
  }
  return launch_piece_out(h, data, dtype, ld, p, row_idx, out_idx, pd, nleaves, max_m, r, 0, mu, Uc,
                          tvec, mean, out, st);
}

}  // namespace mdsx
