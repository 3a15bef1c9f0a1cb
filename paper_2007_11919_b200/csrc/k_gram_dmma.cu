// K1+K2 fused for form-0 pieces (p < m): the p x p Gram of the centred rows
// on the fp64 tensor pipe (DMMA, mma.sync.m8n8k4.f64; tcgen05 has no f64 kind).
//
// Centring without a second pass over the rows: with a shift row x0 (the
// piece's first row) and y = x - x0,
//     C = sum_i (x_i - mu)(x_i - mu)^T = sum_i y_i y_i^T - s s^T / m,  s = sum_i y_i
// which is exact in real arithmetic and, because y is centred to within one
// row's spread, free of the cancellation an unshifted Gram trick suffers.
// The diagonal tiles also publish mu = x0 + s/m (needed by the points
// kernel) and flag non-finite input.  Output: lower triangle computed,
// mirrored to the upper -> exactly symmetric; fixed reduction order.
#include "mdsx_common.cuh"
#include "bulk.cuh"
#include "gram_ring.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace {

constexpr int TT = 64;          // output tile (features x features)
constexpr int KC = 32;          // rows staged per chunk
constexpr int LD = TT + 4;      // smem row pitch (conflict-free fragment loads)
constexpr int NT = 256;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <typename T>
__global__ void __launch_bounds__(NT)
gram_dmma_kernel(const T* __restrict__ X, int64_t ld, int p, const int64_t* __restrict__ row_idx,
                 const PieceDesc* __restrict__ pd, const int4* __restrict__ tiles,
                 double* __restrict__ A, double* __restrict__ mu_all,
                 mdsx_piece_status* __restrict__ status) {
  __shared__ __align__(16) double ya[KC][LD];
  __shared__ __align__(16) double yb[KC][LD];
  __shared__ double x0a[TT], x0b[TT], sa[TT], sb[TT];
  __shared__ int bad;
  const int4 tl = tiles[blockIdx.x];
  const PieceDesc d = pd[tl.x];
  const int ti = tl.y, tj = tl.z, k = d.k, m = d.m;
  const bool diag = ti == tj;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;     // warp sub-tile: rows 16*wr.., cols 32*wc..
  const int64_t* ridx = row_idx + d.row_off;
  const int ca = ti * TT, cb = tj * TT;

  if (tid == 0) bad = 0;
  if (tid < TT) {
    const T* r0 = X + ridx[0] * ld;
    x0a[tid] = ca + tid < k ? mdsx::ld_val(r0 + ca + tid) : 0.0;
    x0b[tid] = cb + tid < k ? mdsx::ld_val(r0 + cb + tid) : 0.0;
    sa[tid] = 0.0;
    sb[tid] = 0.0;
  }
  __syncthreads();

  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // register prefetch of chunk c+1 while the DMMAs run on chunk c:
  // warp w owns rows 4w..4w+3 of a chunk, lane owns columns lane, lane+32
  constexpr int RPW = KC / (NT / 32);          // 4 rows per warp
  double pre[2][RPW][2];
  bool nonfinite = false;
  const int nchunks = (m + KC - 1) / KC;
  auto fetch = [&](int c) {
    const int r0 = c * KC, nr = min(KC, m - r0);
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const int rr = warp * RPW + j;
      const bool live = rr < nr;
      const T* src = X + (live ? ridx[r0 + rr] : ridx[0]) * ld;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = lane + 32 * h;
        pre[0][j][h] = (live && ca + col < k) ? mdsx::ld_val(src + ca + col) : 0.0;
        pre[1][j][h] = (!diag && live && cb + col < k) ? mdsx::ld_val(src + cb + col) : 0.0;
      }
    }
  };
  auto store = [&](int c) {
    const int nr = min(KC, m - c * KC);
#pragma unroll
    for (int j = 0; j < RPW; ++j) {
      const int rr = warp * RPW + j;
      const bool live = rr < nr;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = lane + 32 * h;
        const double va = pre[0][j][h];
        nonfinite |= !isfinite(va);
        ya[rr][col] = (live && ca + col < k) ? va - x0a[col] : 0.0;
        if (!diag) yb[rr][col] = (live && cb + col < k) ? pre[1][j][h] - x0b[col] : 0.0;
      }
    }
  };
  const double (*YB)[LD] = diag ? ya : yb;     // diagonal tiles: one operand block
  fetch(0);
  for (int c = 0; c < nchunks; ++c) {
    const int nr = min(KC, m - c * KC);
    store(c);
    __syncthreads();
    if (c + 1 < nchunks) fetch(c + 1);          // in flight during the DMMAs below
    if (tid < TT) {                              // column sums of the chunk, fixed order
      double s = 0.0;
      for (int rr = 0; rr < nr; ++rr) s += ya[rr][tid];
      sa[tid] += s;
    } else if (tid < 2 * TT) {
      double s = 0.0;
      for (int rr = 0; rr < nr; ++rr) s += YB[rr][tid - TT];
      sb[tid - TT] += s;
    }
#pragma unroll
    for (int k4 = 0; k4 < KC; k4 += 4) {
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = ya[k4 + tig][wr * 16 + i * 8 + gid];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = YB[k4 + tig][wc * 32 + j * 8 + gid];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  if (nonfinite) bad = 1;
  __syncthreads();

  const double inv_m = 1.0 / (double)m;
  double* out = A + d.a_off;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int li = wr * 16 + i * 8 + gid, lj = wc * 32 + j * 8 + 2 * tig + v;
        const int gi = ca + li, gj = cb + lj;
        if (gi < k && gj < k && (!diag || gi >= gj)) {
          const double c = fma(-sa[li] * inv_m, sb[lj], acc[i][j][v]);
          out[(int64_t)gi * k + gj] = c;
          out[(int64_t)gj * k + gi] = c;
        }
      }
  if (diag) {
    if (tid < TT && ca + tid < k) mu_all[(int64_t)d.id * p + ca + tid] = x0a[tid] + sa[tid] * inv_m;
    if (tid == 0 && bad) status[d.id].code = MDSX_INVALID_INPUT;
  }
}


// ---- large k (config 5, p = 784): 64 x 64 output tiles of the Gram, rows
// gathered with cp.async into a 3-deep ring of raw column slices (the row
// indices of a chunk are loaded in parallel and broadcast), converted and
// shifted by x0 at fragment-load time.  Same arithmetic and outputs as
// gram_dmma_kernel, without its dependent index -> value load chains.
constexpr int TS_KC = 32;                 // rows per chunk
constexpr int TS_NS = 3;                  // ring depth

template <typename T>
struct TsPitch {                          // conflict-free fragment pitch (elements)
  static constexpr int value = sizeof(T) == 4 ? 72 : 68;
};

// Column sums of the shifted rows, once per 64-column slice of a piece (the
// diagonal tiles of the tile list; the other CTAs exit): mu = x0 + s / m and the
// non-finite flag.  The tile kernel recovers s = (mu - x0) m for its two
// slices, so no tile repeats the sums (a piece has up to 36 tiles).
template <typename T>
__global__ void __launch_bounds__(NT)
gram_tile_sums_kernel(const T* __restrict__ X, int64_t ld, int p,
                      const int64_t* __restrict__ row_idx, const PieceDesc* __restrict__ pd,
                      const int4* __restrict__ tiles, double* __restrict__ mu_all,
                      mdsx_piece_status* __restrict__ status) {
  const int4 tl = tiles[blockIdx.x];
  if (tl.y != tl.z) return;
  __shared__ double part[4][TT];
  const PieceDesc d = pd[tl.x];
  const int ca = tl.y * TT, k = d.k, m = d.m;
  const int col = threadIdx.x & (TT - 1), grp = threadIdx.x >> 6;      // 4 row groups
  const int64_t* ridx = row_idx + d.row_off;
  const bool live = ca + col < k;
  const double x0 = live ? (double)X[ridx[0] * ld + ca + col] : 0.0;
  double s0 = 0.0, s1 = 0.0;
  if (live) {
    int i = grp;
    for (; i + 4 < m; i += 8) {
      const double v0 = (double)X[ridx[i] * ld + ca + col];
      const double v1 = (double)X[ridx[i + 4] * ld + ca + col];
      s0 += v0 - x0;
      s1 += v1 - x0;
    }
    if (i < m) s0 += (double)X[ridx[i] * ld + ca + col] - x0;
  }
  part[grp][col] = s0 + s1;
  __syncthreads();
  if (threadIdx.x < TT && live) {
    const double sum = (part[0][col] + part[1][col]) + (part[2][col] + part[3][col]);
    mu_all[(int64_t)d.id * p + ca + col] = x0 + sum / (double)m;
    if (!isfinite(sum)) status[d.id].code = MDSX_INVALID_INPUT;
  }
}

// Fragments carry no predicates: columns past k of a slice are zero in every
// stage (written once; their shift is 0), the rows that round the last chunk
// up to a multiple of 4 hold the shift row (x - x0 = 0 exactly), and the k4
// loop stops at the last valid group.
template <typename T>
__global__ void __launch_bounds__(NT)
gram_tile_async_kernel(const T* __restrict__ X, int64_t ld, int p,
                       const int64_t* __restrict__ row_idx, const PieceDesc* __restrict__ pd,
                       const int4* __restrict__ tiles, double* __restrict__ A,
                       const double* __restrict__ mu_all) {
  constexpr int P = TsPitch<T>::value;
  constexpr int SLICE = TS_KC * P;                       // elements per slice per stage
  extern __shared__ __align__(16) unsigned char ts_smem[];
  T* ring = reinterpret_cast<T*>(ts_smem);               // TS_NS x 2 slices
  __shared__ double x0a[TT], x0b[TT], sa[TT], sb[TT];
  const int4 tl = tiles[blockIdx.x];
  const PieceDesc d = pd[tl.x];
  const int ti = tl.y, tj = tl.z, k = d.k, m = d.m;
  const bool diag = ti == tj;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wr = warp >> 1, wc = warp & 1;              // warp sub-tile: rows 16*wr.., cols 32*wc..
  const int64_t* ridx = row_idx + d.row_off;
  const int ca = ti * TT, cb = tj * TT;
  const int na = min(TT, k - ca), nb = min(TT, k - cb);  // valid columns of each slice
  const int pa16 = (int)((size_t)na * sizeof(T) / 16), pb16 = (int)((size_t)nb * sizeof(T) / 16);
  const int nchunks = (m + TS_KC - 1) / TS_KC;

  // columns past k: zero once in every stage (the copies never touch them)
  if (na < TT || nb < TT)
    for (int e = tid; e < TS_NS * 2 * TS_KC * TT; e += NT) {
      const int col = e % TT, row = (e / TT) % TS_KC, sl = (e / (TT * TS_KC)) & 1,
                stg = e / (2 * TT * TS_KC);
      if (col >= (sl ? nb : na)) ring[((size_t)stg * 2 + sl) * SLICE + row * P + col] = T(0);
    }

  auto issue = [&](int c) {
    if (c < nchunks) {
      const int r0 = c * TS_KC, nr = min(TS_KC, m - r0);
      T* dst_a = ring + (size_t)(c % TS_NS) * 2 * SLICE;
      T* dst_b = dst_a + SLICE;
      // warp w copies rows w, w+8, w+16, w+24; their indices loaded in parallel
      const int myr = warp + 8 * lane;
      const int64_t myidx = (lane < TS_KC / 8 && myr < nr) ? ridx[r0 + myr] : 0;
#pragma unroll
      for (int i = 0; i < TS_KC / 8; ++i) {
        const int rr = warp + 8 * i;
        const int64_t gi = __shfl_sync(0xffffffffu, myidx, i);
        if (rr < nr) {
          const char* src = reinterpret_cast<const char*>(X + gi * ld);
          for (int q = lane; q < pa16 + (diag ? 0 : pb16); q += 32) {
            const bool second = q >= pa16;
            const int qq = second ? q - pa16 : q;
            const char* s16 = src + (size_t)(second ? cb : ca) * sizeof(T) + 16 * qq;
            char* d16 = reinterpret_cast<char*>((second ? dst_b : dst_a) + (size_t)rr * P) + 16 * qq;
            const unsigned sa_ = (unsigned)__cvta_generic_to_shared(d16);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa_), "l"(s16));
          }
        }
      }
      // the last chunk: the shift row completes its last group of four rows
      const int nr4 = (nr + 3) & ~3;
      if (nr4 > nr) {
        const T* r0p = X + ridx[0] * ld;
        for (int e = tid; e < (nr4 - nr) * 2 * TT; e += NT) {
          const int col = e % TT, sl = (e / TT) & 1, row = nr + e / (2 * TT);
          if (sl && diag) continue;
          const int nv = sl ? nb : na;
          (sl ? dst_b : dst_a)[(size_t)row * P + col] = col < nv ? r0p[(sl ? cb : ca) + col] : T(0);
        }
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  __syncthreads();                                         // zeroed columns before any copy lands
#pragma unroll
  for (int c = 0; c < TS_NS - 1; ++c) issue(c);
  if (tid < TT) {
    const T* r0p = X + ridx[0] * ld;
    x0a[tid] = tid < na ? (double)r0p[ca + tid] : 0.0;
    x0b[tid] = tid < nb ? (double)r0p[cb + tid] : 0.0;
    // column sums of the shifted rows from the published means (gram_tile_sums_kernel)
    const double* mu = mu_all + (int64_t)d.id * p;
    sa[tid] = tid < na ? (mu[ca + tid] - x0a[tid]) * (double)m : 0.0;
    sb[tid] = tid < nb ? (mu[cb + tid] - x0b[tid]) * (double)m : 0.0;
  }
  __syncthreads();
  double xa4[2], xb4[4];                                   // per-lane shifts of the fragment columns
#pragma unroll
  for (int i = 0; i < 2; ++i) xa4[i] = x0a[wr * 16 + i * 8 + gid];
#pragma unroll
  for (int j = 0; j < 4; ++j) xb4[j] = diag ? x0a[wc * 32 + j * 8 + gid] : x0b[wc * 32 + j * 8 + gid];
  double acc[2][4][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int c = 0; c < nchunks; ++c) {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(TS_NS - 2));
    __syncthreads();                 // chunk c landed for everyone; stage (c - 1) % NS is free
    issue(c + TS_NS - 1);
    const T* sta = ring + (size_t)(c % TS_NS) * 2 * SLICE;
    const T* stb = diag ? sta : sta + SLICE;
    const int nks = (min(TS_KC, m - c * TS_KC) + 3) >> 2;
    const T* pa = sta + tig * P + wr * 16 + gid;
    const T* pb = stb + tig * P + wc * 32 + gid;
#pragma unroll
    for (int ks = 0; ks < TS_KC / 4; ++ks) {
      if (ks >= nks) break;
      double af[2], bf[4];
#pragma unroll
      for (int i = 0; i < 2; ++i) af[i] = (double)pa[4 * ks * P + i * 8] - xa4[i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = (double)pb[4 * ks * P + j * 8] - xb4[j];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
  const double inv_m = 1.0 / (double)m;
  double* out = A + d.a_off;
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int li = wr * 16 + i * 8 + gid, lj = wc * 32 + j * 8 + 2 * tig + v;
        const int gi = ca + li, gj = cb + lj;
        if (gi < k && gj < k && (!diag || gi >= gj)) {
          const double cv = fma(-sa[li] * inv_m, diag ? sa[lj] : sb[lj], acc[i][j][v]);
          out[(int64_t)gi * k + gj] = cv;
          out[(int64_t)gj * k + gi] = cv;
        }
      }
}

// ---- one CTA per piece for k <= 104 (the config 2/3 shape).  The lower
// triangle of the k x k Gram in 8x8 blocks (NB*(NB+1)/2 block pairs) is split
// over 4 compute warps; each warp runs all rows, so no cross-warp reduction.
//
// Rows reach shared memory through a warp-specialised ring: a producer warp
// gathers GP_KC rows per stage, one cp.async.bulk (TMA engine) per row issued
// by its own lane (row index loaded a stage ahead), completing on the stage's
// `full` mbarrier; the compute warps release a stage on its `empty` mbarrier,
// so no CTA-wide barrier sits in the main loop.  Padding columns [p, P) of the
// stage are zero (written once), the producer fills the rows that round the
// last stage up to a multiple of 4 with the shift row, and only the last
// 8-feature block masks features >= p, so (x - x0) is exactly 0 on every
// padded position.  The pitch P is congruent so that the 32 lanes of an
// m8n8k4 fragment load hit distinct banks.
// One fragment per 8-feature block and k4-step serves both the A (rows) and B
// (columns) operand of every block pair that touches it.  Shift x0 = first
// row; the producer also accumulates the column sums s = sum (x - x0) of each
// stage after the compute warps were handed it (C = sum y y^T - s s^T / m);
// mu = x0 + s/m is published with the Gram.
using gring::GP_THREADS;
using gring::GP_CTA;
using gring::GP_KC;
using gring::GP_HDR;
using gring::gram_piece_body;

template <typename T, int NB, int NS>
__global__ void __launch_bounds__(GP_CTA, 2)
gram_piece_kernel(const T* __restrict__ X, int64_t ld, int p, int P,
                  const int64_t* __restrict__ row_idx, const PieceDesc* __restrict__ pd,
                  double* __restrict__ A, double* __restrict__ mu_all,
                  mdsx_piece_status* __restrict__ status) {
  extern __shared__ __align__(128) unsigned char gp_smem[];
  gram_piece_body<T, NB, NS, GP_THREADS / 32>(X, ld, p, P, row_idx, pd, blockIdx.x, A, mu_all, status,
                                              gp_smem);
}

// Combine the centred Grams of a piece's row ranges (parallel-variance
// formula): mu = sum_q m_q mu_q / m,  C = sum_q C_q + m_q (mu_q - mu)(mu_q - mu)^T;
// splits in fixed order (deterministic).  Grid (entry blocks of 256, pieces);
// every CTA stages the split sizes and means and forms mu itself.
constexpr int GC_SMAX = 32;

__global__ void __launch_bounds__(256)
gram_combine_kernel(const PieceDesc* __restrict__ pd, const int4* __restrict__ rng,
                    const PieceDesc* __restrict__ pds, const double* __restrict__ As,
                    const double* __restrict__ mus, const mdsx_piece_status* __restrict__ sts, int p,
                    double* __restrict__ A, double* __restrict__ mu_all,
                    mdsx_piece_status* __restrict__ status) {
  __shared__ double mu[104], dm[GC_SMAX][104], mq_s[GC_SMAX];
  __shared__ int64_t aoff[GC_SMAX];
  const int4 g = rng[blockIdx.y];
  const int q0 = g.x, S = g.y;
  const PieceDesc d = pd[blockIdx.y];
  const int k = d.k;
  if (threadIdx.x < S) {
    const PieceDesc v = pds[q0 + threadIdx.x];
    mq_s[threadIdx.x] = (double)v.m;
    aoff[threadIdx.x] = v.a_off;
  }
  for (int e = threadIdx.x; e < S * k; e += blockDim.x) {
    const int q = e / k, a = e - q * k;
    dm[q][a] = mus[(int64_t)(q0 + q) * p + a];
  }
  __syncthreads();
  for (int a = threadIdx.x; a < k; a += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < S; ++q) s = fma(mq_s[q], dm[q][a], s);
    mu[a] = s / (double)d.m;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < S * k; e += blockDim.x) {
    const int q = e / k, a = e - q * k;
    dm[q][a] -= mu[a];
  }
  __syncthreads();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < k * k) {
    const int a = e / k, b = e - a * k;
    if (b <= a) {
      double c = 0.0;
#pragma unroll 4
      for (int q = 0; q < S; ++q) c += As[aoff[q] + e] + mq_s[q] * (dm[q][a] * dm[q][b]);
      double* out = A + d.a_off;
      out[(int64_t)a * k + b] = c;
      out[(int64_t)b * k + a] = c;
    }
  }
  if (blockIdx.x == 0) {
    for (int a = threadIdx.x; a < k; a += blockDim.x) mu_all[(int64_t)d.id * p + a] = mu[a];
    if (threadIdx.x == 0) {
      bool bad = false;
      for (int q = 0; q < S; ++q) bad = bad || sts[q0 + q].code == MDSX_INVALID_INPUT;
      if (bad) status[d.id].code = MDSX_INVALID_INPUT;
    }
  }
}

}  // namespace

namespace mdsx {

int launch_gram_combine(mdsx_handle* h, const PieceDesc* pd, const int4* rng, int npieces,
                        const PieceDesc* pd_split, const double* A_split, const double* mu_split,
                        const mdsx_piece_status* st_split, int p, double* A, double* mu,
                        mdsx_piece_status* status, cudaStream_t st) {
  if (npieces == 0) return MDSX_OK;
  mdsx::pre(h, st);
  gram_combine_kernel<<<dim3((104 * 104 + 255) / 256, npieces), 256, 0, st>>>(
      pd, rng, pd_split, A_split, mu_split, st_split, p, A, mu, status);
  return launched(h, "gram_combine_kernel", st);
}


// Pitch (elements) of a staged row: >= p, 16-byte multiple, and congruent so that the 32 lanes of an m8n8k4 fragment load hit
// distinct banks.
static int gp_pitch(int p, size_t es) {
  int P = p;
  if (es == 8) { while (P % 16 != 4) ++P; }
  else { while (P % 32 != 8) ++P; }
  return P;
}

bool gram_piece_ok(const void* data, int dtype, int64_t ld, int p) {
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  return p <= 104 && ((size_t)p * es) % 16 == 0 && ((size_t)ld * es) % 16 == 0 &&
         (reinterpret_cast<uintptr_t>(data) & 15) == 0;
}

int launch_gram_piece(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                      const int64_t* row_idx, const PieceDesc* pd, int npieces, double* A,
                      double* mu, mdsx_piece_status* status, cudaStream_t st) {
  if (npieces == 0) return MDSX_OK;
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  auto go = [&](auto tag, auto nb) {
    using T = decltype(tag);
    constexpr int NB = decltype(nb)::value;
    constexpr int NS = 4;
    const int P = gp_pitch(std::max(p, 8 * (NB - 1)), es);   // only the last block can pass P
    const size_t smem = GP_HDR + (size_t)NS * GP_KC * P * es + 64;   // + overrun of the last fragment
    auto kern = gram_piece_kernel<T, NB, NS>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mdsx::pre(h, st);
    kern<<<npieces, GP_CTA, smem, st>>>((const T*)data, ld, p, P, row_idx, pd, A, mu, status);
    return launched(h, "gram_piece_kernel", st);
  };
  using N4 = std::integral_constant<int, 4>;
  using N8 = std::integral_constant<int, 8>;
  using N13 = std::integral_constant<int, 13>;
  if (dtype == MDSX_F64)
    return p <= 32 ? go(double{}, N4{}) : p <= 64 ? go(double{}, N8{}) : go(double{}, N13{});
  return p <= 32 ? go(float{}, N4{}) : p <= 64 ? go(float{}, N8{}) : go(float{}, N13{});
}

int launch_gram_dmma(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                     const int64_t* row_idx, const PieceDesc* pd, const int4* tiles, int ntiles,
                     double* A, double* mu, mdsx_piece_status* status, cudaStream_t st) {
  if (ntiles == 0) return MDSX_OK;
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  if (((size_t)p * es) % 16 == 0 && ((size_t)ld * es) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(data) & 15) == 0 && !getenv("MDSX_GRAM_TILED_SYNC")) {
    auto go = [&](auto tag) {
      using T = decltype(tag);
      const size_t smem = (size_t)TS_NS * 2 * TS_KC * TsPitch<T>::value * sizeof(T);
      cudaFuncSetAttribute(gram_tile_async_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      mdsx::pre(h, st);
      gram_tile_sums_kernel<T><<<ntiles, NT, 0, st>>>((const T*)data, ld, p, row_idx, pd, tiles, mu,
                                                      status);
      const int rc = launched(h, "gram_tile_sums_kernel", st);
      if (rc) return rc;
      mdsx::pre(h, st);
      gram_tile_async_kernel<T><<<ntiles, NT, smem, st>>>((const T*)data, ld, p, row_idx, pd, tiles,
                                                          A, mu);
      return launched(h, "gram_tile_async_kernel", st);
    };
    return dtype == MDSX_F64 ? go(double{}) : go(float{});
  }
  mdsx::pre(h, st);
  if (dtype == MDSX_F64)
    gram_dmma_kernel<double><<<ntiles, NT, 0, st>>>((const double*)data, ld, p, row_idx, pd, tiles,
                                                   A, mu, status);
  else
    gram_dmma_kernel<float><<<ntiles, NT, 0, st>>>((const float*)data, ld, p, row_idx, pd, tiles, A,
                                                  mu, status);
  return launched(h, "gram_dmma_kernel", st);
}

}  // namespace mdsx
