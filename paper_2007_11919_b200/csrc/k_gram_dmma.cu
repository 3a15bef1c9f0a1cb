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

}  // namespace

namespace mdsx {

int launch_gram_dmma(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                     const int64_t* row_idx, const PieceDesc* pd, const int4* tiles, int ntiles,
                     double* A, double* mu, mdsx_piece_status* status, cudaStream_t st) {
  if (ntiles == 0) return MDSX_OK;
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
