// K4 Gower interpolation (algorithms.py:193-242).
//
// Reference: x = S^-1 [ (q - A2) X1 / (2l) ]  with A2_j = |y - x_j|^2 (clamped),
// q_j = diag(Q)_j = |x_j - xbar|^2, S = X1c^T X1c / l.
// Expanding A2 around the landmark centroid xbar (yc = y - xbar):
//   q_j - A2_j = 2 yc.(x_j - xbar) - |yc|^2
// so the l-long landmark sum folds, once per context, into
//   x = yc^T M - |yc|^2 v,   M = (Xl_c^T X1) S^-1 / l,  v = S^-1 (1^T X1) / (2l).
// The n x l distance tile is never formed (nor written to HBM); each
// interpolated row costs p*r + p FMAs and one streaming read of its p
// inputs — the kernel is HBM-bound.  Equality with the reference formula is
// exact in real arithmetic; the clamp at 0 of A2 only acts on round-off
// negatives of |y - x_j|^2 ~ 0, below the 1e-6 tolerance by ~10 orders.
// The literal tile form (distance tile -> subtract from q -> project) is
// kept as gower_tile_kernel for the function-level seam and verification.
#include "mdsx_common.cuh"
#include "bulk.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace {

// ---- context: per-feature mean and W = Xl_c^T X1 (block per feature)
template <typename T, int RM>
__global__ void __launch_bounds__(256)
ctx_feature_kernel(const T* __restrict__ X, int64_t ld, const int64_t* __restrict__ idx, int64_t l,
                   int p, const double* __restrict__ X1, int r, double* __restrict__ mean,
                   double* __restrict__ W) {
  __shared__ double red[256];
  __shared__ double mu_s;
  const int a = blockIdx.x;
  const int tid = threadIdx.x;
  double s = 0.0;
  for (int64_t j = tid; j < l; j += 256) {
    const int64_t row = idx ? idx[j] : j;
    s += mdsx::ld_val(X + row * ld + a);
  }
  red[tid] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  if (tid == 0) { mu_s = red[0] / (double)l; mean[a] = mu_s; }
  __syncthreads();
  const double mu = mu_s;
  double acc[RM];
#pragma unroll
  for (int c = 0; c < RM; ++c) acc[c] = 0.0;
  for (int64_t j = tid; j < l; j += 256) {
    const int64_t row = idx ? idx[j] : j;
    const double y = mdsx::ld_val(X + row * ld + a) - mu;
#pragma unroll
    for (int c = 0; c < RM; ++c)
      if (c < r) acc[c] = fma(y, X1[j * r + c], acc[c]);
  }
  for (int c = 0; c < r; ++c) {
    __syncthreads();
    red[tid] = acc[c];
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (tid < o) red[tid] += red[tid + o];
      __syncthreads();
    }
    if (tid == 0) W[(int64_t)a * r + c] = red[0];
  }
}

// ---- q_j = |x_j - xbar|^2 (GowerContext.q_diag)
template <typename T>
__global__ void ctx_qdiag_kernel(const T* __restrict__ X, int64_t ld, const int64_t* __restrict__ idx,
                                 int64_t l, int p, const double* __restrict__ mean,
                                 double* __restrict__ q) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= l) return;
  const int64_t row = idx ? idx[j] : j;
  double s = 0.0;
  for (int a = 0; a < p; ++a) {
    const double y = mdsx::ld_val(X + row * ld + a) - mean[a];
    s = fma(y, y, s);
  }
  q[j] = s;
}

// S = X1c^T X1c / l for r <= RM: every thread walks rows tid, tid + nt, ...
// with the centred row and the whole upper triangle in registers; warp
// shuffles, then the per-warp partials in `scr` (>= RM(RM+1)/2 x nw) summed
// in fixed order.
template <int RM>
__device__ void ctx_S_upper(const double* __restrict__ X1, int64_t l, int r, const double* m1,
                            double* scr, double* Ssh, double* S, int tid, int lane, int warp, int nw) {
  constexpr int NE = RM * (RM + 1) / 2;
  double ac[NE];
#pragma unroll
  for (int u = 0; u < NE; ++u) ac[u] = 0.0;
  for (int64_t j = tid; j < l; j += blockDim.x) {
    double xr[RM];
#pragma unroll
    for (int c = 0; c < RM; ++c) xr[c] = c < r ? X1[j * r + c] - m1[c] : 0.0;
#pragma unroll
    for (int a = 0, u = 0; a < RM; ++a)
#pragma unroll
      for (int b = a; b < RM; ++b, ++u) ac[u] = fma(xr[a], xr[b], ac[u]);
  }
#pragma unroll
  for (int u = 0; u < NE; ++u) {
    const double t = mdsx::warp_sum(ac[u]);
    if (lane == 0) scr[u * nw + warp] = t;
  }
  __syncthreads();
  for (int u = tid; u < NE; u += blockDim.x) {
    int a = 0, rem = u;
    while (rem >= RM - a) { rem -= RM - a; ++a; }
    const int b = a + rem;
    if (a < r && b < r) {
      double t = 0.0;
      for (int w2 = 0; w2 < nw; ++w2) t += scr[u * nw + w2];
      t /= (double)l;
      Ssh[a * r + b] = Ssh[b * r + a] = t;
      S[a * r + b] = S[b * r + a] = t;
    }
  }
  __syncthreads();
}

// ---- S, s, eigen-condition, Cholesky, M, v (one block)
__global__ void __launch_bounds__(256)
ctx_finalize_kernel(const double* __restrict__ X1, int64_t l, int p, int r,
                    double* __restrict__ W_to_M, double* __restrict__ v, double* __restrict__ S,
                    double* __restrict__ cond, int32_t* __restrict__ flag) {
  __shared__ double m1[MDSX_MAX_R], s1[MDSX_MAX_R];
  __shared__ double Ssh[MDSX_MAX_R * MDSX_MAX_R], E[MDSX_MAX_R * MDSX_MAX_R];
  __shared__ double L[MDSX_MAX_R * MDSX_MAX_R];
  __shared__ double scr[136 * 8];                 // S partials (16 * 17 / 2 entries x 8 warps)
  __shared__ int ok;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  // column sums / means of X1, then S = X1c^T X1c / l: every thread walks
  // rows tid, tid + 256, ... with the row in registers (coalesced-by-row
  // loads, no strided column walks), then fixed-order warp + block trees
  {
    double cs[MDSX_MAX_R];
    for (int c = 0; c < r; ++c) cs[c] = 0.0;
    for (int64_t j = tid; j < l; j += blockDim.x)
      for (int c = 0; c < r; ++c) cs[c] += X1[j * r + c];
    for (int c = 0; c < r; ++c) {
      const double t = mdsx::warp_sum(cs[c]);
      if (lane == 0) E[c * nw + warp] = t;            // E as scratch (r x nw <= 32 x 32)
    }
    __syncthreads();
    if (tid < r) {
      double t = 0.0;
      for (int w2 = 0; w2 < nw; ++w2) t += E[tid * nw + w2];
      s1[tid] = t;
      m1[tid] = t / (double)l;
    }
    __syncthreads();
  }
  if (r <= 10) ctx_S_upper<10>(X1, l, r, m1, scr, Ssh, S, tid, lane, warp, nw);

  else {
    // upper-triangle entries in chunks of 32, same walk (r > 16)
    const int ne = r * (r + 1) / 2;
    for (int e0 = 0; e0 < ne; e0 += 32) {
      double ac[32];
      int ea[32], eb[32];
      int cnt = 0;
      for (int a = 0, e = 0; a < r; ++a)
        for (int b = a; b < r; ++b, ++e)
          if (e >= e0 && e < e0 + 32) { ea[cnt] = a; eb[cnt] = b; ++cnt; }
      for (int u = 0; u < 32; ++u) ac[u] = 0.0;
      for (int64_t j = tid; j < l; j += blockDim.x) {
        double xr[MDSX_MAX_R];
        for (int c = 0; c < r; ++c) xr[c] = X1[j * r + c] - m1[c];
        for (int u = 0; u < cnt; ++u) ac[u] = fma(xr[ea[u]], xr[eb[u]], ac[u]);
      }
      for (int u = 0; u < cnt; ++u) {
        const double t = mdsx::warp_sum(ac[u]);
        if (lane == 0) L[u * nw + warp] = t;          // L as scratch (32 x nw)
      }
      __syncthreads();
      if (tid < cnt) {
        double t = 0.0;
        for (int w2 = 0; w2 < nw; ++w2) t += L[tid * nw + w2];
        t /= (double)l;
        const int a = ea[tid], b = eb[tid];
        Ssh[a * r + b] = Ssh[b * r + a] = t;
        S[a * r + b] = S[b * r + a] = t;
      }
      __syncthreads();
    }
  }
  for (int e = tid; e < r * r; e += blockDim.x) E[e] = Ssh[e];
  __syncthreads();
  if (warp == 0) {
    // condition test (algorithms.py:209-216).  S is the covariance of the base
    // configuration, whose columns are orthogonal (classical MDS), so S is
    // diagonal up to rounding and the Gershgorin discs [d_a - R_a, d_a + R_a]
    // already certify cond(S) <= max(d + R) / min(d - R) far below the limit:
    // then that bound is the reported estimate and no eigenvalue is computed.
    // Otherwise (and always for a base configuration that is not diagonal
    // enough): the eigenvalues by Jacobi as below, the reference's exact test.
    double glo = 1e308, ghi = 0.0;
    if (lane < r) {
      double rad = 0.0;
      for (int c = 0; c < r; ++c)
        if (c != lane) rad += fabs(Ssh[lane * r + c]);
      glo = Ssh[lane * r + lane] - rad;
      ghi = Ssh[lane * r + lane] + rad;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      glo = fmin(glo, __shfl_xor_sync(0xffffffffu, glo, o));
      ghi = fmax(ghi, __shfl_xor_sync(0xffffffffu, ghi, o));
    }
    const bool certified = glo > 0.0 && ghi <= 1e10 * glo;
    if (certified && lane == 0) {
      cond[0] = ghi / glo;
      ok = 1;
    }
    // eigenvalues of the symmetric PSD S as the singular values of S: one-sided
    // Jacobi on its columns, lane a owns row a, the three column dots of a pair
    // reduced by one interleaved shuffle tree
    for (int sweep = 0; sweep < 60 && !certified; ++sweep) {
      int nrot = 0;
      for (int i = 0; i < r - 1; ++i)
        for (int j = i + 1; j < r; ++j) {
          const double x = lane < r ? E[lane * r + i] : 0.0;
          const double y = lane < r ? E[lane * r + j] : 0.0;
          double al = x * x, be = y * y, ga = x * y;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
            al += __shfl_xor_sync(0xffffffffu, al, o);
            be += __shfl_xor_sync(0xffffffffu, be, o);
            ga += __shfl_xor_sync(0xffffffffu, ga, o);
          }
          if (ga != 0.0 && ga * ga > 1e-30 * (al * be)) {
            const double h = 0.5 * (be - al);
            const double t = ga / (h + copysign(sqrt(fma(h, h, ga * ga)), h == 0.0 ? 1.0 : h));
            const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
            if (lane < r) {
              E[lane * r + i] = c * x - sn * y;
              E[lane * r + j] = sn * x + c * y;
            }
            ++nrot;
          }
          __syncwarp();
        }
      if (nrot == 0) break;
    }
    if (!certified) {
      double lo = 1e308, hi = 0.0;
      for (int i = 0; i < r; ++i) {
        const double x = lane < r ? E[lane * r + i] : 0.0;
        const double sv = sqrt(mdsx::warp_sum(x * x));
        lo = fmin(lo, sv);
        hi = fmax(hi, sv);
      }
      if (lane == 0) {
        const double cd = lo <= 0.0 ? INFINITY : hi / lo;
        cond[0] = cd;
        ok = cd <= 1e12 ? 1 : 0;
      }
    }
  }
  __syncthreads();
  if (tid == 0) {
    int good = ok;
    const double cd = cond[0];
    // Cholesky S = L L^T (scipy cho_factor lower)
    for (int j = 0; j < r && good; ++j) {
      double d = Ssh[j * r + j];
      for (int k = 0; k < j; ++k) d -= L[j * r + k] * L[j * r + k];
      if (!(d > 0.0)) { good = 0; break; }
      const double ljj = sqrt(d);
      L[j * r + j] = ljj;
      for (int i = j + 1; i < r; ++i) {
        double s = Ssh[i * r + j];
        for (int k = 0; k < j; ++k) s -= L[i * r + k] * L[j * r + k];
        L[i * r + j] = s / ljj;
      }
      for (int i = 0; i < j; ++i) L[i * r + j] = 0.0;
    }
    ok = good;
    flag[0] = good ? 0 : (cd > 1e12 ? 1 : 2);
  }
  __syncthreads();
  if (!ok) return;
  // rows of W (and s) -> solve S x = w (S symmetric): M = W S^-1 / l, v = S^-1 s / (2l)
  for (int a = tid; a <= p; a += blockDim.x) {
    double x[MDSX_MAX_R];
    for (int i = 0; i < r; ++i) x[i] = (a < p) ? W_to_M[(int64_t)a * r + i] : s1[i];
    for (int i = 0; i < r; ++i) {            // L y = w
      double s = x[i];
      for (int k = 0; k < i; ++k) s -= L[i * r + k] * x[k];
      x[i] = s / L[i * r + i];
    }
    for (int i = r - 1; i >= 0; --i) {       // L^T z = y
      double s = x[i];
      for (int k = i + 1; k < r; ++k) s -= L[k * r + i] * x[k];
      x[i] = s / L[i * r + i];
    }
    if (a < p)
      for (int i = 0; i < r; ++i) W_to_M[(int64_t)a * r + i] = x[i] / (double)l;
    else
      for (int i = 0; i < r; ++i) v[i] = x[i] / (2.0 * (double)l);
  }
}

// ---- streaming affine interpolation: out_i = (y_i - xbar)^T M - |y_i - xbar|^2 v
template <typename T, int RM>
__global__ void __launch_bounds__(256)
gower_affine_kernel(const T* __restrict__ X, int64_t ld, int64_t m, int p, int r,
                    const double* __restrict__ ctx_mean, const double* __restrict__ ctx_M,
                    const double* __restrict__ ctx_v, double* __restrict__ out, int64_t ldo,
                    int32_t* __restrict__ nonfinite) {
  extern __shared__ double sm[];
  double* sM = sm;                     // p x RM (zero padded)
  double* smu = sm + (int64_t)p * RM;  // p
  for (int e = threadIdx.x; e < p * RM; e += blockDim.x) {
    const int a = e / RM, c = e % RM;
    sM[e] = c < r ? ctx_M[(int64_t)a * r + c] : 0.0;
  }
  for (int e = threadIdx.x; e < p; e += blockDim.x) smu[e] = ctx_mean[e];
  double vv[RM];
#pragma unroll
  for (int c = 0; c < RM; ++c) vv[c] = c < r ? ctx_v[c] : 0.0;
  __syncthreads();
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const T* row = X + i * ld;
    double acc[RM];
#pragma unroll
    for (int c = 0; c < RM; ++c) acc[c] = 0.0;
    double nrm = 0.0;
    for (int a = 0; a < p; ++a) {
      const double raw = mdsx::ld_val(row + a);
      bad |= !isfinite(raw);
      const double y = raw - smu[a];
      nrm = fma(y, y, nrm);
      const double* Ma = sM + a * RM;
#pragma unroll
      for (int c = 0; c < RM; ++c) acc[c] = fma(y, Ma[c], acc[c]);
    }
    double* o = out + i * ldo;
#pragma unroll
    for (int c = 0; c < RM; ++c)
      if (c < r) o[c] = acc[c] - nrm * vv[c];
  }
  if (bad) atomicOr(nonfinite, 1);
}


// ---- streaming Gower over contiguous rows, cp.async double buffering.
// Stage = TR rows x p inputs, copied global -> shared in 16-byte cp.async
// chunks (the rows of a tile are one contiguous block), so the copy of tile
// t+1 proceeds while the CTA computes tile t.  Thread i owns row i of the
// stage: x read as float4/double2 vectors along the features (conflict-free),
// centred with the broadcast mean; a thread pair shares a row, each thread
// owning half of the r outputs (+ |x|^2) in registers; M rows are
// warp-broadcast loads.  128-row stages -> two CTAs per SM.
template <typename T, int RM>
__global__ void __launch_bounds__(256, 2)
gower_stream_kernel(const T* __restrict__ X, int64_t m, int p, int r,
                    const double* __restrict__ ctx_mean, const double* __restrict__ ctx_M,
                    const double* __restrict__ ctx_v, double* __restrict__ out,
                    int32_t* __restrict__ nonfinite, int TR) {
  extern __shared__ __align__(16) unsigned char smraw[];
  double* sM = reinterpret_cast<double*>(smraw);          // p x RM
  double* smu = sM + (size_t)p * RM;                      // p
  T* stage0 = reinterpret_cast<T*>(smu + p);              // 2 x TR x p
  const int tid = threadIdx.x;
  for (int e = tid; e < p * RM; e += blockDim.x) {
    const int a = e / RM, c = e % RM;
    sM[e] = c < r ? ctx_M[(int64_t)a * r + c] : 0.0;
  }
  for (int e = tid; e < p; e += blockDim.x) smu[e] = ctx_mean[e];
  double vv[RM];
#pragma unroll
  for (int c = 0; c < RM; ++c) vv[c] = c < r ? ctx_v[c] : 0.0;

  const int64_t ntiles = (m + TR - 1) / TR;
  const size_t stage_elems = (size_t)TR * p;
  auto issue = [&](int64_t t, int b) {        // async copy of tile t into stage b
    const int64_t r0 = t * TR;
    const int64_t nr = min((int64_t)TR, m - r0);
    const char* src = reinterpret_cast<const char*>(X + r0 * p);
    char* dst = reinterpret_cast<char*>(stage0 + (size_t)b * stage_elems);
    const int64_t bytes = nr * p * (int64_t)sizeof(T);
    for (int64_t o = (int64_t)tid * 16; o < bytes; o += (int64_t)blockDim.x * 16) {
      const unsigned saddr = (unsigned)__cvta_generic_to_shared(dst + o);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" :: "r"(saddr), "l"(src + o));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  bool bad = false;
  int64_t t = blockIdx.x;
  if (t < ntiles) issue(t, 0);
  __syncthreads();
  for (int b = 0; t < ntiles; t += gridDim.x, b ^= 1) {
    const int64_t tn = t + gridDim.x;
    if (tn < ntiles) {
      issue(tn, b ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::);
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::);
    }
    __syncthreads();
    const int64_t r0 = t * TR;
    const int nr = (int)min((int64_t)TR, m - r0);
    constexpr int RH = RM / 2;                    // outputs per thread
    const int half = tid & 1;
    for (int i = tid >> 1; i < nr; i += blockDim.x >> 1) {
      const T* xr = stage0 + (size_t)b * stage_elems + (size_t)i * p;
      double acc[RH];
#pragma unroll
      for (int c = 0; c < RH; ++c) acc[c] = 0.0;
      double nrm = 0.0;
      const double* mh = sM + half * RH;
      constexpr int VW = 16 / sizeof(T);           // features per vector load
      int a = 0;
      for (; a + VW <= p; a += VW) {
        double xv[VW];
        if constexpr (sizeof(T) == 4) {
          const float4 f = *reinterpret_cast<const float4*>(xr + a);
          xv[0] = f.x; xv[1] = f.y; xv[2] = f.z; xv[3] = f.w;
        } else {
          const double2 f = *reinterpret_cast<const double2*>(xr + a);
          xv[0] = f.x; xv[1] = f.y;
        }
#pragma unroll
        for (int u = 0; u < VW; ++u) {
          bad |= !isfinite(xv[u]);
          const double y = xv[u] - smu[a + u];
          nrm = fma(y, y, nrm);
          const double2* mr = reinterpret_cast<const double2*>(mh + (size_t)(a + u) * RM);
#pragma unroll
          for (int c = 0; c < RH / 2; ++c) {
            const double2 mm = mr[c];
            acc[2 * c] = fma(y, mm.x, acc[2 * c]);
            acc[2 * c + 1] = fma(y, mm.y, acc[2 * c + 1]);
          }
        }
      }
      for (; a < p; ++a) {
        const double raw = (double)xr[a];
        bad |= !isfinite(raw);
        const double y = raw - smu[a];
        nrm = fma(y, y, nrm);
#pragma unroll
        for (int c = 0; c < RH; ++c) acc[c] = fma(y, mh[(size_t)a * RM + c], acc[c]);
      }
      double* o = out + (r0 + i) * r + half * RH;
#pragma unroll
      for (int c = 0; c < RH; ++c)
        if (half * RH + c < r) o[c] = fma(-nrm, vv[half * RH + c], acc[c]);
    }
    __syncthreads();                              // stage b is refilled next-but-one
  }
  if (bad) atomicOr(nonfinite, 1);
}

// ---- bulk-copy streaming Gower (dense rows, 16-byte aligned rows).
//
// Warp-specialised pipeline.  A tile of TR contiguous rows is one contiguous
// byte range: a producer warp moves it global -> shared with one
// cp.async.bulk (the TMA engine) completing on the stage's `full` mbarrier;
// NSTAGE tiles are in flight.  Eight compute warps consume the ring; each warp
// releases a stage on its `empty` mbarrier, so no CTA-wide barrier sits in the
// steady state.  Compute: a group of TPR lanes owns R = 2 rows of the tile; lane
// j of the group takes the 16-byte feature chunks j, j+TPR, ... of both rows, so
// every per-feature record (M row, mean, mask) read from shared memory feeds 2
// rows.  The records are stored chunk-interleaved so the TPR lanes of a group
// read consecutive 16-byte words (conflict-free) and the groups of a warp
// broadcast.  Epilogue: a butterfly reduce-scatter leaves lane j of a group the
// full sums of output columns [j*KF, (j+1)*KF); it writes them and adds them to
// its per-column running sums (fixed order -> per-CTA column partials for the
// final re-centring of the single call).
//
// TILES (the sharded interpolation, mdsx_gower_tiles): per-TILE column sums
// instead, so that the re-centring's fold does not depend on which CTA -- or
// which rank (rank row ranges start on tile boundaries) -- processed a tile.
// Each warp folds its rows of a tile by a fixed butterfly into a shared-memory
// slot; the producer warp, idle between its copies, adds the eight warp slots
// in warp order and writes one r-vector per tile (it folds tile k - PSLOTS
// before issuing tile k's copy, so a slot is never rewritten unread).

constexpr int GB_THREADS = 256;                  // compute threads (8 warps)
constexpr int GB_CTA = GB_THREADS + 32;          // + one producer warp
constexpr int GB_MAX_STAGES = 4;
constexpr int GB_PSLOTS = 8;                     // TILES: tile-sum slots in flight
// header: full[4], empty[4] mbarriers [0, 64), c0 [64, 192), v [192, 320),
// TILES: psum[8] [320, 384)
constexpr int GB_HEADER = 512;

// N32 (fp32 rows, fused interpolation only): the squared norm |x - xbar|^2 is
// accumulated on the fp32 pipe.  It enters the result only through
// -|x - xbar|^2 v with v = S^-1 (1^T X1) / (2l), and X1 (the landmarks'
// classical configuration) has zero column sums up to rounding, so its 1e-7
// relative error reaches the output at ~1e-22; the fp64 pipe keeps the linear
// term (11 instead of 13 fp64 operations per row-feature).
template <typename T, int RM, int TPR, int CPS, bool N32, bool TILES>
__global__ void __launch_bounds__(GB_CTA, CPS)
gower_bulk_kernel(const T* __restrict__ X, int64_t m, int p, int r,
                  const double* __restrict__ ctx_mean, const double* __restrict__ ctx_M,
                  const double* __restrict__ ctx_v, double* __restrict__ out,
                  double* __restrict__ colpart, int32_t* __restrict__ nonfinite, int nstage) {
  constexpr int VW = 16 / sizeof(T);        // features per 16-byte chunk
  constexpr int W = RM / 2 + 1;             // double2 per feature record: M pairs, (mean, mask)
  constexpr int G = GB_THREADS / TPR;       // row groups
  constexpr int R = 2;                      // rows per group
  constexpr int TR = R * G;                 // rows per tile
  constexpr int RMP = (RM + TPR - 1) / TPR * TPR;   // columns padded to the group width
  constexpr int KF = RMP / TPR;             // columns owned per lane after the reduce-scatter
  extern __shared__ __align__(128) unsigned char smraw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smraw);
  uint64_t* empty = full + GB_MAX_STAGES;
  double* c0s = reinterpret_cast<double*>(smraw + 64);    // xbar^T M
  double* vvs = c0s + 16;                                   // v
  const int nchunks = p / VW;
  const int nit = (nchunks + TPR - 1) / TPR;
  uint64_t* psum = reinterpret_cast<uint64_t*>(smraw + 320);
  double2* rec = reinterpret_cast<double2*>(smraw + GB_HEADER);
  double* pslot = reinterpret_cast<double*>(smraw + GB_HEADER + (size_t)nit * VW * W * TPR * sizeof(double2));
  T* stage0 = reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(pslot) +
                                   (TILES ? (size_t)GB_PSLOTS * (GB_THREADS / 32) * RMP * sizeof(double) : 0));
  const int tid = threadIdx.x;
  const int64_t ntiles = (m + TR - 1) / TR;
  const size_t stage_elems = (size_t)TR * p;

  if (tid == 0) {
    for (int s = 0; s < nstage; ++s) {
      bulk::bar_init(&full[s], 1);
      bulk::bar_init(&empty[s], GB_THREADS / 32);
    }
    if (TILES)
      for (int s = 0; s < GB_PSLOTS; ++s) bulk::bar_init(&psum[s], (GB_THREADS / 32) * TPR);
    bulk::bar_fence();
  }
  __syncthreads();

  if (TILES && tid >= GB_THREADS) {         // ---- producer warp (+ tile-sum fold)
    const int lane = tid & 31;
    auto fold = [&](int kk) {
      const int sl = kk % GB_PSLOTS;
      bulk::wait(&psum[sl], (unsigned)((kk / GB_PSLOTS) & 1));
      if (lane < r) {
        const double* ps = pslot + (size_t)sl * (GB_THREADS / 32) * RMP + lane;
        double acc = 0.0;
#pragma unroll
        for (int w = 0; w < GB_THREADS / 32; ++w) acc += ps[w * RMP];
        colpart[((int64_t)blockIdx.x + (int64_t)kk * gridDim.x) * r + lane] = acc;
      }
      __syncwarp();
    };
    int k = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
      if (k >= GB_PSLOTS) fold(k - GB_PSLOTS);
      if (lane == 0) {
        const int s = k % nstage;
        if (k >= nstage) bulk::wait(&empty[s], (unsigned)((k / nstage - 1) & 1));
        const int64_t nr = min((int64_t)TR, m - t * TR);
        bulk::load(stage0 + (size_t)s * stage_elems, X + t * TR * p,
                   (unsigned)(nr * p * sizeof(T)), &full[s]);
      }
      __syncwarp();
    }
    for (int kk = max(0, k - GB_PSLOTS); kk < k; ++kk) fold(kk);
    return;
  }
  if (tid >= GB_THREADS) {                  // ---- producer warp
    if (tid == GB_THREADS) {
      int k = 0;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int s = k % nstage;
        if (k >= nstage) bulk::wait(&empty[s], (unsigned)((k / nstage - 1) & 1));
        const int64_t nr = min((int64_t)TR, m - t * TR);
        bulk::load(stage0 + (size_t)s * stage_elems, X + t * TR * p,
                   (unsigned)(nr * p * sizeof(T)), &full[s]);
      }
    }
    return;
  }

  // ---- compute warps: feature records, chunk-interleaved ((it*VW + u)*W + w)*TPR + jj
  const int nrec = nit * VW * W * TPR;
  for (int e = tid; e < nrec; e += GB_THREADS) {
    const int jj = e % TPR, w = (e / TPR) % W, fu = e / (TPR * W);
    const int it = fu / VW, u = fu % VW;
    const int a = (jj + TPR * it) * VW + u;
    double2 v2 = make_double2(0.0, 0.0);
    if (a < p) {
      if (w < RM / 2) {
        const int c = 2 * w;
        v2.x = c < r ? ctx_M[(int64_t)a * r + c] : 0.0;
        v2.y = c + 1 < r ? ctx_M[(int64_t)a * r + c + 1] : 0.0;
      } else {
        v2.x = ctx_mean[a];
        v2.y = N32 ? __hiloint2double(__float_as_int(1.0f), __float_as_int((float)ctx_mean[a]))
                   : 1.0;                   // feature mask (N32: packed with the fp32 mean)
      }
    }
    rec[e] = v2;
  }
  if (tid < 16) {                            // c0 = xbar^T M (fixed order), v
    double sacc = 0.0;
    if (tid < r)
      for (int a = 0; a < p; ++a) sacc = fma(ctx_mean[a], ctx_M[(int64_t)a * r + tid], sacc);
    c0s[tid] = sacc;
    vvs[tid] = tid < r ? ctx_v[tid] : 0.0;
  }
  asm volatile("bar.sync 1, %0;\n" ::"n"(GB_THREADS) : "memory");
  const int j = tid % TPR, g = tid / TPR, lane = tid & 31;
  double c0r[KF], vr[KF], csum[KF];
#pragma unroll
  for (int i = 0; i < KF; ++i) {
    const int c = j * KF + i;
    c0r[i] = c < 16 ? c0s[c] : 0.0;
    vr[i] = c < 16 ? vvs[c] : 0.0;
    csum[i] = 0.0;
  }
  bool bad = false;

  int k = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
    const int s = k % nstage;
    bulk::wait(&full[s], (unsigned)((k / nstage) & 1));
    const T* xs = stage0 + (size_t)s * stage_elems;
    const int64_t r0 = t * TR;
    const int nr = (int)min((int64_t)TR, m - r0);
    double acc[R][RMP], nrm[R];
    float nrm32[R];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      nrm[q] = 0.0;
      nrm32[q] = 0.0f;
#pragma unroll
      for (int c = 0; c < RMP; ++c) acc[q][c] = 0.0;
    }
    const T* x0 = xs + (size_t)g * p;
    const T* x1 = xs + (size_t)(g + G) * p;
    // branch-free, software-pipelined chunk loads: chunk indices past the row
    // are clamped to a valid chunk whose record is all-zero with mask 0
    using V = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    V n0 = *reinterpret_cast<const V*>(x0 + min(j, nchunks - 1) * VW);
    V n1 = *reinterpret_cast<const V*>(x1 + min(j, nchunks - 1) * VW);
#pragma unroll 1
    for (int it = 0; it < nit; ++it) {
      const V c0v = n0, c1v = n1;
      {
        const int chn = min(j + TPR * (it + 1), nchunks - 1);
        n0 = *reinterpret_cast<const V*>(x0 + chn * VW);
        n1 = *reinterpret_cast<const V*>(x1 + chn * VW);
      }
      double xv[R][VW];
      if constexpr (sizeof(T) == 4) {
        xv[0][0] = c0v.x; xv[0][1] = c0v.y; xv[0][2] = c0v.z; xv[0][3] = c0v.w;
        xv[1][0] = c1v.x; xv[1][1] = c1v.y; xv[1][2] = c1v.z; xv[1][3] = c1v.w;
      } else {
        xv[0][0] = c0v.x; xv[0][1] = c0v.y;
        xv[1][0] = c1v.x; xv[1][1] = c1v.y;
      }
      const double2* rp = rec + (size_t)it * VW * W * TPR + j;
#pragma unroll
      for (int u = 0; u < VW; ++u) {
        double2 mw[W];
#pragma unroll
        for (int w = 0; w < W; ++w) mw[w] = rp[(u * W + w) * TPR];
        const double mu = mw[W - 1].x, msk = mw[W - 1].y;
#pragma unroll
        for (int q = 0; q < R; ++q) {
          // linear term on the raw value (its centring is the constant c0);
          // the squared norm on the centred value (fma(x, 1, -mu) == x - mu)
          const double xq = xv[q][u];
          if constexpr (N32) {
            const float xf = (float)xq;                      // exact: the input is fp32
            const float y32 = (xf - __int_as_float(__double2loint(msk))) *
                              __int_as_float(__double2hiint(msk));
            nrm32[q] = fmaf(y32, y32, nrm32[q]);
          } else {
            const double y = fma(xq, msk, -mu);
            nrm[q] = fma(y, y, nrm[q]);
          }
#pragma unroll
          for (int w = 0; w < RM / 2; ++w) {
            acc[q][2 * w] = fma(xq, mw[w].x, acc[q][2 * w]);
            acc[q][2 * w + 1] = fma(xq, mw[w].y, acc[q][2 * w + 1]);
          }
        }
      }
    }
    // the stage is no longer read (the non-finite rescan below re-reads only
    // rows whose norm overflowed, before the release)
    bool rescan = false;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      if constexpr (N32) nrm[q] = (double)nrm32[q];
#pragma unroll
      for (int o = TPR / 2; o > 0; o >>= 1) nrm[q] += __shfl_xor_sync(0xffffffffu, nrm[q], o);
      rescan |= (g + q * G < nr) && !isfinite(nrm[q]);
    }
    if (rescan)
#pragma unroll
      for (int q = 0; q < R; ++q)
        if (g + q * G < nr && !isfinite(nrm[q])) {
          // a squared norm can overflow on finite data (fp64 rows; fp32 norms of
          // |x| > 1e19): decide on the values, recompute the norm in fp64
          const T* xr = xs + (size_t)(g + q * G) * p;
          double s2 = 0.0;
          for (int a = 0; a < p; ++a) {
            const double xa = (double)xr[a];
            bad |= !isfinite(xa);
            const double ya = xa - ctx_mean[a];
            s2 = fma(ya, ya, s2);
          }
          nrm[q] = s2;
        }
    __syncwarp();
    if (lane == 0) bulk::arrive(&empty[s]);
    double tsum[KF];
#pragma unroll
    for (int i = 0; i < KF; ++i) tsum[i] = 0.0;
#pragma unroll
    for (int q = 0; q < R; ++q) {
      // butterfly reduce-scatter: lane j keeps columns [j*KF, (j+1)*KF)
#pragma unroll
      for (int o = TPR / 2, K = RMP / 2; o > 0; o >>= 1, K >>= 1) {
        const bool up = (j & o) != 0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
          const double send = up ? acc[q][i] : acc[q][i + K];
          const double keep = up ? acc[q][i + K] : acc[q][i];
          acc[q][i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      const int row = g + q * G;
      if constexpr (TILES) {
        // branch-free sums (the butterfly below must see converged lanes)
        double* o = out + (r0 + row) * r + j * KF;
#pragma unroll
        for (int i = 0; i < KF; ++i) {
          const bool ok = row < nr && j * KF + i < r;
          const double val = fma(-nrm[q], vr[i], acc[q][i] - c0r[i]);
          if (ok) o[i] = val;
          tsum[i] += ok ? val : 0.0;
        }
      } else if (row < nr) {
        double* o = out + (r0 + row) * r + j * KF;
#pragma unroll
        for (int i = 0; i < KF; ++i)
          if (j * KF + i < r) {
            const double val = fma(-nrm[q], vr[i], acc[q][i] - c0r[i]);
            o[i] = val;
            csum[i] += val;
          }
      }
    }
    if (TILES) {
      __syncwarp();
      // the warp's rows of the tile: butterfly over the groups (fixed order)
#pragma unroll
      for (int o = TPR; o < 32; o <<= 1)
#pragma unroll
        for (int i = 0; i < KF; ++i) tsum[i] += __shfl_xor_sync(0xffffffffu, tsum[i], o);
      if (lane < TPR) {
        const int sl = k % GB_PSLOTS;
        double* ps = pslot + ((size_t)sl * (GB_THREADS / 32) + (tid >> 5)) * RMP + j * KF;
#pragma unroll
        for (int i = 0; i < KF; ++i) ps[i] = tsum[i];
        bulk::arrive(&psum[sl]);
      }
    }
  }
  if (bad) atomicOr(nonfinite, 1);
  if (!TILES && colpart != nullptr) {
    asm volatile("bar.sync 1, %0;\n" ::"n"(GB_THREADS) : "memory");   // all tiles consumed
    double* red = reinterpret_cast<double*>(stage0);
#pragma unroll
    for (int c = 0; c < RMP; ++c) red[c * GB_THREADS + tid] = (c / KF == j) ? csum[c % KF] : 0.0;
    asm volatile("bar.sync 1, %0;\n" ::"n"(GB_THREADS) : "memory");
    if (tid < r) {
      double sacc = 0.0;
      for (int i = 0; i < GB_THREADS; ++i) sacc += red[tid * GB_THREADS + i];
      colpart[(int64_t)blockIdx.x * r + tid] = sacc;
    }
  }
}

// Interpolation's landmark overwrite (algorithms.py:264-268) fused with the
// correction of the column sums: out[idx[i]] = base[i]; corr = sum(base - old).
// landmark rows <- the classical configuration; per CTA (256 landmark rows)
// the column sums of (base - old) go to corr_part[blockIdx.x] (fed to the
// re-centring as extra partials; fixed-order tree).  Rows in registers.
template <int RM>
__global__ void __launch_bounds__(256)
landmark_overwrite_kernel(const double* __restrict__ base, const int64_t* __restrict__ idx,
                          int64_t l, int r, double* __restrict__ out, double* __restrict__ corr_part) {
  __shared__ double red[256];
  double acc[RM];
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
#pragma unroll
  for (int c = 0; c < RM; ++c) acc[c] = 0.0;
  if (i < l) {
    double* o = out + idx[i] * r;
#pragma unroll
    for (int c = 0; c < RM; ++c) {
      if (c < r) {
        const double bv = base[i * r + c];
        acc[c] = bv - o[c];
        o[c] = bv;
      }
    }
  }
#pragma unroll
  for (int c = 0; c < RM; ++c) {
    if (c >= r) break;
    red[threadIdx.x] = acc[c];
    __syncthreads();
    for (int s2 = 128; s2 > 0; s2 >>= 1) {
      if (threadIdx.x < s2) red[threadIdx.x] += red[threadIdx.x + s2];
      __syncthreads();
    }
    if (threadIdx.x == 0) corr_part[(size_t)blockIdx.x * r + c] = red[0];
    __syncthreads();
  }
}

// Interpolation's landmark overwrite (algorithms.py:264-268) with the column-sum
// correction: out[pos[i]] = base[s], corr[s] = base[s] - old, s = sel[i] (the
// landmark's place in the sample; sel null -> i).  corr is indexed by sample
// position, so the re-centring folds it in the same order however the rows
// (and their landmarks) are spread over ranks.
__global__ void __launch_bounds__(256)
landmark_corr_kernel(const double* __restrict__ base, const int64_t* __restrict__ sel,
                     const int64_t* __restrict__ pos, int64_t nl, int r, double* __restrict__ out,
                     double* __restrict__ corr) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nl * r) return;
  const int64_t i = e / r;
  const int c = (int)(e - i * r);
  const int64_t si = sel ? sel[i] : i;
  double* o = out + pos[i] * r + c;
  const double bv = base[si * r + c];
  corr[si * r + c] = bv - *o;
  *o = bv;
}

// Column sums of two row-major (rows x r) arrays, level 1: block b sums the
// FOLD_ROWS-row chunk b of the concatenation [A (na rows) | B (nb rows)]
// (chunks never straddle the two), rows strided over the threads in a fixed
// order, then a fixed tree.  Level 2 (fold_total_kernel): one thread per column
// adds the chunk sums in chunk order.  The result depends on the arrays only.
constexpr int FOLD_ROWS = 1024;
constexpr int FOLD_T = 128;
template <int RM>
__global__ void __launch_bounds__(FOLD_T)
fold_chunks_kernel(const double* __restrict__ A, int64_t na, const double* __restrict__ B,
                   int64_t nb, int r, double* __restrict__ csum) {
  __shared__ double red[RM][FOLD_T];
  const int64_t cha = (na + FOLD_ROWS - 1) / FOLD_ROWS;
  const bool inA = blockIdx.x < cha;
  const double* X = inA ? A : B;
  const int64_t nx = inA ? na : nb;
  const int64_t lo = (inA ? blockIdx.x : blockIdx.x - cha) * (int64_t)FOLD_ROWS;
  const int64_t hi = min(nx, lo + FOLD_ROWS);
  double acc[RM];
#pragma unroll
  for (int c = 0; c < RM; ++c) acc[c] = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += FOLD_T)
#pragma unroll
    for (int c = 0; c < RM; ++c)
      if (c < r) acc[c] += X[i * r + c];
#pragma unroll
  for (int c = 0; c < RM; ++c) red[c][threadIdx.x] = acc[c];
  __syncthreads();
  for (int s2 = FOLD_T / 2; s2 > 0; s2 >>= 1) {
    if (threadIdx.x < s2)
#pragma unroll
      for (int c = 0; c < RM; ++c) red[c][threadIdx.x] += red[c][threadIdx.x + s2];
    __syncthreads();
  }
  if (threadIdx.x < r) csum[(int64_t)blockIdx.x * r + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void fold_total_kernel(const double* __restrict__ csum, int nch, int r,
                                  double* __restrict__ total) {
  const int c = threadIdx.x;
  if (c >= r) return;
  double s = 0.0;
  for (int b = 0; b < nch; ++b) s += csum[(int64_t)b * r + c];
  total[c] = s;
}

}  // namespace

namespace mdsx {

int launch_landmark_overwrite(mdsx_handle* h, const double* base, const int64_t* idx, int64_t l,
                              int r, double* out, double* corr, cudaStream_t st) {
  mdsx::pre(h, st);
  const unsigned nb = (unsigned)((l + 255) / 256);
  auto go = [&](auto rm) {
    constexpr int RM = decltype(rm)::value;
    landmark_overwrite_kernel<RM><<<nb, 256, 0, st>>>(base, idx, l, r, out, corr);
  };
  if (r <= 4) go(std::integral_constant<int, 4>{});
  else if (r <= 10) go(std::integral_constant<int, 10>{});
  else if (r <= 16) go(std::integral_constant<int, 16>{});
  else go(std::integral_constant<int, 32>{});
  return launched(h, "landmark_overwrite_kernel", st);
}

int launch_landmark_corr(mdsx_handle* h, const double* base, const int64_t* sel,
                         const int64_t* pos, int64_t nl, int r, double* out, double* corr,
                         cudaStream_t st) {
  if (nl == 0) return MDSX_OK;
  mdsx::pre(h, st);
  landmark_corr_kernel<<<(unsigned)((nl * r + 255) / 256), 256, 0, st>>>(base, sel, pos, nl, r, out, corr);
  return launched(h, "landmark_corr_kernel", st);
}

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

size_t fold_ws_bytes(int64_t na, int64_t nb, int r) {
  const int64_t nch = (na + FOLD_ROWS - 1) / FOLD_ROWS + (nb + FOLD_ROWS - 1) / FOLD_ROWS;
  return al256((size_t)std::max<int64_t>(nch, 1) * r * sizeof(double)) + al256((size_t)r * sizeof(double));
}

// total[c] = sum of column c over A (na x r) then B (nb x r); ws: fold_ws_bytes
int launch_fold_sums(mdsx_handle* h, const double* A, int64_t na, const double* B, int64_t nb,
                     int r, double* ws, double** total, cudaStream_t st) {
  const int64_t nch = (na + FOLD_ROWS - 1) / FOLD_ROWS + (nb + FOLD_ROWS - 1) / FOLD_ROWS;
  double* csum = ws;
  *total = ws + al256((size_t)std::max<int64_t>(nch, 1) * r * sizeof(double)) / sizeof(double);
  if (nch > 0) {
    mdsx::pre(h, st);
    if (r <= 4) fold_chunks_kernel<4><<<(unsigned)nch, FOLD_T, 0, st>>>(A, na, B, nb, r, csum);
    else if (r <= 10) fold_chunks_kernel<10><<<(unsigned)nch, FOLD_T, 0, st>>>(A, na, B, nb, r, csum);
    else if (r <= 16) fold_chunks_kernel<16><<<(unsigned)nch, FOLD_T, 0, st>>>(A, na, B, nb, r, csum);
    else fold_chunks_kernel<32><<<(unsigned)nch, FOLD_T, 0, st>>>(A, na, B, nb, r, csum);
    int rc = launched(h, "fold_chunks_kernel", st);
    if (rc) return rc;
  }
  mdsx::pre(h, st);
  fold_total_kernel<<<1, 32, 0, st>>>(csum, (int)nch, r, *total);
  return launched(h, "fold_total_kernel", st);
}

// Bulk-copy Gower over m dense rows.  colpart (optional) receives column sums:
// tiles = false: one r-vector per CTA, *nparts = the number of CTAs; tiles =
// true: one r-vector per tile (tile t at colpart[t * r]), *nparts = rows per
// tile.  *nparts = 0 when the shape does not fit (nothing launched).
struct GbConfig { int TPR = 0, nstage = 0; size_t smem = 0; };

static GbConfig gower_bulk_config(mdsx_handle* h, int dtype, int p, int r, bool tiles) {
  GbConfig g;
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  const int VW = (int)(16 / es);
  const int RM = r <= 4 ? 4 : r <= 8 ? 8 : r <= 10 ? 10 : r <= 12 ? 12 : 16;
  if (r > 16 || ((size_t)p * es) % 16 != 0) return g;
  const size_t cap = (size_t)(h && h->max_smem_optin > 0 ? h->max_smem_optin : 227 * 1024);
  const size_t sm_total = 228 * 1024;               // shared memory per SM
  const char* e_tpr = getenv("MDSX_GB_TPR");
  const int force_tpr = e_tpr ? atoi(e_tpr) : 0;
  // one CTA (8 compute warps + producer) per SM; TPR as small as the stage allows
  for (int tpr = 2; tpr <= 32 && !g.TPR; tpr *= 2) {
    if (force_tpr && tpr != force_tpr) continue;
    const int TR = 2 * GB_THREADS / tpr;
    const int nit = (p / VW + tpr - 1) / tpr;
    const size_t recb = (size_t)nit * VW * (RM / 2 + 1) * tpr * 16;
    const size_t stage = (size_t)TR * p * es;
    const size_t rmp = (size_t)((RM + tpr - 1) / tpr * tpr);
    const size_t red = tiles ? 0 : rmp * GB_THREADS * 8;
    const size_t slots = tiles ? (size_t)GB_PSLOTS * (GB_THREADS / 32) * rmp * 8 : 0;
    for (int ns = GB_MAX_STAGES; ns >= 2; --ns) {
      const size_t need = GB_HEADER + recb + slots + std::max(ns * stage, red);
      if (stage <= 112 * 1024 && need <= cap && need + 1024 <= sm_total) {
        g.TPR = tpr; g.nstage = ns; g.smem = need;
        break;
      }
    }
  }
  return g;
}

int gower_tile_rows(mdsx_handle* h, int dtype, int p, int r) {
  const GbConfig g = gower_bulk_config(h, dtype, p, r, true);
  return g.TPR ? 2 * GB_THREADS / g.TPR : 0;
}

int launch_gower_bulk(mdsx_handle* h, const void* X, int dtype, int64_t m, int p, int r,
                      const double* mean, const double* M, const double* v, double* out,
                      double* colpart, int32_t* nonfinite, int* nparts, cudaStream_t st,
                      bool norm32, bool tiles) {
  *nparts = 0;
  const int RM = r <= 4 ? 4 : r <= 8 ? 8 : r <= 10 ? 10 : r <= 12 ? 12 : 16;
  tiles = tiles && colpart != nullptr;
  const GbConfig cfg = gower_bulk_config(h, dtype, p, r, tiles);
  const int TPR = cfg.TPR, nstage = cfg.nstage;
  const size_t smem = cfg.smem;
  if (!TPR) return MDSX_OK;
  if (m == 0) {
    *nparts = tiles ? 2 * GB_THREADS / TPR : 0;
    return MDSX_OK;
  }
  auto go = [&](auto tag, auto rm, auto tpr) -> int {
    using T = decltype(tag);
    constexpr int RMc = decltype(rm)::value;
    constexpr int TPRc = decltype(tpr)::value;
    auto kern = tiles ? gower_bulk_kernel<T, RMc, TPRc, 1, false, true>
                      : gower_bulk_kernel<T, RMc, TPRc, 1, false, false>;
    if constexpr (sizeof(T) == 4)
      if (norm32) kern = tiles ? gower_bulk_kernel<T, RMc, TPRc, 1, true, true>
                               : gower_bulk_kernel<T, RMc, TPRc, 1, true, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t TR = 2 * GB_THREADS / TPRc;
    const int64_t ntiles = (m + TR - 1) / TR;
    const int blocks = (int)std::min<int64_t>(ntiles, (int64_t)h->num_sms);
    mdsx::pre(h, st);
    kern<<<blocks, GB_CTA, smem, st>>>((const T*)X, m, p, r, mean, M, v, out, colpart,
                                           nonfinite, nstage);
    const int rc = launched(h, "gower_bulk_kernel", st);
    if (!rc) *nparts = tiles ? (int)TR : colpart ? blocks : -1;
    return rc;
  };
  auto by_tpr = [&](auto tag, auto rm) -> int {
    switch (TPR) {
      case 2: return go(tag, rm, std::integral_constant<int, 2>{});
      case 4: return go(tag, rm, std::integral_constant<int, 4>{});
      case 8: return go(tag, rm, std::integral_constant<int, 8>{});
      case 16: return go(tag, rm, std::integral_constant<int, 16>{});
      default: return go(tag, rm, std::integral_constant<int, 32>{});
    }
  };
  auto by_rm = [&](auto tag) -> int {
    switch (RM) {
      case 4: return by_tpr(tag, std::integral_constant<int, 4>{});
      case 8: return by_tpr(tag, std::integral_constant<int, 8>{});
      case 10: return by_tpr(tag, std::integral_constant<int, 10>{});
      case 12: return by_tpr(tag, std::integral_constant<int, 12>{});
      default: return by_tpr(tag, std::integral_constant<int, 16>{});
    }
  };
  return dtype == MDSX_F32 ? by_rm(float{}) : by_rm(double{});
}

int launch_gower_context(mdsx_handle* h, const void* X, int dtype, int64_t ld, int p,
                         const int64_t* idx, int64_t l, const double* X1, int r, double* mean,
                         double* M, double* v, double* S, double* q, double* cond, int32_t* flag,
                         cudaStream_t st) {
  auto feat = [&](auto tag) {
    using T = decltype(tag);
    const T* x = (const T*)X;
    if (r <= 4) { mdsx::pre(h, st); ctx_feature_kernel<T, 4><<<p, 256, 0, st>>>(x, ld, idx, l, p, X1, r, mean, M); }
    else if (r <= 8) { mdsx::pre(h, st); ctx_feature_kernel<T, 8><<<p, 256, 0, st>>>(x, ld, idx, l, p, X1, r, mean, M); }
    else if (r <= 16) { mdsx::pre(h, st); ctx_feature_kernel<T, 16><<<p, 256, 0, st>>>(x, ld, idx, l, p, X1, r, mean, M); }
    else { mdsx::pre(h, st); ctx_feature_kernel<T, 32><<<p, 256, 0, st>>>(x, ld, idx, l, p, X1, r, mean, M); }
    int rc = launched(h, "ctx_feature_kernel", st);
    if (rc) return rc;
    mdsx::pre(h, st);
    ctx_qdiag_kernel<T><<<(unsigned)((l + 255) / 256), 256, 0, st>>>(x, ld, idx, l, p, mean, q);
    return launched(h, "ctx_qdiag_kernel", st);
  };
  int rc = dtype == MDSX_F64 ? feat(double{}) : feat(float{});
  if (rc) return rc;
  mdsx::pre(h, st);
  ctx_finalize_kernel<<<1, 256, 0, st>>>(X1, l, p, r, M, v, S, cond, flag);
  return launched(h, "ctx_finalize_kernel", st);
}

int launch_gower_stream(mdsx_handle* h, const void* X, int dtype, int64_t m, int p, int r,
                        const double* mean, const double* M, const double* v, double* out,
                        int32_t* nonfinite, cudaStream_t st) {
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  auto go = [&](auto tag, auto rm) {
    using T = decltype(tag);
    constexpr int RM = decltype(rm)::value;
    auto kern = gower_stream_kernel<T, RM>;
    const size_t fixed = ((size_t)p * RM + p) * sizeof(double);
    int TR = 128;                                 // rows per stage: one per thread pair
    while (TR > 8 && fixed + 2 * (size_t)TR * p * es > 110 * 1024) TR >>= 1;
    const size_t smem = fixed + 2 * (size_t)TR * p * es;
    if (smem > 222 * 1024) return -1;             // caller falls back to the per-row kernel
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t ntiles = (m + TR - 1) / TR;
    const int blocks = (int)std::min<int64_t>(ntiles, (int64_t)h->num_sms * 2);
    mdsx::pre(h, st);
    kern<<<blocks, 256, smem, st>>>((const T*)X, m, p, r, mean, M, v, out, nonfinite, TR);
    return launched(h, "gower_stream_kernel", st);
  };
  using I4 = std::integral_constant<int, 4>;
  using I8 = std::integral_constant<int, 8>;
  using I12 = std::integral_constant<int, 12>;
  using I16 = std::integral_constant<int, 16>;
  if (dtype == MDSX_F32)
    return r <= 4 ? go(float{}, I4{}) : r <= 8 ? go(float{}, I8{}) : r <= 12 ? go(float{}, I12{}) : go(float{}, I16{});
  return r <= 4 ? go(double{}, I4{}) : r <= 8 ? go(double{}, I8{}) : r <= 12 ? go(double{}, I12{}) : go(double{}, I16{});
}


int launch_gower_affine(mdsx_handle* h, const void* X, int dtype, int64_t ld, int64_t m, int p,
                        int r, const double* mean, const double* M, const double* v, double* out,
                        int64_t ldo, int32_t* nonfinite, cudaStream_t st) {
  if (m == 0) return MDSX_OK;
  // dense rows (ld == p), dense output, 16-byte aligned rows: cp.async streaming kernel
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  if (ld == p && ldo == r && r <= 16 && ((size_t)p * es) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(X) & 15) == 0) {
    int launched_parts = 0;
    int rc = launch_gower_bulk(h, X, dtype, m, p, r, mean, M, v, out, nullptr, nonfinite,
                               &launched_parts, st, false, false);
    if (rc || launched_parts) return rc;
    rc = launch_gower_stream(h, X, dtype, m, p, r, mean, M, v, out, nonfinite, st);
    if (rc >= 0) return rc;                       // -1: shape does not fit the staged kernel
  }
  auto go = [&](auto tag, auto rm) {
    using T = decltype(tag);
    constexpr int RM = decltype(rm)::value;
    auto kern = gower_affine_kernel<T, RM>;
    const size_t smem = ((size_t)p * RM + p) * sizeof(double);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int per_sm = 4;
    const int64_t need = (m + 255) / 256;
    const int blocks = (int)std::min<int64_t>(need, (int64_t)h->num_sms * per_sm);
    mdsx::pre(h, st);
    kern<<<blocks, 256, smem, st>>>((const T*)X, ld, m, p, r, mean, M, v, out, ldo, nonfinite);
    return launched(h, "gower_affine_kernel", st);
  };
  using I4 = std::integral_constant<int, 4>;
  using I8 = std::integral_constant<int, 8>;
  using I12 = std::integral_constant<int, 12>;
  using I16 = std::integral_constant<int, 16>;
  using I32 = std::integral_constant<int, 32>;
  if (dtype == MDSX_F64) {
    if (r <= 4) return go(double{}, I4{});
    if (r <= 8) return go(double{}, I8{});
    if (r <= 12) return go(double{}, I12{});
    if (r <= 16) return go(double{}, I16{});
    return go(double{}, I32{});
  }
  if (r <= 4) return go(float{}, I4{});
  if (r <= 8) return go(float{}, I8{});
  if (r <= 12) return go(float{}, I12{});
  if (r <= 16) return go(float{}, I16{});
  return go(float{}, I32{});
}

}  // namespace mdsx
