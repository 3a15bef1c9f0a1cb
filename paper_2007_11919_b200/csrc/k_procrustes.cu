// K5 Procrustes (procrustes.py:46-105, linalg.py:186-205) and K6/K7
// stitching: recentering (algorithms.py:122-125) and row scatters
// (algorithms.py:146-156, 341-342).
//
// fit: one warp per job.  Cross-product of the centred configurations
// (r x r), then a one-sided (Hestenes) Jacobi SVD in shared memory: the
// columns of B = cross are orthogonalised by plane rotations accumulated in
// V, so cross = L diag(sigma) V^T with L = B / sigma.  The rotation is
// T = V L^T = sum_i v_i l_i^T, which is independent of the order and paired
// signs of the singular triplets — the same T thin_svd + right @ left.T gives.
#include "mdsx_common.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace {

constexpr int FIT_WARPS = 4;

// Rotation of the orthogonal Procrustes problem from the r x r cross-product
// B (procrustes.py:46-50): one-sided (Hestenes) Jacobi SVD on the columns of B
// (lane a owns row a; B and V in shared memory, V starts as the identity),
// rank-deficient left bases completed by Gram-Schmidt, T = V L^T written to T
// (row-major, may be global memory).  One warp; smin / smax are the extreme
// singular values (the degenerate flag, procrustes.py:48).
__device__ void rotation_from_cross(double* B, double* V, double* sg, int r, int lane, double* T,
                                    double& smin_out, double& smax_out) {
  // one-sided Jacobi on the columns of B (lane a owns row a)
  for (int sweep = 0; sweep < 60; ++sweep) {
    int nrot = 0;
    for (int i = 0; i < r - 1; ++i)
      for (int j = i + 1; j < r; ++j) {
        const double x = lane < r ? B[lane * r + i] : 0.0;
        const double y = lane < r ? B[lane * r + j] : 0.0;
        // the three column dots reduced together (interleaved shuffle trees)
        double al = x * x, be = y * y, ga = x * y;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (ga != 0.0 && ga * ga > 1e-30 * (al * be)) {
          // t = tan of the rotation angle, |t| <= 1 (one sqrt, one divide, one rsqrt)
          const double h = 0.5 * (be - al);
          const double t = ga / (h + copysign(sqrt(fma(h, h, ga * ga)), h == 0.0 ? 1.0 : h));
          const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
          if (lane < r) {
            B[lane * r + i] = c * x - s * y;
            B[lane * r + j] = s * x + c * y;
            const double vx = V[lane * r + i], vy = V[lane * r + j];
            V[lane * r + i] = c * vx - s * vy;
            V[lane * r + j] = s * vx + c * vy;
          }
          ++nrot;
        }
        __syncwarp();
      }
    if (nrot == 0) break;
  }
  // singular values and left vectors (columns of B normalised)
  double smax = 0.0, smin = 1e308;
  for (int i = 0; i < r; ++i) {
    const double x = lane < r ? B[lane * r + i] : 0.0;
    const double s = sqrt(mdsx::warp_sum(x * x));
    if (lane == 0) sg[i] = s;
    smax = fmax(smax, s);
    smin = fmin(smin, s);
  }
  __syncwarp();
  for (int i = 0; i < r; ++i) {
    const double s = sg[i];
    if (s > 1e-15 * smax && s > 0.0 && lane < r) B[lane * r + i] /= s;
  }
  __syncwarp();
  for (int i = 0; i < r; ++i) {
    const double s = sg[i];
    if (s > 1e-15 * smax && s > 0.0) continue;
    // rank-deficient: complete the left basis by Gram-Schmidt on the e_q that
    // leaves the largest remainder (lane q's squared row norm over the basis)
    double n2 = 1.0;
    for (int l = 0; l < r; ++l) {
      if (l == i) continue;
      const bool good = sg[l] > 1e-15 * smax && sg[l] > 0.0;
      if (!good && l > i) continue;
      const double ll = lane < r ? B[lane * r + l] : 0.0;
      n2 -= ll * ll;
    }
    double best = lane < r ? n2 : -2.0;
    int qb = lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double b2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int q2 = __shfl_xor_sync(0xffffffffu, qb, o);
      if (b2 > best || (b2 == best && q2 < qb)) { best = b2; qb = q2; }
    }
    double v = (lane == qb) ? 1.0 : 0.0;
    for (int pass = 0; pass < 2; ++pass)
      for (int l = 0; l < r; ++l) {
        if (l == i) continue;
        const bool good = sg[l] > 1e-15 * smax && sg[l] > 0.0;
        if (!good && l > i) continue;
        const double ll = lane < r ? B[lane * r + l] : 0.0;
        const double dot = mdsx::warp_sum(ll * v);
        v -= dot * ll;
      }
    const double nv = sqrt(mdsx::warp_sum(lane < r ? v * v : 0.0));
    if (lane < r) B[lane * r + i] = v / nv;
    __syncwarp();
  }
  // T = V L^T  (row a of T on lane a)
  if (lane < r)
    for (int b = 0; b < r; ++b) {
      double s = 0.0;
      for (int i = 0; i < r; ++i) s = fma(V[lane * r + i], B[b * r + i], s);
      T[lane * r + b] = s;
    }
  smin_out = smin;
  smax_out = smax;
}

__global__ void __launch_bounds__(FIT_WARPS * 32)
procrustes_fit_kernel(const double* __restrict__ tgt, const int64_t* __restrict__ tgt_rows,
                      const double* __restrict__ src, const int64_t* __restrict__ src_rows,
                      const int64_t* __restrict__ job_off, int njobs, int r,
                      double* __restrict__ rot, double* __restrict__ trans,
                      double* __restrict__ loss, int32_t* __restrict__ degenerate) {
  extern __shared__ double sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int job = blockIdx.x * FIT_WARPS + warp;
  if (job >= njobs) return;
  double* B = sm + (size_t)warp * (2 * r * r + 3 * r);
  double* V = B + r * r;
  double* mt = V + r * r;
  double* ms = mt + r;
  double* sg = ms + r;
  const int64_t o = job_off[job];
  const int K = (int)(job_off[job + 1] - o);
  const int64_t* tr = tgt_rows + o;
  const int64_t* sr = src_rows + o;

  if (lane < r) {
    double a = 0.0, b = 0.0;
    for (int t = 0; t < K; ++t) {
      a += tgt[tr[t] * r + lane];
      b += src[sr[t] * r + lane];
    }
    mt[lane] = a / K;
    ms[lane] = b / K;
  }
  __syncwarp();
  for (int e = lane; e < r * r; e += 32) {
    const int a = e / r, b = e % r;
    double s = 0.0;
    for (int t = 0; t < K; ++t)
      s = fma(tgt[tr[t] * r + a] - mt[a], src[sr[t] * r + b] - ms[b], s);
    B[e] = s;
    V[e] = (a == b) ? 1.0 : 0.0;
  }
  __syncwarp();

  double smin, smax;
  double* T = rot + (size_t)job * r * r;
  rotation_from_cross(B, V, sg, r, lane, T, smin, smax);
  __syncwarp();
  // translation t = mean(tgt) - mean(src) T ; loss
  double* tv = trans + (size_t)job * r;
  if (lane < r) {
    double s = 0.0;
    for (int a = 0; a < r; ++a) s = fma(ms[a], T[a * r + lane], s);
    tv[lane] = mt[lane] - s;
  }
  __syncwarp();
  double ls = 0.0;
  if (lane < r) {
    const double tl = tv[lane];
    for (int t = 0; t < K; ++t) {
      double s = 0.0;
      for (int a = 0; a < r; ++a) s = fma(src[sr[t] * r + a], T[a * r + lane], s);
      const double e = tgt[tr[t] * r + lane] - s - tl;
      ls = fma(e, e, ls);
    }
  }
  ls = mdsx::warp_sum(ls);
  if (lane == 0) {
    loss[job] = ls;
    degenerate[job] = (r == 0 || smin <= 1e-12 * smax) ? 1 : 0;
  }
}

// ---- register-resident fit for r <= 16: a group of P = ceil(r/2) lanes per
// fit, 32/P fits per warp.  Lane l of a group holds two columns of B (and of
// V) in registers, so the three column dots of a Jacobi rotation are local
// FMAs (no shuffle trees); the P lanes rotate P disjoint column pairs at once
// and then pass columns along a round-robin (Brent-Luk tournament) ordering,
// so one sweep visits every pair in 2P-1 rounds.  A sweep with no rotation
// ends the fit (further sweeps are no-ops, so groups of one warp simply run
// until the slowest converges).  T = V L^T, t, loss and the degenerate flag
// as procrustes_fit_kernel (the same rule for rank-deficient left bases).
// ---- fast path for well-conditioned fits (r <= 16, K <= NS_KMAX rows):
// one warp per fit, the K target/source rows staged in shared memory, the
// cross-product B (r x r) formed by the 32 lanes, and its orthogonal polar
// factor Q = L V^T (B = L S V^T) by the Newton-Schulz iteration
//     X_0 = B / |B|_F,   X_{k+1} = X_k (3 I - X_k^T X_k) / 2,
// quadratically convergent once the singular values of X_k are near 1 and
// multiplying small ones by ~1.5 per step before that: a warp-parallel
// sequence of r x r products instead of the serial plane rotations of the
// Jacobi SVD.  T = V L^T = Q^T (the rotation procrustes.py:46-78 forms as
// right @ left.T; the polar factor is unique for nonsingular B, so T is the
// same).  Converged within NS_ITMAX steps  =>  s_min / s_max >~ 1e-7, so the
// fit is not degenerate (procrustes.py:48, ratio 1e-12).  Fits that do not
// converge (near-singular or rank-deficient B, whose rotation depends on the
// completion of the left basis) or have more than NS_KMAX rows are marked
// degenerate = -1 and recomputed by the Jacobi kernel launched right after.
constexpr int NS_WARPS = 4;
constexpr int NS_KMAX = 64;
constexpr int NS_ITMAX = 40;

// The Newton-Schulz fit of one warp: xs / ys hold the K target / source rows
// (R values each, overwritten by the centred rows); on success T (row-major,
// global), t and the loss are written and true returned; false when the
// iteration did not converge (the Jacobi kernel takes the fit).  On return Gs
// holds T, mx / my the column means.
template <int R>
__device__ bool ns_fit_warp(double* xs, double* ys, double* Xs, double* Gs, double* mx, double* my,
                            double* tv, int K, int lane, double* __restrict__ T,
                            double* __restrict__ trans_j, double* __restrict__ loss_j) {
  constexpr int RR = R * R;
  constexpr int Q = (RR + 31) / 32;                 // matrix entries per lane
  // lane entries e = lane + 32 q of an R x R matrix: row ea[q], column eb[q]
  int ea[Q], eb[Q];
  bool ev[Q];
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    const int e = lane + 32 * q;
    ev[q] = e < RR;
    ea[q] = ev[q] ? e / R : 0;
    eb[q] = ev[q] ? e - ea[q] * R : 0;
  }
  __syncwarp();
  if (lane < R || (lane >= 16 && lane - 16 < R)) {
    const int a = lane & 15;
    const double* v = lane < 16 ? xs : ys;
    double m0 = 0.0, m1 = 0.0;
    int t = 0;
    for (; t + 1 < K; t += 2) {
      m0 += v[t * R + a];
      m1 += v[(t + 1) * R + a];
    }
    if (t < K) m0 += v[t * R + a];
    (lane < 16 ? mx : my)[a] = (m0 + m1) / K;
  }
  __syncwarp();
  for (int e = lane; e < K * R; e += 32) {          // centre in place
    const int a = e % R;
    xs[e] -= mx[a];
    ys[e] -= my[a];
  }
  __syncwarp();
  // B[a][b] = sum_t x_t[a] y_t[b] (centred)
  double fro = 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (ev[q]) {
      double c0 = 0.0, c1 = 0.0;
      int t = 0;
      for (; t + 1 < K; t += 2) {
        c0 = fma(xs[t * R + ea[q]], ys[t * R + eb[q]], c0);
        c1 = fma(xs[(t + 1) * R + ea[q]], ys[(t + 1) * R + eb[q]], c1);
      }
      if (t < K) c0 = fma(xs[t * R + ea[q]], ys[t * R + eb[q]], c0);
      const double bv = c0 + c1;
      Gs[lane + 32 * q] = bv;
      fro = fma(bv, bv, fro);
    }
  }
  fro = mdsx::warp_sum(fro);
  __syncwarp();
  // scale by a guaranteed upper bound of s_max, min(|B|_F, sqrt(|B|_1 |B|_inf)):
  // every singular value of X_0 then lies in (0, 1] and the iteration stays
  // monotone (a value above sqrt(3) would converge to -1, a wrong rotation)
  double smax = sqrt(fro);
  {
    double rs = 0.0, cs = 0.0;
    if (lane < R) {
#pragma unroll
      for (int c = 0; c < R; ++c) {
        rs += fabs(Gs[lane * R + c]);
        cs += fabs(Gs[c * R + lane]);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      rs = fmax(rs, __shfl_xor_sync(0xffffffffu, rs, off));
      cs = fmax(cs, __shfl_xor_sync(0xffffffffu, cs, off));
    }
    smax = fmin(smax, sqrt(rs * cs));
  }
  const double inv = fro > 0.0 ? 1.0 / smax : 0.0;
#pragma unroll
  for (int q = 0; q < Q; ++q)
    if (ev[q]) Xs[lane + 32 * q] = Gs[lane + 32 * q] * inv;
  __syncwarp();
  bool conv = false, last = false;
  for (int it = 0; it < NS_ITMAX && fro > 0.0; ++it) {
    double dev = 0.0;
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if (ev[q]) {
        double g = 0.0;
#pragma unroll
        for (int i = 0; i < R; ++i) g = fma(Xs[i * R + ea[q]], Xs[i * R + eb[q]], g);
        Gs[lane + 32 * q] = g;
        dev = fmax(dev, fabs(g - (ea[q] == eb[q] ? 1.0 : 0.0)));
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dev = fmax(dev, __shfl_xor_sync(0xffffffffu, dev, off));
    if (dev < 1e-10) last = true;                   // one more step: error ~ dev^2, rounding-limited
    __syncwarp();
    double nx[Q];
#pragma unroll
    for (int q = 0; q < Q; ++q) {
      if (ev[q]) {
        double s2 = 0.0;
#pragma unroll
        for (int a = 0; a < R; ++a) s2 = fma(Xs[ea[q] * R + a], Gs[a * R + eb[q]], s2);
        nx[q] = fma(1.5, Xs[lane + 32 * q], -0.5 * s2);
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < Q; ++q)
      if (ev[q]) Xs[lane + 32 * q] = nx[q];
    __syncwarp();
    if (last) { conv = true; break; }
  }
  if (!conv) return false;
  // T = Q^T (row-major), t = mx - my T, loss
#pragma unroll
  for (int q = 0; q < Q; ++q) {
    if (ev[q]) {
      const double v = Xs[eb[q] * R + ea[q]];
      T[lane + 32 * q] = v;
      Gs[lane + 32 * q] = v;
    }
  }
  __syncwarp();
  if (lane < R) {
    double s2 = 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a) s2 = fma(my[a], Gs[a * R + lane], s2);
    const double t = mx[lane] - s2;
    tv[lane] = t;
    trans_j[lane] = t;
  }
  __syncwarp();
  // residuals of the centred rows: x_c - y_c T (the translation absorbs the means)
  double ls = 0.0;
  for (int e = lane; e < K * R; e += 32) {
    const int t = e / R, b = e - t * R;
    double s2 = 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a) s2 = fma(ys[t * R + a], Gs[a * R + b], s2);
    const double d = xs[e] - s2;
    ls = fma(d, d, ls);
  }
  ls = mdsx::warp_sum(ls);
  if (lane == 0) *loss_j = ls;
  return true;
}


template <int R>
__global__ void __launch_bounds__(NS_WARPS * 32)
procrustes_fit_ns_kernel(const double* __restrict__ tgt, const int64_t* __restrict__ tgt_rows,
                         const double* __restrict__ src, const int64_t* __restrict__ src_rows,
                         const int64_t* __restrict__ job_off, int njobs,
                         double* __restrict__ rot, double* __restrict__ trans,
                         double* __restrict__ loss, int32_t* __restrict__ degenerate) {
  constexpr int RR = R * R;
  constexpr int WS = 2 * NS_KMAX * R + 2 * RR + 3 * R;
  extern __shared__ double nsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int job = blockIdx.x * NS_WARPS + warp;
  if (job >= njobs) return;
  double* xs = nsm + (size_t)warp * WS;
  double* ys = xs + NS_KMAX * R;
  double* Xs = ys + NS_KMAX * R;
  double* Gs = Xs + RR;
  double* mx = Gs + RR;
  double* my = mx + R;
  double* tv = my + R;
  const int64_t o = job_off[job];
  const int K = (int)(job_off[job + 1] - o);
  if (K > NS_KMAX || K < 1) {
    if (lane == 0) degenerate[job] = -1;
    return;
  }
  {
    // row indices then values, loads batched (K <= NS_KMAX = 64 rows: two passes
    // of 32 lanes), so a fit waits for two dependent latencies, not 2 K R / 32
    int64_t tr0 = 0, sr0 = 0, tr1 = 0, sr1 = 0;
    if (lane < K) { tr0 = tgt_rows[o + lane]; sr0 = src_rows[o + lane]; }
    if (lane + 32 < K) { tr1 = tgt_rows[o + lane + 32]; sr1 = src_rows[o + lane + 32]; }
    constexpr int EPL = (NS_KMAX * R + 31) / 32;      // elements per lane (upper bound)
    double xv[EPL], yv[EPL];
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int e = lane + 32 * u;
      const int t = min(e, K * R - 1) / R, a = min(e, K * R - 1) - t * R;
      const int64_t ta = __shfl_sync(0xffffffffu, tr0, t & 31), tb = __shfl_sync(0xffffffffu, tr1, t & 31);
      const int64_t sa = __shfl_sync(0xffffffffu, sr0, t & 31), sb = __shfl_sync(0xffffffffu, sr1, t & 31);
      if (e < K * R) {
        xv[u] = tgt[(t < 32 ? ta : tb) * R + a];
        yv[u] = src[(t < 32 ? sa : sb) * R + a];
      }
    }
#pragma unroll
    for (int u = 0; u < EPL; ++u) {
      const int e = lane + 32 * u;
      if (e < K * R) {
        xs[e] = xv[u];
        ys[e] = yv[u];
      }
    }
  }
  const bool ok = ns_fit_warp<R>(xs, ys, Xs, Gs, mx, my, tv, K, lane, rot + (size_t)job * RR,
                                 trans + (size_t)job * R, loss + job);
  if (lane == 0) degenerate[job] = ok ? 0 : -1;   // -1: the Jacobi kernel takes this fit
}

// ---- D&C tail of one subset j >= 1 in one warp (k_dcout.cu route): the
// points of its c connecting rows P = (x - mu_j) U_j (written to Pc for a
// Jacobi redo), the Newton-Schulz fit onto the anchor's signed targets, and
// when it converged the composition U'_j = U_j T_j, t_j and the subset's
// contribution to the column sum, -(sum_i P_i) T_j + (m_j - c) t_j
// (dc_compose_kernel's arithmetic); otherwise pending[j] = 1 and the Jacobi
// fit + dc_compose_kernel (pending mode) finish it.
template <int R, typename T>
__global__ void __launch_bounds__(NS_WARPS * 32)
dc_fit_kernel(const T* __restrict__ X, int64_t ld, int p, const int64_t* __restrict__ row_idx,
              const PieceDesc* __restrict__ pd, int npieces, int c,
              const double* __restrict__ mu_all, const double* __restrict__ Uall,
              double* __restrict__ Pc, double* __restrict__ rot, double* __restrict__ trans,
              double* __restrict__ loss, int32_t* __restrict__ degenerate,
              double* __restrict__ Uc, double* __restrict__ tvec, double* __restrict__ contrib,
              int32_t* __restrict__ pending) {
  constexpr int RR = R * R;
  constexpr int WS = 2 * NS_KMAX * R + 2 * RR + 3 * R + R;
  extern __shared__ double nsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = 1 + blockIdx.x * NS_WARPS + warp;
  // layout: per-warp NS areas, then the c connecting rows (shared: the same rows
  // for every subset), then per warp U_j (p x R) and mu_j (p)
  double* xs = nsm + (size_t)warp * WS;
  double* ys = xs + NS_KMAX * R;
  double* Xs = ys + NS_KMAX * R;
  double* Gs = Xs + RR;
  double* mx = Gs + RR;
  double* my = mx + R;
  double* tv = my + R;
  double* cs = tv + R;
  double* rows = nsm + (size_t)NS_WARPS * WS;
  double* Us = rows + (size_t)c * p + (size_t)warp * (p * R + p);
  double* mus = Us + (size_t)p * R;
  const bool act = j < npieces;
  const PieceDesc d = pd[act ? j : 1];
  {
    // connecting rows: subset 1's first c row indices (every subset starts with them)
    const PieceDesc d1 = pd[1];
    for (int e = threadIdx.x; e < c * p; e += blockDim.x) {
      const int t = e / p, a = e - t * p;
      rows[e] = (double)X[row_idx[d1.row_off + t] * ld + a];
    }
  }
  if (act) {
    const double* U = Uall + d.u_off;
    const double* mu = mu_all + (int64_t)d.id * p;
    for (int e = lane; e < p * R; e += 32) Us[e] = U[e];
    for (int e = lane; e < p; e += 32) mus[e] = mu[e];
  }
  __syncthreads();
  if (!act) return;
  const int K = c;
  for (int e = lane; e < K * R; e += 32) xs[e] = Pc[e];   // the anchor's signed targets
  // sources: points of the c connecting rows, lanes over (row, column) outputs
  double* Pj = Pc + (int64_t)j * c * R;
  for (int e = lane; e < K * R; e += 32) {
    const int t = e / R, q = e - t * R;
    const double* row = rows + (size_t)t * p;
    double s0 = 0.0, s1 = 0.0;
    int a = 0;
    for (; a + 1 < p; a += 2) {
      s0 = fma(row[a] - mus[a], Us[a * R + q], s0);
      s1 = fma(row[a + 1] - mus[a + 1], Us[(a + 1) * R + q], s1);
    }
    if (a < p) s0 = fma(row[a] - mus[a], Us[a * R + q], s0);
    const double v = s0 + s1;
    ys[e] = v;
    Pj[e] = v;
  }
  __syncwarp();
  if (lane < R) {                                    // column sums of the raw source points
    double s2 = 0.0;
    for (int t = 0; t < K; ++t) s2 += ys[t * R + lane];
    cs[lane] = s2;
  }
  const bool ok = ns_fit_warp<R>(xs, ys, Xs, Gs, mx, my, tv, K, lane, rot + (size_t)(j - 1) * RR,
                                 trans + (size_t)(j - 1) * R, loss + (j - 1));
  if (lane == 0) {
    degenerate[j - 1] = ok ? 0 : -1;
    pending[j] = ok ? 0 : 1;
  }
  if (!ok) return;
  __syncwarp();
  double* O = Uc + (int64_t)j * p * R;
  for (int e = lane; e < p * R; e += 32) {
    const int a = e / R, q = e - a * R;
    double v = 0.0;
#pragma unroll
    for (int b = 0; b < R; ++b) v = fma(Us[a * R + b], Gs[b * R + q], v);
    O[e] = v;
  }
  if (lane < R) {
    double v = 0.0;
#pragma unroll
    for (int b = 0; b < R; ++b) v = fma(cs[b], Gs[b * R + lane], v);
    const double t = tv[lane];
    tvec[(int64_t)j * R + lane] = t;
    contrib[(int64_t)j * R + lane] = (double)(d.m - c) * t - v;
  }
}

constexpr int FR_WARPS = 2;

template <int RM>
__global__ void __launch_bounds__(FR_WARPS * 32)
procrustes_fit_reg_kernel(const double* __restrict__ tgt, const int64_t* __restrict__ tgt_rows,
                          const double* __restrict__ src, const int64_t* __restrict__ src_rows,
                          const int64_t* __restrict__ job_off, int njobs, int r,
                          double* __restrict__ rot, double* __restrict__ trans,
                          double* __restrict__ loss, int32_t* __restrict__ degenerate, int redo) {
  extern __shared__ double sm[];
  const int P = (r + 1) >> 1;                  // lanes per fit
  const int FPW = 32 / P;                      // fits per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / P, l = lane - g * P;
  const int gbase = g * P;
  const int job = (blockIdx.x * FR_WARPS + warp) * FPW + g;
  // redo: only the fits the Newton-Schulz kernel handed over (degenerate == -1)
  const bool act = g < FPW && job < njobs && (!redo || degenerate[job] == -1);
  if (__ballot_sync(0xffffffffu, act) == 0u) return;
  // per-fit shared area: L, V (r x r, column-major), T (r x r, row-major), ms (r)
  double* Ls = sm + ((size_t)warp * FPW + (g < FPW ? g : 0)) * (3 * r * r + r);
  double* Vs = Ls + r * r;
  double* Ts = Vs + r * r;
  double* mss = Ts + r * r;

  int64_t o = 0;
  int K = 0;
  if (act) {
    o = job_off[job];
    K = (int)(job_off[job + 1] - o);
  }
  const int64_t* tr = tgt_rows + o;
  const int64_t* sr = src_rows + o;
  int ct = 2 * l, cb = 2 * l + 1;              // column indices held (>= r: zero dummy)
  // means: all r target columns, the two source columns this lane owns
  double mt[RM], bt[RM], bb[RM], vt[RM], vb[RM];
#pragma unroll
  for (int a = 0; a < RM; ++a) mt[a] = 0.0;
  double mst = 0.0, msb = 0.0;
#pragma unroll 4
  for (int t = 0; t < K; ++t) {
    const double* xr = tgt + tr[t] * r;
    const double* yr = src + sr[t] * r;
#pragma unroll
    for (int a = 0; a < RM; ++a)
      if (a < r) mt[a] += xr[a];
    if (ct < r) mst += yr[ct];
    if (cb < r) msb += yr[cb];
  }
  const double iK = K > 0 ? 1.0 / K : 0.0;
#pragma unroll
  for (int a = 0; a < RM; ++a) mt[a] *= iK;
  mst *= iK;
  msb *= iK;
  if (act) {
    if (ct < r) mss[ct] = mst;
    if (cb < r) mss[cb] = msb;
  }
  // B[:, c] = sum_t (x_t - mt)(y_t[c] - ms[c]); V = I
#pragma unroll
  for (int a = 0; a < RM; ++a) {
    bt[a] = 0.0;
    bb[a] = 0.0;
    vt[a] = (a == ct) ? 1.0 : 0.0;
    vb[a] = (a == cb) ? 1.0 : 0.0;
  }
#pragma unroll 4
  for (int t = 0; t < K; ++t) {
    const double* xr = tgt + tr[t] * r;
    const double* yr = src + sr[t] * r;
    const double yt = ct < r ? yr[ct] - mst : 0.0;
    const double yb = cb < r ? yr[cb] - msb : 0.0;
#pragma unroll
    for (int a = 0; a < RM; ++a) {
      const double x = a < r ? xr[a] - mt[a] : 0.0;
      bt[a] = fma(x, yt, bt[a]);
      bb[a] = fma(x, yb, bb[a]);
    }
  }
  // one-sided Jacobi sweeps, P disjoint pairs per round, tournament ordering
  const unsigned gmask = (P == 32 ? 0xffffffffu : ((1u << P) - 1u)) << gbase;
  const int src_top = l == 0 ? lane : lane - 1;           // top' source lane
  const int src_bot = l == P - 1 ? lane : (lane + 1) & 31;  // bot' source lane
  for (int sweep = 0; sweep < 60; ++sweep) {
    int nrot = 0;
    for (int round = 0; round < 2 * P - 1; ++round) {
      double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
      for (int a = 0; a < RM; ++a) {
        al = fma(bt[a], bt[a], al);
        be = fma(bb[a], bb[a], be);
        ga = fma(bt[a], bb[a], ga);
      }
      if (ga != 0.0 && ga * ga > 1e-30 * (al * be)) {
        const double h = 0.5 * (be - al);
        const double t = ga / (h + copysign(sqrt(fma(h, h, ga * ga)), h == 0.0 ? 1.0 : h));
        const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
#pragma unroll
        for (int a = 0; a < RM; ++a) {
          const double x = bt[a], y = bb[a];
          bt[a] = c * x - s * y;
          bb[a] = s * x + c * y;
          const double vx = vt[a], vy = vb[a];
          vt[a] = c * vx - s * vy;
          vb[a] = s * vx + c * vy;
        }
        ++nrot;
      }
      if (P > 1) {
        // top'_0 = top_0, top'_1 = bot_0, top'_l = top_{l-1};  bot'_l = bot_{l+1},
        // bot'_{P-1} = top_{P-1}.  The SENDER picks the value: on the top channel
        // lane 0 sends its bottom column, every other lane its top column.
#pragma unroll
        for (int a = 0; a < RM; ++a) {
          const double ntb = __shfl_sync(0xffffffffu, l == 0 ? bb[a] : bt[a], src_top);
          const double ntv = __shfl_sync(0xffffffffu, l == 0 ? vb[a] : vt[a], src_top);
          const double nbb = __shfl_sync(0xffffffffu, bb[a], src_bot);
          const double nbv = __shfl_sync(0xffffffffu, vb[a], src_bot);
          if (l == P - 1) { bb[a] = bt[a]; vb[a] = vt[a]; }
          else { bb[a] = nbb; vb[a] = nbv; }
          if (l != 0) { bt[a] = ntb; vt[a] = ntv; }
        }
        const int nct = __shfl_sync(0xffffffffu, l == 0 ? cb : ct, src_top);
        const int ncb = __shfl_sync(0xffffffffu, cb, src_bot);
        if (l == P - 1) cb = ct;
        else cb = ncb;
        if (l != 0) ct = nct;
      }
    }
    const unsigned any = __ballot_sync(0xffffffffu, act && nrot > 0);
    if (any == 0u) break;
  }
  // singular values, extreme ones over the group, normalised left vectors
  double st2 = 0.0, sb2 = 0.0;
#pragma unroll
  for (int a = 0; a < RM; ++a) {
    st2 = fma(bt[a], bt[a], st2);
    sb2 = fma(bb[a], bb[a], sb2);
  }
  const double sgt = sqrt(st2), sgb = sqrt(sb2);
  double smax = fmax(ct < r ? sgt : 0.0, cb < r ? sgb : 0.0);
  double smin = fmin(ct < r ? sgt : 1e308, cb < r ? sgb : 1e308);
  for (int q = 0; q < P; ++q) {
    const double a1 = __shfl_sync(0xffffffffu, smax, gbase + q);
    const double a2 = __shfl_sync(0xffffffffu, smin, gbase + q);
    if (q != l) { smax = fmax(smax, a1); smin = fmin(smin, a2); }
  }
  const bool okt = sgt > 1e-15 * smax && sgt > 0.0, okb = sgb > 1e-15 * smax && sgb > 0.0;
  if (act) {
#pragma unroll
    for (int a = 0; a < RM; ++a) {
      if (a < r && ct < r) {
        Ls[ct * r + a] = okt ? bt[a] / sgt : 0.0;
        Vs[ct * r + a] = vt[a];
      }
      if (a < r && cb < r) {
        Ls[cb * r + a] = okb ? bb[a] / sgb : 0.0;
        Vs[cb * r + a] = vb[a];
      }
    }
  }
  // rank-deficient left bases: complete by Gram-Schmidt on e_q (group lane 0,
  // columns in index order as procrustes_fit_kernel)
  const bool bad = act && ((ct < r && !okt) || (cb < r && !okb));
  const unsigned badm = __ballot_sync(0xffffffffu, bad) & gmask;
  __syncwarp();

  if (badm != 0u && l == 0) {
    bool good[RM];
#pragma unroll
    for (int i = 0; i < RM; ++i) {
      double s2 = 0.0;
      if (i < r)
        for (int a = 0; a < r; ++a) s2 = fma(Ls[i * r + a], Ls[i * r + a], s2);
      good[i] = s2 > 0.5;                       // normalised columns have norm 1, the rest 0
    }
    for (int i = 0; i < r; ++i) {
      if (good[i]) continue;
      // e_q minus its projection on the basis so far, for the q that leaves the
      // largest remainder (>= 1/sqrt(r): a fixed acceptance threshold can fail
      // for every q once r > 4)
      int qb = 0;
      double nb = -1.0;
      for (int q = 0; q < r; ++q) {
        double n2 = 1.0;
        for (int c = 0; c < r; ++c) {
          if (c == i || (!good[c] && c > i)) continue;
          const double d = Ls[c * r + q];
          n2 -= d * d;
        }
        if (n2 > nb) { nb = n2; qb = q; }
      }
      double v[RM];
#pragma unroll
      for (int a = 0; a < RM; ++a) v[a] = (a == qb) ? 1.0 : 0.0;
      for (int pass = 0; pass < 2; ++pass)         // twice: orthogonal to working precision
        for (int c = 0; c < r; ++c) {
          if (c == i || (!good[c] && c > i)) continue;
          double dot = 0.0;
#pragma unroll
          for (int a = 0; a < RM; ++a)
            if (a < r) dot = fma(Ls[c * r + a], v[a], dot);
#pragma unroll
          for (int a = 0; a < RM; ++a)
            if (a < r) v[a] -= dot * Ls[c * r + a];
        }
      double nv = 0.0;
#pragma unroll
      for (int a = 0; a < RM; ++a)
        if (a < r) nv = fma(v[a], v[a], nv);
      nv = sqrt(nv);
#pragma unroll
      for (int a = 0; a < RM; ++a)
        if (a < r) Ls[i * r + a] = v[a] / nv;
      good[i] = true;
    }
  }
  __syncwarp();
  // T = V L^T (rows a = 2l, 2l+1 on lane l), t = mt - ms T, loss
  double* T = rot + (size_t)job * r * r;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int a = 2 * l + h;
    if (act && a < r)
      for (int b = 0; b < r; ++b) {
        double s = 0.0;
        for (int i = 0; i < r; ++i) s = fma(Vs[i * r + a], Ls[i * r + b], s);
        Ts[a * r + b] = s;
        T[a * r + b] = s;
      }
  }
  __syncwarp();
  // translation: lane l owns entries b = 2l, 2l+1 of t (written to Vs[0..r), free now)
  double* tv = trans + (size_t)job * r;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int b = 2 * l + h;
    if (act && b < r) {
      double s = 0.0;
      for (int a = 0; a < r; ++a) s = fma(mss[a], Ts[a * r + b], s);
      double mtb = 0.0;
#pragma unroll
      for (int a = 0; a < RM; ++a)
        if (a == b) mtb = mt[a];
      tv[b] = mtb - s;
      Ls[b] = mtb - s;
    }
  }
  __syncwarp();
  // loss: lane l takes rows t = l, l+P, ...
  double ls = 0.0;
  if (act)
#pragma unroll 2
    for (int t = l; t < K; t += P) {
      const double* xr = tgt + tr[t] * r;
      const double* yr = src + sr[t] * r;
      double y[RM];
#pragma unroll
      for (int a = 0; a < RM; ++a) y[a] = a < r ? yr[a] : 0.0;
      for (int b = 0; b < r; ++b) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < RM; ++a)
          if (a < r) s = fma(y[a], Ts[a * r + b], s);
        const double e = xr[b] - s - Ls[b];
        ls = fma(e, e, ls);
      }
    }
  for (int q = 1; q < P; ++q) {
    const double v = __shfl_sync(0xffffffffu, ls, gbase + q);
    if (l == 0) ls += v;
  }
  if (act && l == 0) {
    loss[job] = ls;
    degenerate[job] = (r == 0 || smin <= 1e-12 * smax) ? 1 : 0;
  }
}

// X[start_j + i] <- X[start_j + i] T_j + t_j for the rows of job j (in place);
// grid (row chunks of AP_ROWS, jobs).  The chunk is contiguous (rows x r
// doubles): it is staged through shared memory with coalesced 16-byte loads,
// and every thread then produces flat output elements (row, column) that are
// stored coalesced -- a thread-per-row walk over 80-byte rows would touch ~20
// L1 lines per warp instruction.
template <int RM>
__host__ __device__ constexpr int ap_rows() { return RM <= 16 ? 256 : 128; }

template <int RM>
__global__ void __launch_bounds__(256)
apply_kernel(double* __restrict__ buf, int r, const int64_t* __restrict__ start,
             const int64_t* __restrict__ len, const double* __restrict__ rot,
             const double* __restrict__ trans) {
  __shared__ double Ts[RM * RM], ts[RM];
  constexpr int AP_ROWS = ap_rows<RM>();
  __shared__ __align__(16) double xs[AP_ROWS * RM];
  const int job = blockIdx.y;
  const int64_t n = len[job];
  const int64_t i0 = (int64_t)blockIdx.x * AP_ROWS;
  if (i0 >= n) return;
  const int rows = (int)min((int64_t)AP_ROWS, n - i0);
  for (int e = threadIdx.x; e < RM * RM; e += blockDim.x) {
    const int a = e / RM, b = e % RM;
    Ts[e] = (a < r && b < r) ? rot[(size_t)job * r * r + a * r + b] : 0.0;
  }
  if (threadIdx.x < RM) ts[threadIdx.x] = threadIdx.x < r ? trans[(size_t)job * r + threadIdx.x] : 0.0;
  double* base = buf + (start[job] + i0) * r;
  const int ne = rows * r;
  if ((reinterpret_cast<uintptr_t>(base) & 15) == 0) {
    const double2* b2 = reinterpret_cast<const double2*>(base);
    for (int e = threadIdx.x; e < ne / 2; e += blockDim.x) reinterpret_cast<double2*>(xs)[e] = b2[e];
    if ((ne & 1) && threadIdx.x == 0) xs[ne - 1] = base[ne - 1];
  } else {
    for (int e = threadIdx.x; e < ne; e += blockDim.x) xs[e] = base[e];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    const int row = e / r, b = e - row * r;
    const double* xr = xs + row * r;
    double s2 = 0.0;
    for (int a = 0; a < r; ++a) s2 = fma(xr[a], Ts[a * RM + b], s2);
    base[e] = s2 + ts[b];
  }
}

// D&C stitch (algorithms.py:151-156): piece 0 verbatim, piece j>0 rows c..
// through fit j-1, scattered to original rows, minus the final column mean
// (algorithms.py:122-125) when `mean` is given.  One CTA per piece: T, t and
// the mean in shared memory; the piece's rows (contiguous in P) are staged in
// ST_ROWS-row chunks with coalesced loads, then every thread produces flat
// (row, column) elements, so a warp store covers ~3 output rows' contiguous
// 80-byte segments instead of 32 scattered rows.
constexpr int ST_ROWS = 256;
constexpr int ST_CR = 1024;       // rows per CTA of the stitch (multiple of ST_ROWS)
constexpr int OS_CR = 2048;       // rows per CTA of the per-job sums

template <int RM>
__global__ void __launch_bounds__(256)
dc_stitch_kernel(const double* __restrict__ P, const int64_t* __restrict__ row_idx,
                 const int64_t* __restrict__ off, int c, int r, const double* __restrict__ rot,
                 const double* __restrict__ trans, const double* __restrict__ mean,
                 double* __restrict__ out, int first_identity) {
  constexpr int SR = RM <= 16 ? ST_ROWS : ST_ROWS / 2;
  __shared__ double Ts[RM * RM], ts[RM], ms[RM];
  __shared__ double xs[SR * RM];
  __shared__ int64_t dsts[SR];
  // D&C (first_identity): piece 0 verbatim, fit j-1 for piece j, own rows from c;
  // fast MDS finish: fit j for job j, all rows
  const int j = blockIdx.y;
  const bool ident = first_identity && j == 0;
  const int fj = first_identity ? j - 1 : j;
  const int64_t o = off[j], m = off[j + 1] - o;
  for (int e = threadIdx.x; e < RM * RM; e += blockDim.x) {
    const int a = e / RM, b = e % RM;
    Ts[e] = (a < r && b < r) ? (ident ? (a == b ? 1.0 : 0.0) : rot[(size_t)fj * r * r + a * r + b])
                             : 0.0;
  }
  if (threadIdx.x < RM) {
    const int b = threadIdx.x;
    ts[b] = (ident || b >= r) ? 0.0 : trans[(size_t)fj * r + b];
    ms[b] = (mean && b < r) ? mean[b] : 0.0;
  }
  const int64_t first = (ident || !first_identity) ? 0 : c;
  // blockIdx.x: this CTA's range of ST_CR rows of the job (long jobs over many CTAs)
  const int64_t lo = first + (int64_t)blockIdx.x * ST_CR, hi = min(m, lo + ST_CR);
  for (int64_t i0 = lo; i0 < hi; i0 += SR) {
    const int rows = (int)min((int64_t)SR, hi - i0);
    __syncthreads();                                  // previous chunk consumed
    const double* src = P + (o + i0) * r;
    for (int e = threadIdx.x; e < rows * r; e += blockDim.x) xs[e] = src[e];
    for (int q = threadIdx.x; q < rows; q += blockDim.x) dsts[q] = row_idx[o + i0 + q] * r;
    __syncthreads();
    for (int e = threadIdx.x; e < rows * r; e += blockDim.x) {
      const int row = e / r, b = e - row * r;
      const double* xr = xs + row * r;
      double v;
      if (ident) {
        v = xr[b];
      } else {
        double s2 = 0.0;
        for (int a2 = 0; a2 < r; ++a2) s2 = fma(xr[a2], Ts[a2 * RM + b], s2);
        v = s2 + ts[b];
      }
      out[dsts[row] + b] = v - ms[b];
    }
  }
}

// Column sums of each piece's OWN rows of the piece points P (piece 0: all
// rows, piece j > 0: rows c..), pushed through the piece's fit; coalesced:
// thread (g, col) of RG = 256 / r row groups walks rows g, g + RG, ...
template <int RM>
__global__ void __launch_bounds__(256)
dc_own_sums_kernel(const double* __restrict__ P, const int64_t* __restrict__ off, int c, int r,
                   const double* __restrict__ rot, const double* __restrict__ trans,
                   double* __restrict__ sums, int first_identity) {
  __shared__ double red[256];
  __shared__ double colsum[RM];
  const int j = blockIdx.y;
  const int64_t o = off[j], m = off[j + 1] - o;
  const int RG = 256 / r;
  const int g = threadIdx.x / r, col = threadIdx.x - g * r;
  double acc = 0.0;
  const bool ident = first_identity && j == 0;
  const int fj = first_identity ? j - 1 : j;
  const int64_t first = (ident || !first_identity) ? 0 : c;
  // blockIdx.x: this CTA's range of OS_CR rows of the job
  const int64_t lo = min(m, first + (int64_t)blockIdx.x * OS_CR), hi = min(m, lo + OS_CR);
  if (g < RG) {
    double a4[4] = {0.0, 0.0, 0.0, 0.0};          // four loads in flight, fixed combine order
    int64_t i = lo + g;
    for (; i + 3 * RG < hi; i += 4 * RG) {
#pragma unroll
      for (int u = 0; u < 4; ++u) a4[u] += P[(o + i + u * RG) * r + col];
    }
    for (; i < hi; i += RG) a4[0] += P[(o + i) * r + col];
    acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
  }
  red[threadIdx.x] = g < RG ? acc : 0.0;
  __syncthreads();
  if (threadIdx.x < r) {
    double v = 0.0;
    for (int gg = 0; gg < RG; ++gg) v += red[gg * r + threadIdx.x];   // fixed order
    colsum[threadIdx.x] = v;
  }
  __syncthreads();
  // contribution of the piece to the stitched column sums: S (piece 0) or
  // S T_{j-1} + n_j t_{j-1}
  if (threadIdx.x < r) {
    const int b = threadIdx.x;
    double v;
    if (ident) {
      v = colsum[b];
    } else {
      const double* T = rot + (size_t)fj * r * r;
      v = (double)(hi - lo) * trans[(size_t)fj * r + b];
      for (int a2 = 0; a2 < r; ++a2) v = fma(colsum[a2], T[a2 * r + b], v);
    }
    sums[((size_t)j * gridDim.x + blockIdx.x) * r + b] = v;
  }
}

// Final column mean of the stitched configuration from the per-piece
// contributions (dc_own_sums_kernel): thread t adds pieces t, t+256, ... in
// order (independent loads, unrolled), then a fixed tree.
template <int RM>
__global__ void __launch_bounds__(256)
dc_mean_kernel(const double* __restrict__ sums, int npieces, int r, int64_t n,
               double* __restrict__ mean) {
  __shared__ double red[256];
  double acc[RM];
#pragma unroll
  for (int b = 0; b < RM; ++b) acc[b] = 0.0;
#pragma unroll 4
  for (int j = threadIdx.x; j < npieces; j += 256) {
    const double* S = sums + (size_t)j * r;
#pragma unroll
    for (int b = 0; b < RM; ++b)
      if (b < r) acc[b] += S[b];
  }
#pragma unroll
  for (int b = 0; b < RM; ++b) {
    if (b >= r) break;
    red[threadIdx.x] = acc[b];
    __syncthreads();
    for (int s2 = 128; s2 > 0; s2 >>= 1) {
      if (threadIdx.x < s2) red[threadIdx.x] += red[threadIdx.x + s2];
      __syncthreads();
    }
    if (threadIdx.x == 0) mean[b] = red[0] / (double)n;
    __syncthreads();
  }
}

__global__ void scatter_kernel(const double* __restrict__ src, const int64_t* __restrict__ idx,
                               int64_t n, int r, double* __restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * r) return;
  const int64_t i = e / r;
  const int b = (int)(e - i * r);
  out[idx[i] * r + b] = src[e];
}

constexpr int RC_BLOCKS = 296;

// deterministic column sums: block b owns a fixed contiguous row range
template <int RM>
__global__ void __launch_bounds__(256)
colsum_partial_kernel(const double* __restrict__ X, int64_t n, int r, double* __restrict__ part) {
  __shared__ double red[256];
  const int64_t lo = n * blockIdx.x / gridDim.x, hi = n * (blockIdx.x + 1) / gridDim.x;
  double acc[RM];
#pragma unroll
  for (int c = 0; c < RM; ++c) acc[c] = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += 256)
#pragma unroll
    for (int c = 0; c < RM; ++c)
      if (c < r) acc[c] += X[i * r + c];
  for (int c = 0; c < r; ++c) {
    red[threadIdx.x] = acc[c];
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) part[(int64_t)blockIdx.x * r + c] = red[0];
    __syncthreads();
  }
}

// X -= (sum_b part[b] + corr) / n, elementwise over the n x r block; four
// independent loads in flight per thread, the column tracked incrementally
// (no 64-bit modulo per element).
__global__ void __launch_bounds__(256)
subtract_mean_kernel(double* __restrict__ X, int64_t n, int r, const double* __restrict__ part,
                     int nparts, const double* __restrict__ corr, double ndiv) {
  __shared__ double mean[MDSX_MAX_R];
  if (threadIdx.x < r) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += part[(int64_t)b * r + threadIdx.x];
    if (corr) s += corr[threadIdx.x];
    mean[threadIdx.x] = s / ndiv;
  }
  __syncthreads();
  const int64_t total = n * r;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int cs = (int)(stride % r);
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int c = (int)(e % r);
  auto adv = [&](int c0) { c0 += cs; return c0 >= r ? c0 - r : c0; };
  for (; e + 3 * stride < total; e += 4 * stride) {
    const int c1 = adv(c), c2 = adv(c1), c3 = adv(c2);
    const double x0 = X[e], x1 = X[e + stride], x2 = X[e + 2 * stride], x3 = X[e + 3 * stride];
    X[e] = x0 - mean[c];
    X[e + stride] = x1 - mean[c1];
    X[e + 2 * stride] = x2 - mean[c2];
    X[e + 3 * stride] = x3 - mean[c3];
    c = adv(c3);
  }
  for (; e < total; e += stride) {
    X[e] -= mean[c];
    c = adv(c);
  }
}

// per-segment column sums over listed rows (segment j = rows idx[off_j .. off_j+1)),
// one warp per (segment, column), fixed order -> deterministic, world-size independent
__global__ void seg_colsum_kernel(const double* __restrict__ X, const int64_t* __restrict__ idx,
                                  const int64_t* __restrict__ off, int nseg, int r,
                                  double* __restrict__ sums) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nseg * r) return;
  const int seg = warp / r, c = warp % r;
  double s = 0.0;
  for (int64_t i = off[seg] + lane; i < off[seg + 1]; i += 32) s += X[(idx ? idx[i] : i) * r + c];
  s = mdsx::warp_sum(s);
  if (lane == 0) sums[(int64_t)seg * r + c] = s;
}

// Contiguous segments (no row index): one CTA per segment streams the
// segment's r * len doubles coalesced; the stride S = r * floor(T / r) keeps
// thread t on column t % r, so each thread accumulates one column and the
// per-column partials are folded in fixed thread order (deterministic).
constexpr int SR_T = 500;
__global__ void __launch_bounds__(SR_T)
seg_colsum_rows_kernel(const double* __restrict__ X, const int64_t* __restrict__ off, int r,
                       double* __restrict__ sums) {
  __shared__ double red[SR_T];
  const int t = threadIdx.x;
  const int S = r * (SR_T / r);
  const int64_t a = off[blockIdx.x] * r, b = off[blockIdx.x + 1] * r;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  if (t < S) {
    int64_t e = a + t;
    for (; e + 3 * S < b; e += 4 * S) {
      s0 += X[e];
      s1 += X[e + S];
      s2 += X[e + 2 * S];
      s3 += X[e + 3 * S];
    }
    for (; e < b; e += S) s0 += X[e];
  }
  red[t] = t < S ? (s0 + s1) + (s2 + s3) : 0.0;
  __syncthreads();
  if (t < r) {
    double tot = 0.0;
    for (int u = t; u < S; u += r) tot += red[u];
    sums[(int64_t)blockIdx.x * r + t] = tot;
  }
}

// X[0..n) rows -= shift: grid-stride over the n * r doubles with a stride that
// is a multiple of r (each thread keeps one column's shift in a register)
__global__ void __launch_bounds__(SR_T)
shift_all_kernel(double* __restrict__ X, int64_t total, int r, const double* __restrict__ shift) {
  const int t = threadIdx.x;
  const int S = r * (SR_T / r);
  if (t >= S) return;
  const double sh = shift[t % r];
  const int64_t step = (int64_t)gridDim.x * S;
  for (int64_t e = (int64_t)blockIdx.x * S + t; e < total; e += step) X[e] -= sh;
}

__global__ void shift_rows_kernel(double* __restrict__ X, const int64_t* __restrict__ idx, int64_t n,
                                  int r, const double* __restrict__ shift) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * r) return;
  const int64_t i = e / r;
  const int c = (int)(e - i * r);
  X[(idx ? idx[i] : i) * r + c] -= shift[c];
}

// ---- harness metric (simulation.py:83-108): aligned_correlations on the device.
// U = [X | D] (n x 2r: the configuration and the dominant columns).  Pass 1:
// each CTA owns a contiguous row range, stages rows shifted by row 0 into a
// shared tile and accumulates the shifted column sums and the upper triangle
// of U'U (one value per thread slot, fixed order); pass 2 (one CTA): the
// partials reduced in block order, centred (P - s s^T / n), the Procrustes
// rotation of the dominant onto X from the cross-product D~'X~ (the warp SVD
// above), then per column corr_j = (X~T)_j . D~_j / (|X~T_j| |D~_j|), all from
// the 2r x 2r Gram: the n x r aligned matrix is never formed.
constexpr int AC_T = 256;
constexpr int AC_TILE = 64;

template <typename T>
__global__ void __launch_bounds__(AC_T)
corr_partial_kernel(const double* __restrict__ X, int64_t n, int r, const T* __restrict__ Dm,
                    int64_t ld, double* __restrict__ part, int nq) {
  __shared__ double tile[AC_TILE * 32];
  __shared__ double u0[32];
  __shared__ unsigned char pa[560], pb[560];
  const int w = 2 * r, tid = threadIdx.x;
  if (tid < w) u0[tid] = tid < r ? X[tid] : (double)Dm[tid - r];
  if (tid == 0) {
    int q = w;
    for (int a = 0; a < w; ++a)
      for (int b = a; b < w; ++b) { pa[q] = (unsigned char)a; pb[q] = (unsigned char)b; ++q; }
  }
  __syncthreads();
  const int64_t r0 = n * blockIdx.x / gridDim.x, r1 = n * (blockIdx.x + 1) / gridDim.x;
  double acc[3] = {0.0, 0.0, 0.0};
  for (int64_t t0 = r0; t0 < r1; t0 += AC_TILE) {
    const int rows = (int)(r1 - t0 < AC_TILE ? r1 - t0 : AC_TILE);
    for (int e = tid; e < rows * w; e += AC_T) {
      const int i = e / w, c = e - i * w;
      const int64_t row = t0 + i;
      const double v = c < r ? X[row * r + c] : (double)Dm[row * ld + (c - r)];
      tile[i * w + c] = v - u0[c];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int q = tid + k * AC_T;
      if (q < nq) {
        double s = 0.0;
        if (q < w) {
          for (int i = 0; i < rows; ++i) s += tile[i * w + q];
        } else {
          const int a = pa[q], b = pb[q];
          for (int i = 0; i < rows; ++i) s = fma(tile[i * w + a], tile[i * w + b], s);
        }
        acc[k] += s;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const int q = tid + k * AC_T;
    if (q < nq) part[(size_t)blockIdx.x * nq + q] = acc[k];
  }
}

__global__ void __launch_bounds__(AC_T)
corr_finish_kernel(const double* __restrict__ part, int nparts, int nq, int64_t n, int r,
                   double* __restrict__ corr, double* __restrict__ rot_out,
                   int32_t* __restrict__ zero_var) {
  __shared__ double val[560];
  __shared__ double C[32 * 32];
  __shared__ double B[16 * 16], V[16 * 16], Tm[16 * 16], sg[16];
  const int w = 2 * r, tid = threadIdx.x;
  for (int q = tid; q < nq; q += AC_T) {
    double s = 0.0;
    for (int g = 0; g < nparts; ++g) s += part[(size_t)g * nq + q];   // fixed order
    val[q] = s;
  }
  __syncthreads();
  if (tid == 0) {                                  // centred Gram C = P - s s^T / n
    const double dn = (double)n;
    int q = w;
    for (int a = 0; a < w; ++a)
      for (int b = a; b < w; ++b, ++q) {
        const double c = val[q] - val[a] * val[b] / dn;
        C[a * w + b] = c;
        C[b * w + a] = c;
      }
  }
  __syncthreads();
  if (tid < 32) {
    const int lane = tid;
    for (int e = lane; e < r * r; e += 32) {       // B = D~' X~ (target = dominant, source = X)
      const int a = e / r, b = e % r;
      B[e] = C[(r + a) * w + b];
      V[e] = a == b ? 1.0 : 0.0;
    }
    __syncwarp();
    double smin, smax;
    rotation_from_cross(B, V, sg, r, lane, Tm, smin, smax);
    __syncwarp();
    int zero = 0;
    if (lane < r) {
      const int j = lane;
      double num = 0.0, da = 0.0;
      for (int a = 0; a < r; ++a) {
        num = fma(Tm[a * r + j], C[a * w + (r + j)], num);
        double t = 0.0;
        for (int b = 0; b < r; ++b) t = fma(C[a * w + b], Tm[b * r + j], t);
        da = fma(Tm[a * r + j], t, da);
      }
      const double dd = C[(r + j) * w + (r + j)];
      zero = !(da > 0.0) || !(dd > 0.0);
      corr[j] = zero ? 0.0 : num / (sqrt(da) * sqrt(dd));
    }
    zero = __any_sync(0xffffffffu, zero);
    if (lane == 0) *zero_var = zero;
    if (rot_out)
      for (int e = lane; e < r * r; e += 32) rot_out[e] = Tm[e];
  }
}

}  // namespace

namespace mdsx {

int launch_seg_colsum(mdsx_handle* h, const double* X, const int64_t* idx, const int64_t* off,
                      int nseg, int r, double* sums, cudaStream_t st) {
  if (nseg == 0) return MDSX_OK;
  if (!idx && r <= 32) {
    mdsx::pre(h, st);
    seg_colsum_rows_kernel<<<nseg, SR_T, 0, st>>>(X, off, r, sums);
    return launched(h, "seg_colsum_kernel", st);
  }
  const int64_t threads = (int64_t)nseg * r * 32;
  mdsx::pre(h, st);
  seg_colsum_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(X, idx, off, nseg, r, sums);
  return launched(h, "seg_colsum_kernel", st);
}

int launch_shift_rows(mdsx_handle* h, double* X, const int64_t* idx, int64_t n, int r,
                      const double* shift, cudaStream_t st) {
  if (n == 0) return MDSX_OK;
  if (!idx && r <= 32) {
    const int64_t total = n * r;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>((total + 4 * SR_T - 1) / (4 * SR_T),
                                                                  (int64_t)h->num_sms * 4));
    mdsx::pre(h, st);
    shift_all_kernel<<<blocks, SR_T, 0, st>>>(X, total, r, shift);
    return launched(h, "shift_rows_kernel", st);
  }
  mdsx::pre(h, st);
  shift_rows_kernel<<<(unsigned)((n * r + 255) / 256), 256, 0, st>>>(X, idx, n, r, shift);
  return launched(h, "shift_rows_kernel", st);
}


// D&C tail of subsets 1 .. npieces-1 (dc_fit_kernel); r <= 16, c <= NS_KMAX.
bool dc_fit_ok(int r, int c, int p) {
  const size_t sm = ((size_t)NS_WARPS * (2 * NS_KMAX * r + 2 * r * r + 4 * r) + (size_t)c * p +
                     (size_t)NS_WARPS * ((size_t)p * r + p)) * sizeof(double);
  return r >= 1 && r <= 16 && c >= 1 && c <= NS_KMAX && sm <= 200 * 1024;
}

int launch_dc_fit(mdsx_handle* h, const void* data, int dtype, int64_t ld, int p,
                  const int64_t* row_idx, const PieceDesc* pd, int npieces, int r, int c,
                  const double* mu, const double* U, double* Pc, double* rot, double* trans,
                  double* loss, int32_t* degen, double* Uc, double* tvec, double* contrib,
                  int32_t* pending, cudaStream_t st) {
  if (npieces <= 1) return MDSX_OK;
  auto go = [&](auto rc_) -> int {
    constexpr int R = decltype(rc_)::value;
    const size_t sm = ((size_t)NS_WARPS * (2 * NS_KMAX * R + 2 * R * R + 4 * R) + (size_t)c * p +
                       (size_t)NS_WARPS * ((size_t)p * R + p)) * sizeof(double);
    const int blocks = (npieces - 1 + NS_WARPS - 1) / NS_WARPS;
    mdsx::pre(h, st);
    if (dtype == MDSX_F32) {
      auto kern = dc_fit_kernel<R, float>;
      if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<blocks, NS_WARPS * 32, sm, st>>>((const float*)data, ld, p, row_idx, pd, npieces, c, mu, U,
                                              Pc, rot, trans, loss, degen, Uc, tvec, contrib, pending);
    } else {
      auto kern = dc_fit_kernel<R, double>;
      if (sm > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<blocks, NS_WARPS * 32, sm, st>>>((const double*)data, ld, p, row_idx, pd, npieces, c, mu,
                                               U, Pc, rot, trans, loss, degen, Uc, tvec, contrib, pending);
    }
    return launched(h, "dc_fit_kernel", st);
  };
  switch (r) {
    case 1: return go(std::integral_constant<int, 1>{});
    case 2: return go(std::integral_constant<int, 2>{});
    case 3: return go(std::integral_constant<int, 3>{});
    case 4: return go(std::integral_constant<int, 4>{});
    case 5: return go(std::integral_constant<int, 5>{});
    case 6: return go(std::integral_constant<int, 6>{});
    case 7: return go(std::integral_constant<int, 7>{});
    case 8: return go(std::integral_constant<int, 8>{});
    case 9: return go(std::integral_constant<int, 9>{});
    case 10: return go(std::integral_constant<int, 10>{});
    case 11: return go(std::integral_constant<int, 11>{});
    case 12: return go(std::integral_constant<int, 12>{});
    case 13: return go(std::integral_constant<int, 13>{});
    case 14: return go(std::integral_constant<int, 14>{});
    case 15: return go(std::integral_constant<int, 15>{});
    default: return go(std::integral_constant<int, 16>{});
  }
}

int launch_procrustes_fit(mdsx_handle* h, const double* tgt, const int64_t* tgt_rows,
                          const double* src, const int64_t* src_rows, const int64_t* job_off_dev,
                          int njobs, int r, double* rot, double* trans, double* loss,
                          int32_t* degenerate, cudaStream_t st, bool redo_only) {
  if (njobs == 0) return MDSX_OK;
  if (r <= 16 && !getenv("MDSX_FIT_WARP")) {
    if (!redo_only) {                            // Newton-Schulz fast path first
      auto ns = [&](auto rc_) -> int {
        constexpr int R = decltype(rc_)::value;
        auto kern = procrustes_fit_ns_kernel<R>;
        const size_t sm1 = (size_t)NS_WARPS * (2 * NS_KMAX * R + 2 * R * R + 3 * R) * sizeof(double);
        if (sm1 > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
        mdsx::pre(h, st);
        kern<<<(njobs + NS_WARPS - 1) / NS_WARPS, NS_WARPS * 32, sm1, st>>>(
            tgt, tgt_rows, src, src_rows, job_off_dev, njobs, rot, trans, loss, degenerate);
        return launched(h, "procrustes_ns_kernel", st);
      };
      int rc = MDSX_OK;
      switch (r) {
        case 1: rc = ns(std::integral_constant<int, 1>{}); break;
        case 2: rc = ns(std::integral_constant<int, 2>{}); break;
        case 3: rc = ns(std::integral_constant<int, 3>{}); break;
        case 4: rc = ns(std::integral_constant<int, 4>{}); break;
        case 5: rc = ns(std::integral_constant<int, 5>{}); break;
        case 6: rc = ns(std::integral_constant<int, 6>{}); break;
        case 7: rc = ns(std::integral_constant<int, 7>{}); break;
        case 8: rc = ns(std::integral_constant<int, 8>{}); break;
        case 9: rc = ns(std::integral_constant<int, 9>{}); break;
        case 10: rc = ns(std::integral_constant<int, 10>{}); break;
        case 11: rc = ns(std::integral_constant<int, 11>{}); break;
        case 12: rc = ns(std::integral_constant<int, 12>{}); break;
        case 13: rc = ns(std::integral_constant<int, 13>{}); break;
        case 14: rc = ns(std::integral_constant<int, 14>{}); break;
        case 15: rc = ns(std::integral_constant<int, 15>{}); break;
        default: rc = ns(std::integral_constant<int, 16>{}); break;
      }
      if (rc) return rc;
    }
    const int P = (r + 1) / 2, fpw = 32 / P;
    const size_t sm2 = (size_t)FR_WARPS * fpw * (3 * r * r + r) * sizeof(double);
    const int blocks = (int)((njobs + (int64_t)FR_WARPS * fpw - 1) / ((int64_t)FR_WARPS * fpw));
    auto go = [&](auto rm) {
      constexpr int RMc = decltype(rm)::value;
      auto kern = procrustes_fit_reg_kernel<RMc>;
      if (sm2 > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
      mdsx::pre(h, st);
      kern<<<blocks, FR_WARPS * 32, sm2, st>>>(tgt, tgt_rows, src, src_rows, job_off_dev, njobs, r,
                                                rot, trans, loss, degenerate, 1);
      return launched(h, "procrustes_fit_kernel", st);
    };
    if (r <= 4) return go(std::integral_constant<int, 4>{});
    if (r <= 8) return go(std::integral_constant<int, 8>{});
    if (r <= 10) return go(std::integral_constant<int, 10>{});
    if (r <= 12) return go(std::integral_constant<int, 12>{});
    return go(std::integral_constant<int, 16>{});
  }
  const size_t smem = (size_t)FIT_WARPS * (2 * r * r + 3 * r) * sizeof(double);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(procrustes_fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
  const int blocks = (njobs + FIT_WARPS - 1) / FIT_WARPS;
  mdsx::pre(h, st);
  procrustes_fit_kernel<<<blocks, FIT_WARPS * 32, smem, st>>>(tgt, tgt_rows, src, src_rows,
                                                               job_off_dev, njobs, r, rot, trans,
                                                               loss, degenerate);
  return launched(h, "procrustes_fit_kernel", st);
}

int launch_apply(mdsx_handle* h, double* buf, int r, const int64_t* start, const int64_t* len,
                 int njobs, int64_t max_len, const double* rot, const double* trans,
                 cudaStream_t st) {
  if (njobs == 0 || max_len == 0) return MDSX_OK;
  auto go = [&](auto rm) {
    constexpr int RM = decltype(rm)::value;
    dim3 grid((unsigned)((max_len + ap_rows<RM>() - 1) / ap_rows<RM>()), (unsigned)njobs);
    mdsx::pre(h, st);
    apply_kernel<RM><<<grid, 256, 0, st>>>(buf, r, start, len, rot, trans);
  };
  if (r <= 4) go(std::integral_constant<int, 4>{});
  else if (r <= 8) go(std::integral_constant<int, 8>{});
  else if (r <= 10) go(std::integral_constant<int, 10>{});
  else if (r <= 16) go(std::integral_constant<int, 16>{});
  else go(std::integral_constant<int, 32>{});
  return launched(h, "apply_kernel", st);
}

int launch_dc_stitch(mdsx_handle* h, const double* P, const int64_t* row_idx, const int64_t* off,
                     int npieces, int64_t max_m, int c, int r, const double* rot,
                     const double* trans, double* out, cudaStream_t st, int64_t n_recenter,
                     double* ws, int first_identity) {
  const unsigned nch_s = (unsigned)std::max<int64_t>(1, (max_m + OS_CR - 1) / OS_CR);
  const unsigned nch_t = (unsigned)std::max<int64_t>(1, (max_m + ST_CR - 1) / ST_CR);
  auto go = [&](auto rm) {
    constexpr int RM = decltype(rm)::value;
    const double* mean = nullptr;
    if (n_recenter > 0) {
      double* sums = ws;
      double* mn = ws + (size_t)npieces * nch_s * r;
      mdsx::pre(h, st);
      dc_own_sums_kernel<RM><<<dim3(nch_s, npieces), 256, 0, st>>>(P, off, c, r, rot, trans, sums,
                                                                   first_identity);
      int rc = launched(h, "dc_own_sums_kernel", st);
      if (rc) return rc;
      mdsx::pre(h, st);
      dc_mean_kernel<RM><<<1, 256, 0, st>>>(sums, npieces * (int)nch_s, r, n_recenter, mn);
      if ((rc = launched(h, "dc_mean_kernel", st))) return rc;
      mean = mn;
    }
    mdsx::pre(h, st);
    dc_stitch_kernel<RM><<<dim3(nch_t, npieces), 256, 0, st>>>(P, row_idx, off, c, r, rot, trans,
                                                                mean, out, first_identity);
    return launched(h, "dc_stitch_kernel", st);
  };
  if (r <= 4) return go(std::integral_constant<int, 4>{});
  if (r <= 8) return go(std::integral_constant<int, 8>{});
  if (r <= 10) return go(std::integral_constant<int, 10>{});
  if (r <= 16) return go(std::integral_constant<int, 16>{});
  return go(std::integral_constant<int, 32>{});
}

size_t dc_stitch_ws_bytes(int npieces, int r, int64_t max_m) {
  const size_t nch = (size_t)std::max<int64_t>(1, (max_m + OS_CR - 1) / OS_CR);
  return ((size_t)npieces * nch * r + 32) * sizeof(double);
}

int launch_scatter(mdsx_handle* h, const double* src, const int64_t* idx, int64_t n, int r,
                   double* out, cudaStream_t st) {
  if (n == 0) return MDSX_OK;
  const int64_t total = n * r;
  mdsx::pre(h, st);
  scatter_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(src, idx, n, r, out);
  return launched(h, "scatter_kernel", st);
}

size_t recenter_ws_bytes(int r) { return (size_t)RC_BLOCKS * r * sizeof(double); }

int launch_subtract_mean(mdsx_handle* h, double* X, int64_t n, int r, const double* part,
                         int nparts, const double* corr, cudaStream_t st, int64_t ndiv = 0);

int launch_recenter(mdsx_handle* h, double* X, int64_t n, int r, double* part, cudaStream_t st) {
  if (n == 0) return MDSX_OK;
  if (r <= 4) { mdsx::pre(h, st); colsum_partial_kernel<4><<<RC_BLOCKS, 256, 0, st>>>(X, n, r, part); }
  else if (r <= 8) { mdsx::pre(h, st); colsum_partial_kernel<8><<<RC_BLOCKS, 256, 0, st>>>(X, n, r, part); }
  else if (r <= 16) { mdsx::pre(h, st); colsum_partial_kernel<16><<<RC_BLOCKS, 256, 0, st>>>(X, n, r, part); }
  else { mdsx::pre(h, st); colsum_partial_kernel<32><<<RC_BLOCKS, 256, 0, st>>>(X, n, r, part); }
  int rc = launched(h, "colsum_partial_kernel", st);
  if (rc) return rc;
  return launch_subtract_mean(h, X, n, r, part, RC_BLOCKS, nullptr, st);
}

// X (n rows) -= (sum of the partials + corr) / ndiv (ndiv 0: n)
int launch_subtract_mean(mdsx_handle* h, double* X, int64_t n, int r, const double* part,
                         int nparts, const double* corr, cudaStream_t st, int64_t ndiv) {
  if (n == 0) return MDSX_OK;
  const int64_t total = n * r;
  int blocks = (int)std::min<int64_t>((total + 1023) / 1024, (int64_t)h->num_sms * 8);
  mdsx::pre(h, st);
  subtract_mean_kernel<<<blocks, 256, 0, st>>>(X, n, r, part, nparts, corr,
                                               (double)(ndiv > 0 ? ndiv : n));
  return launched(h, "subtract_mean_kernel", st);
}

int corr_ws_doubles(int64_t n, int r, int num_sms) {
  const int nq = 2 * r + (2 * r) * (2 * r + 1) / 2;
  const int64_t g = std::max<int64_t>(1, std::min<int64_t>((n + AC_TILE - 1) / AC_TILE, 2 * num_sms));
  return (int)(g * nq);
}

int launch_aligned_corr(mdsx_handle* h, const double* X, int64_t n, int r, const void* D,
                        int dtype, int64_t ld, double* part, double* corr, double* rot,
                        int32_t* zero_var, cudaStream_t st) {
  const int nq = 2 * r + (2 * r) * (2 * r + 1) / 2;
  const int g = (int)std::max<int64_t>(1, std::min<int64_t>((n + AC_TILE - 1) / AC_TILE, 2 * h->num_sms));
  mdsx::pre(h, st);
  if (dtype == MDSX_F32)
    corr_partial_kernel<float><<<g, AC_T, 0, st>>>(X, n, r, (const float*)D, ld, part, nq);
  else
    corr_partial_kernel<double><<<g, AC_T, 0, st>>>(X, n, r, (const double*)D, ld, part, nq);
  int rc = launched(h, "corr_partial_kernel", st);
  if (rc) return rc;
  mdsx::pre(h, st);
  corr_finish_kernel<<<1, AC_T, 0, st>>>(part, g, nq, n, r, corr, rot, zero_var);
  return launched(h, "corr_finish_kernel", st);
}

}  // namespace mdsx
