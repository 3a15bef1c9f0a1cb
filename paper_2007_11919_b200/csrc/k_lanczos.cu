// K3 top-r eigensolver for the per-piece k x k PSD Gram matrices (k <= 104):
// Krylov subspace iteration (Lanczos) with full re-orthogonalisation, one CTA
// per piece, the matrix A (packed upper triangle) and a Krylov basis Q of at
// most QMAX columns resident in shared memory — ~105 KB, so two pieces run
// per SM and hide each other's barrier/latency stalls.  A piece that needs
// more than QMAX Krylov vectors is flagged (status NUMERICAL, value -2) and
// re-solved by the full Jacobi kernel launched right after (in stream order,
// no host sync).
//
//   step j:  w = A q_j ;  w -= Q (Q^T w) twice (CGS2) ;  alpha_j = q_j^T A q_j ;
//            beta_j = |w| ;  q_{j+1} = w / beta_j
//
// With full re-orthogonalisation Q stays orthonormal to working precision
// and T_j = Q^T A Q is tridiagonal (alpha, beta): this is Householder
// tridiagonalisation restricted to the Krylov space, so it reaches the exact
// answer at j = k at the latest.  Every 8 steps the top-r eigenpairs of T_j
// are computed in parallel — eigenvalues by 16-way multisection on Sturm
// counts (one half-warp per eigenvalue), vectors by a twisted factorisation
// of T - theta I (one O(j) pass, as LAPACK's dlar1v) with MGS only inside
// eigenvalue clusters — and the Lanczos residual |beta_j s_i(j)|, which
// equals |A y_i - theta_i y_i|, is tested against 1e-12 theta_1.  Ritz
// vectors y_i = Q s_i are the eigenvectors returned.
//
// Work per step ~k^2 (matvec) + 4 k j (re-orthogonalisation); typical j for
// the BASELINE pieces is 24-40, against ~9 k^3 for the full dsyevd the
// reference calls (linalg.py:161).  G1/G2 use trace(A) (PSD Gram of
// Euclidean data: Sum|lambda| = trace, G1 == G2 bitwise, classical.py:75-85).
#include "mdsx_common.cuh"
#include "piece_solvers.cuh"

#include <algorithm>
#include <cstdlib>

#ifdef MDSX_LZ_PROF
#define LZ_T0(v) long long v = clock64()
#define LZ_ACC(slot, v) if (blockIdx.x == 0 && threadIdx.x == 0) lzp[slot] += clock64() - v
#else
#define LZ_T0(v)
#define LZ_ACC(slot, v)
#endif

namespace {

constexpr int LT = 256;          // threads per CTA
constexpr int MS = 16;           // multisection width (threads per eigenvalue)
constexpr int LMAX = 104;        // largest k for this kernel (smem budget)
constexpr int RMAX = 16;         // largest r (16 half-warps of 16 threads)
constexpr int QCAP_PIECES = 56;  // Krylov basis capacity for plan pieces (2 CTAs / SM)
constexpr int CHECK_EVERY = 8;

__device__ __forceinline__ double hash_unit(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return (double)(x >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
}

// number of eigenvalues of the m x m tridiagonal (al, be2 = beta^2) below x:
// sign changes of the leading-minor sequence p_i = det(T_i - x I),
// p_i = (al_i - x) p_{i-1} - be2_{i-1} p_{i-2}  (division free; the pair is
// rescaled when it leaves [1e-150, 1e150]; an exact zero counts as a change,
// the limit of the LDL^T pivot rule).
__device__ int sturm_below(const double* al, const double* be2, int m, double x) {
  double pm = 1.0, pc = al[0] - x;
  if (pc == 0.0) pc = -1e-300;
  int cnt = pc < 0.0;
  for (int i = 1; i < m; ++i) {
    double pn = fma(al[i] - x, pc, -be2[i - 1] * pm);
    if (pn == 0.0) pn = pc < 0.0 ? 1e-300 : -1e-300;
    cnt += (pn < 0.0) != (pc < 0.0);
    pm = pc;
    pc = pn;
    if (i & 1) {                        // rescale every other step (off the per-step chain)
      const double ap = fabs(pc);
      if (ap > 1e100) { pc *= 1e-100; pm *= 1e-100; }
      else if (ap < 1e-100) { pc *= 1e100; pm *= 1e100; }
    }
  }
  return cnt;
}

// Reciprocal for the serial recurrences.  Measured on B200 (tools/lat_micro.cu):
// a dependent DDIV costs ~60 clk, a float-seeded Newton reciprocal ~130 clk
// (two F2F conversions + MUFU on the chain), so plain division wins.
__device__ __forceinline__ double fast_rcp(double d) { return 1.0 / d; }

// Eigenvector of the m x m tridiagonal T (al, be) at its eigenvalue theta by a
// twisted factorisation of T - theta I: top-down LDL^T pivots d, bottom-up
// UDU^T pivots u, twist index with the smallest |d_k + u_k - (al_k - theta)|,
// then the vector outward from the twist (z_k = 1).  O(m), no pivoting needed.
// Twisted factorisation of T - theta I (T: m x m tridiagonal, al / be) with
// the pivots in shared-memory columns (stride RMAX, one column per calling
// thread): top-down LDL^T pivots d (in zc), bottom-up UDU^T pivots u (in uc),
// twist kt = argmin |gamma_k|, gamma_k = d_k + u_k - (al_k - theta); then the
// vector outward from the twist (z_kt = 1) overwrites zc.  Returns gamma_kt
// and |z|^2 (z is left unnormalised): (T - theta I) z = gamma_kt e_kt, so
// theta + gamma_kt / |z|^2 is the Rayleigh quotient of z.  O(m).
__device__ void tri_twisted(const double* al, const double* be, int m, double theta,
                            double pivmin, double* zc, double* uc, double& gamma, double& nrm2) {
  // forward LDL^T pivots d (into zc) and backward UDU^T pivots u (into uc):
  // two independent chains, interleaved to overlap their divide latencies
  double t = al[0] - theta;
  double dprev = fabs(t) < pivmin ? -pivmin : t;
  zc[0] = dprev;
  t = al[m - 1] - theta;
  double unext = fabs(t) < pivmin ? -pivmin : t;
  uc[(m - 1) * RMAX] = unext;
  for (int i = 1, j = m - 2; i < m; ++i, --j) {
    const double td = (al[i] - theta) - be[i - 1] * be[i - 1] * fast_rcp(dprev);
    const double tu = (al[j] - theta) - be[j] * be[j] * fast_rcp(unext);
    dprev = fabs(td) < pivmin ? -pivmin : td;
    unext = fabs(tu) < pivmin ? -pivmin : tu;
    zc[i * RMAX] = dprev;
    uc[j * RMAX] = unext;
  }
  // twist: argmin |gamma_k|, gamma_k = d_k + u_k - (al_k - theta)
  int kt = m - 1;
  double gk = zc[(m - 1) * RMAX] + uc[(m - 1) * RMAX] - (al[m - 1] - theta);
  double best = fabs(gk);
  for (int i = m - 2; i >= 0; --i) {
    const double g = zc[i * RMAX] + uc[i * RMAX] - (al[i] - theta);
    if (fabs(g) < best) { best = fabs(g); gk = g; kt = i; }
  }
  // vector outward from the twist (z_kt = 1): both directions interleaved
  double n2 = 1.0, zl = 1.0, zr = 1.0;
  int il = kt - 1, ir = kt + 1;
  while (il >= 0 || ir < m) {
    if (il >= 0) {                              // reads d_il, writes z_il in place
      zl = -(be[il] * fast_rcp(zc[il * RMAX])) * zl;
      zc[il * RMAX] = zl;
      n2 = fma(zl, zl, n2);
      --il;
    }
    if (ir < m) {
      zr = -(be[ir - 1] * fast_rcp(uc[ir * RMAX])) * zr;
      zc[ir * RMAX] = zr;
      n2 = fma(zr, zr, n2);
      ++ir;
    }
  }
  zc[kt * RMAX] = 1.0;
  gamma = gk;
  nrm2 = n2;
}

__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = mdsx::warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < LT / 32; ++w) s += red[w];   // fixed order
  return s;
}

// w -= Q[:, 0..nc) (Q[:, 0..nc)^T w).  Dots: 4 threads per column (k split
// in 4 contiguous parts, 2 accumulators each, 2-level shuffle); update: 2
// threads per row (columns split in halves, 1 shuffle).  Ends with
// hv[0..nc) = the coefficients and wv updated; caller syncs before reading wv.
__device__ void cgs_project(const double* Q, int kq, int k, int nc, double* wv, double* hv) {
  const int tid = threadIdx.x;
  const int part = tid & 3;
  const int seg = (k + 3) >> 2;
  for (int c = tid >> 2; c < ((nc + 7) & ~7); c += LT / 4) {     // warp-uniform trip count
    double h0 = 0.0, h1 = 0.0;
    if (c < nc) {
      const double* qc = Q + (size_t)c * kq;
      const int a1 = min(k, (part + 1) * seg);
      int a = part * seg;
      for (; a + 1 < a1; a += 2) {
        h0 = fma(qc[a], wv[a], h0);
        h1 = fma(qc[a + 1], wv[a + 1], h1);
      }
      if (a < a1) h0 = fma(qc[a], wv[a], h0);
    }
    double h = h0 + h1;
    h += __shfl_xor_sync(0xffffffffu, h, 1);
    h += __shfl_xor_sync(0xffffffffu, h, 2);
    if (c < nc && part == 0) hv[c] = h;
  }
  __syncthreads();
  const int hf = tid & 1;
  const int cmid = (nc + 1) >> 1;
  for (int a = tid >> 1; a < ((k + 15) & ~15); a += LT / 2) {
    double s0 = 0.0, s1 = 0.0;
    if (a < k) {
      const int c1 = hf ? nc : cmid;
      int c = hf ? cmid : 0;
      for (; c + 1 < c1; c += 2) {
        s0 = fma(Q[(size_t)c * kq + a], hv[c], s0);
        s1 = fma(Q[(size_t)(c + 1) * kq + a], hv[c + 1], s1);
      }
      if (c < c1) s0 = fma(Q[(size_t)c * kq + a], hv[c], s0);
    }
    double t = s0 + s1;
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    if (a < k && hf == 0) wv[a] -= t;
  }
}

template <int QMAX>
__global__ void __launch_bounds__(LT, QMAX <= QCAP_PIECES ? 2 : 1)
lanczos_smem_kernel(const PieceDesc* __restrict__ pd, int r, const double* __restrict__ Aall,
                    double* __restrict__ Uout, double* __restrict__ lam_out,
                    double* __restrict__ estimates, double* __restrict__ gof,
                    mdsx_piece_status* __restrict__ status, int only_flagged) {
  extern __shared__ double sm[];
  __shared__ double alpha[QMAX], beta[QMAX], beta2[QMAX];
  __shared__ double wv[LMAX], hv[QMAX + 1];
  __shared__ double theta[RMAX], lo_s[RMAX], hi_s[RMAX];
  __shared__ double red[LT / 32];
  __shared__ double trace_s, anorm_s;
  __shared__ int conv_s;

  const PieceDesc d = pd[blockIdx.x];
  const int pid = d.id, k = d.k;
  const int kq = k | 1;                        // odd leading dim of Q (conflict-free columns)
  const int tid = threadIdx.x;
  const double* Ag = Aall + d.a_off;
  if (only_flagged) {           // fallback pass: only pieces the subspace kernel handed over
    const mdsx_piece_status s0 = status[pid];
    if (!(s0.code == MDSX_NUMERICAL && s0.value == -3.0)) return;
    __syncthreads();
    if (tid == 0) status[pid] = mdsx_piece_status{MDSX_OK, 0, 0.0};
    __syncthreads();
  }
  if (status[pid].code == MDSX_INVALID_INPUT) {   // non-finite rows: nothing to solve
    for (int e = tid; e < k * r; e += LT) Uout[d.u_off + e] = 0.0;
    if (tid < r) {
      estimates[(int64_t)pid * r + tid] = 0.0;
      lam_out[(int64_t)pid * r + tid] = 0.0;
    }
    if (tid < 2) gof[2 * (int64_t)pid + tid] = 0.0;
    return;
  }
  double* A = sm;                              // packed upper: row i = A[i][i..k)
  double* Q = A + (size_t)k * (k + 1) / 2;     // column j at Q + j*kq, j < QMAX
  double* S = Q + (size_t)QMAX * kq;           // Ritz coefficients, S[c*RMAX + i]
  double* U2 = S + (size_t)QMAX * RMAX;        // twisted-factorisation scratch, same layout
  const int qcap = min(QMAX, k);

  double fro = 0.0, tr = 0.0;
  {                                            // packed copy: 4 independent loads in flight
    const int kk2 = k * k;
    for (int e0 = tid; e0 < kk2; e0 += 4 * LT) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * LT;
        v[u] = e < kk2 ? Ag[e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * LT;
        if (e < kk2) {
          const int i = e / k, a = e - i * k;
          if (a >= i) {
            A[i * k - i * (i - 1) / 2 + a - i] = v[u];
            fro = fma((a == i ? 1.0 : 2.0) * v[u], v[u], fro);   // off-diagonal entries count twice
            if (a == i) tr += v[u];
          }
        }
      }
    }
  }
  fro = block_sum(fro, red);
  tr = block_sum(tr, red);
  if (tid == 0) { trace_s = tr; anorm_s = sqrt(fro); }
  // q_0: batch-independent pseudo-random unit vector
  double q0 = tid < k ? hash_unit((uint64_t)tid * 0x9E37ull + 17) : 0.0;
  const double n0 = sqrt(block_sum(q0 * q0, red));
  if (tid < k) Q[tid] = q0 / n0;
  __syncthreads();
  const double anorm = anorm_s;

  int m = 0;                 // current Krylov dimension (columns 0..m-1 of Q valid)
  bool done = false, broke = false, capped = false;
  const int first_check = max(2 * r + 4, 24);
#ifdef MDSX_LZ_PROF
  long long lzp[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  LZ_T0(t_all);
#endif
  while (!done) {
    const double* q = Q + (size_t)m * kq;
    LZ_T0(t_mv);
    // w = A q with the packed symmetric A: row i = sum_{a<i} A[a][i] q_a + sum_{a>=i} A[i][a] q_a;
    // two threads per row (a split in halves, 2 accumulators per part), one shuffle
    {
      const int i = tid >> 1, hf = tid & 1;
      const int kh = (k + 1) >> 1;
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      if (i < k) {
        const int a0 = hf * kh, a1 = min(k, a0 + kh);
        const int cend = min(a1, i);
        int a = a0;
        int off = a * k - a * (a - 1) / 2;      // packed offset of row a
        for (; a + 1 < cend; a += 2) {          // column part
          s0 = fma(A[off + i - a], q[a], s0);
          off += k - a;
          s1 = fma(A[off + i - a - 1], q[a + 1], s1);
          off += k - a - 1;
        }
        if (a < cend) s0 = fma(A[off + i - a], q[a], s0);
        const double* rowp = A + (i * k - i * (i - 1) / 2) - i;
        a = max(a0, i);
        double s4 = 0.0, s5 = 0.0;
        for (; a + 3 < a1; a += 4) {            // own row part, 4 chains
          s2 = fma(rowp[a], q[a], s2);
          s3 = fma(rowp[a + 1], q[a + 1], s3);
          s4 = fma(rowp[a + 2], q[a + 2], s4);
          s5 = fma(rowp[a + 3], q[a + 3], s5);
        }
        for (; a < a1; ++a) s2 = fma(rowp[a], q[a], s2);
        s2 += s4;
        s3 += s5;
      }
      double t = (s0 + s1) + (s2 + s3);
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      if (i < k && hf == 0) wv[i] = t;
    }
    __syncthreads();
    LZ_ACC(0, t_mv);
    LZ_T0(t_cgs);
    double al = 0.0;
    for (int pass = 0; pass < 2; ++pass) {     // CGS2 against Q[:, 0..m]
      cgs_project(Q, kq, k, m + 1, wv, hv);
      al += hv[m];
      __syncthreads();
    }
    LZ_ACC(1, t_cgs);
    LZ_T0(t_b);
    const double b = sqrt(block_sum(tid < k ? wv[tid] * wv[tid] : 0.0, red));
    if (tid == 0) {
      alpha[m] = al;
      beta[m] = b;
      beta2[m] = b * b;
    }
    m += 1;
    const bool full = (m >= k);
    LZ_ACC(2, t_b);
    broke = false;
    if (!full && m < qcap) {
      if (b > 1e-13 * anorm) {
        if (tid < k) Q[(size_t)m * kq + tid] = wv[tid] / b;
      } else {
        // invariant subspace: continue from a fresh direction orthogonal to Q
        // (finds further copies of repeated eigenvalues)
        broke = true;
        if (tid == 0) { beta[m - 1] = 0.0; beta2[m - 1] = 0.0; }
        if (tid < k) wv[tid] = hash_unit(((uint64_t)m << 20) ^ (uint64_t)tid);
        __syncthreads();
        for (int pass = 0; pass < 2; ++pass) {
          cgs_project(Q, kq, k, m, wv, hv);
          __syncthreads();
        }
        const double nb = sqrt(block_sum(tid < k ? wv[tid] * wv[tid] : 0.0, red));
        if (tid < k) Q[(size_t)m * kq + tid] = wv[tid] / nb;
      }
    }
    __syncthreads();
    capped = !full && m >= qcap;
    if (!(full || capped || (!broke && m >= first_check && m % CHECK_EVERY == 0))) continue;

    LZ_T0(t_ck);
    // ---- top-r eigenpairs of T_m: multisection (16 threads per eigenvalue)
    const int rr = r < m ? r : m;
    double gl = 1e308, gu = -1e308, bmax = 0.0;
    for (int i = 0; i < m; ++i) {
      const double off = (i > 0 ? fabs(beta[i - 1]) : 0.0) + (i + 1 < m ? fabs(beta[i]) : 0.0);
      gl = fmin(gl, alpha[i] - off);
      gu = fmax(gu, alpha[i] + off);
      if (i + 1 < m) bmax = fmax(bmax, beta2[i]);
    }
    const double pivmin = 1e-290 * fmax(1.0, bmax);
    const int grp = tid / MS, sl = tid % MS;
    if (tid < RMAX && tid < rr) { lo_s[tid] = gl; hi_s[tid] = gu; }
    __syncthreads();
    // multisection rounds: 6 bring each bracket to ~1e-7 of the Gershgorin
    // width; one Rayleigh-quotient step from the twisted factorisation then
    // lands at working precision (cubic).  A quotient outside its bracket (a
    // cluster tighter than the bracket) falls back to 8 more rounds.
    auto msect = [&](int rounds) {
      for (int it = 0; it < rounds; ++it) {
        const bool active = grp < rr;
        double lo = 0.0, hi = 0.0;
        bool below_ok = false;
        if (active) {
          lo = lo_s[grp];
          hi = hi_s[grp];
          const double x = lo + (hi - lo) * (double)(sl + 1) / (double)(MS + 1);
          below_ok = sturm_below(alpha, beta2, m, x) <= m - 1 - grp;   // grp-th largest
        }
        const unsigned okm = __ballot_sync(0xffffffffu, below_ok);
        // counts are monotone in x: points sl < c are below the eigenvalue
        const int c = __popc((okm >> ((threadIdx.x & 31) & ~(MS - 1))) & 0xFFFFu);
        __syncthreads();
        if (active && sl == 0) {
          lo_s[grp] = c > 0 ? lo + (hi - lo) * (double)c / (double)(MS + 1) : lo;
          hi_s[grp] = c < MS ? lo + (hi - lo) * (double)(c + 1) / (double)(MS + 1) : hi;
        }
        __syncthreads();
      }
    };
    LZ_T0(t_ms6);
    msect(6);
    LZ_ACC(5, t_ms6);
    LZ_T0(t_rq);
    int rq_bad = 0;
    if (tid < rr) {
      const double lo = lo_s[tid], hi = hi_s[tid], th0 = 0.5 * (lo + hi);
      double gam, n2;
      tri_twisted(alpha, beta, m, th0, pivmin + 1e-300, S + tid, U2 + tid, gam, n2);
      const double th1 = th0 + gam / n2;
      if (th1 >= lo && th1 <= hi) theta[tid] = th1;
      else rq_bad = 1;
    }
    const int any_bad = __syncthreads_or(rq_bad);
    LZ_ACC(6, t_rq);
#ifdef MDSX_LZ_PROF
    if (blockIdx.x == 0 && tid == 0) { lzp[8] += any_bad; lzp[9] += 1; }
#endif
    if (any_bad) {
      msect(8);                                    // 17^14 > 1e17: bracket at fp resolution
      if (tid < rr) theta[tid] = 0.5 * (lo_s[tid] + hi_s[tid]);
    }
    __syncthreads();
    // eigenvectors of T_m at the final theta (one thread per eigenvalue), S[c*RMAX + i]
    if (tid < rr) {
      double gam, n2;
      tri_twisted(alpha, beta, m, theta[tid], pivmin + 1e-300, S + tid, U2 + tid, gam, n2);
      const double sc = 1.0 / sqrt(n2);
      for (int c = 0; c < m; ++c) S[c * RMAX + tid] *= sc;
    }
    __syncthreads();
    LZ_ACC(3, t_ck);
    LZ_T0(t_mgs);
    // clusters are runs of adjacent Ritz values (theta is descending): skip the
    // MGS pass entirely when no neighbours are within the cluster tolerance
    const int adj = tid >= 1 && tid < rr && fabs(theta[tid - 1] - theta[tid]) <= 1e-3 * fabs(theta[0]);
    if (__syncthreads_or(adj) && tid < 32) {   // MGS inside eigenvalue clusters only (fixed order, warp 0)
      const int lane = tid;
      const double ctol = 1e-3 * fabs(theta[0]);
      for (int i = 1; i < rr; ++i) {
        bool touched = false;
        for (int j = 0; j < i; ++j) {
          if (fabs(theta[i] - theta[j]) > ctol) continue;
          touched = true;
          double dt = 0.0;
          for (int t = lane; t < m; t += 32) dt = fma(S[t * RMAX + i], S[t * RMAX + j], dt);
          dt = mdsx::warp_sum(dt);
          for (int t = lane; t < m; t += 32) S[t * RMAX + i] = fma(-dt, S[t * RMAX + j], S[t * RMAX + i]);
          __syncwarp();
        }
        if (touched) {
          double nr = 0.0;
          for (int t = lane; t < m; t += 32) nr = fma(S[t * RMAX + i], S[t * RMAX + i], nr);
          nr = sqrt(mdsx::warp_sum(nr));
          for (int t = lane; t < m; t += 32) S[t * RMAX + i] /= nr;
          __syncwarp();
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      int ok = rr == r;
      const double bm = full ? 0.0 : beta[m - 1];
      for (int i = 0; i < rr && ok; ++i)
        if (!(fabs(bm * S[(m - 1) * RMAX + i]) <= 1e-12 * fabs(theta[0]))) ok = 0;
      conv_s = ok || full ? 1 : (capped ? 2 : 0);
    }
    __syncthreads();
    done = conv_s != 0;
    LZ_ACC(4, t_mgs);
  }
#ifdef MDSX_LZ_PROF
  LZ_ACC(7, t_all);
  if (blockIdx.x == 0 && tid == 0)
    printf("lz prof m=%d matvec %lld cgs %lld beta+norm %lld check %lld (msect6 %lld rq %lld fallbacks %lld/%lld) mgs+resid %lld total %lld\n", m,
           lzp[0], lzp[1], lzp[2], lzp[3], lzp[5], lzp[6], lzp[8], lzp[9], lzp[4], lzp[7]);
#endif
  if (conv_s == 2) {          // basis capacity exhausted: the full Jacobi kernel takes over
    if (tid == 0 && status[pid].code == MDSX_OK) status[pid] = mdsx_piece_status{MDSX_NUMERICAL, 0, -2.0};
    return;
  }

  // Ritz vectors y_i = Q s_i  (k x r) and outputs
  for (int e = tid; e < k * r; e += LT) {
    const int a = e / r, i = e % r;
    double u = 0.0;
    if (i < m)
      for (int c = 0; c < m; ++c) u = fma(Q[(size_t)c * kq + a], S[c * RMAX + i], u);
    Uout[d.u_off + e] = u;
  }
  if (tid == 0) {
    const double top = theta[0];
    const double tol = 1e-8 * fabs(top);
    mdsx_piece_status st{MDSX_OK, 0, 0.0};
    if (status[pid].code != MDSX_OK) st.code = status[pid].code;
    double kept = 0.0;
    for (int i = 0; i < r; ++i) {
      double v = i < m ? theta[i] : 0.0;
      if (fabs(v) <= tol) v = 0.0;
      if (st.code == MDSX_OK && v <= 0.0) { st.code = MDSX_DEGENERATE; st.index = i + 1; st.value = v; }
      kept += v;
      lam_out[(int64_t)pid * r + i] = v;
      estimates[(int64_t)pid * r + i] = v / d.m;
    }
    if (st.code == MDSX_OK) st.value = (double)m;      // diagnostics: Krylov dimension used
    status[pid] = st;
    const double g = st.code == MDSX_OK ? kept / trace_s : 0.0;
    gof[2 * (int64_t)pid] = g;
    gof[2 * (int64_t)pid + 1] = g;
  }
}

}  // namespace

namespace mdsx {

int lanczos_kmax() { return LMAX; }
int lanczos_rmax() { return RMAX; }

static size_t lanczos_bytes(int kmax, int qmax) {
  return ((size_t)kmax * (kmax + 1) / 2 + (size_t)qmax * (kmax | 1) + 2 * (size_t)qmax * RMAX) *
         sizeof(double);
}

size_t lanczos_smem_bytes(int kmax) { return lanczos_bytes(kmax, LMAX); }

// full_basis: Krylov capacity = LMAX (one CTA / SM, never flags -2; used for
// the Rayleigh-Ritz matrices of the block-Krylov solver); otherwise
// QCAP_PIECES (two CTAs / SM, capacity overflow -> Jacobi fallback).
int launch_lanczos_smem(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r,
                        const double* A, double* U, double* lam, double* estimates, double* gof,
                        mdsx_piece_status* status, int full_basis, int only_flagged,
                        cudaStream_t st) {
  if (npieces == 0) return MDSX_OK;
  auto go = [&](auto kern, int qmax) {
    size_t smem = lanczos_bytes(kmax, qmax);
    if (getenv("MDSX_LZ_ONE")) smem = std::max<size_t>(smem, 120 * 1024);   // experiment: 1 CTA/SM
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mdsx::pre(h, st);
    kern<<<npieces, LT, smem, st>>>(pd, r, A, U, lam, estimates, gof, status, only_flagged);
    return launched(h, "lanczos_smem_kernel", st);
  };
  return full_basis ? go(lanczos_smem_kernel<LMAX>, LMAX)
                    : go(lanczos_smem_kernel<QCAP_PIECES>, QCAP_PIECES);
}

}  // namespace mdsx
