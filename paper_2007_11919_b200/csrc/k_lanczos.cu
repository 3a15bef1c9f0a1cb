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

// number of eigenvalues of the m x m tridiagonal (al, be2 = beta^2) below x
__device__ int sturm_below(const double* al, const double* be2, int m, double x, double pivmin) {
  double q = al[0] - x;
  if (fabs(q) < pivmin) q = -pivmin;
  int cnt = q < 0.0;
  for (int i = 1; i < m; ++i) {
    q = (al[i] - x) - be2[i - 1] / q;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
  }
  return cnt;
}

// Eigenvector of the m x m tridiagonal T (al, be) at its eigenvalue theta by a
// twisted factorisation of T - theta I: top-down LDL^T pivots d, bottom-up
// UDU^T pivots u, twist index with the smallest |d_k + u_k - (al_k - theta)|,
// then the vector outward from the twist (z_k = 1).  O(m), no pivoting needed.
template <int QMAX>
__device__ void tri_twisted_vector(const double* al, const double* be, int m, double theta,
                                   double pivmin, double* z /* m, out, unit norm */) {
  double d[QMAX], u[QMAX];
  double t = al[0] - theta;
  d[0] = fabs(t) < pivmin ? -pivmin : t;
  for (int i = 1; i < m; ++i) {
    t = (al[i] - theta) - be[i - 1] * be[i - 1] / d[i - 1];
    d[i] = fabs(t) < pivmin ? -pivmin : t;
  }
  t = al[m - 1] - theta;
  u[m - 1] = fabs(t) < pivmin ? -pivmin : t;
  for (int i = m - 2; i >= 0; --i) {
    t = (al[i] - theta) - be[i] * be[i] / u[i + 1];
    u[i] = fabs(t) < pivmin ? -pivmin : t;
  }
  int kt = 0;
  double best = 1e308;
  for (int i = 0; i < m; ++i) {
    const double g = fabs(d[i] + u[i] - (al[i] - theta));
    if (g < best) { best = g; kt = i; }
  }
  z[kt] = 1.0;
  for (int i = kt - 1; i >= 0; --i) z[i] = -(be[i] / d[i]) * z[i + 1];
  for (int i = kt + 1; i < m; ++i) z[i] = -(be[i - 1] / u[i]) * z[i - 1];
  double nrm = 0.0;
  for (int i = 0; i < m; ++i) nrm = fma(z[i], z[i], nrm);
  nrm = 1.0 / sqrt(nrm);
  for (int i = 0; i < m; ++i) z[i] *= nrm;
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

// w -= Q[:, 0..nc) (Q[:, 0..nc)^T w): dot products one warp each (lanes split
// the k entries, shuffle tree), then the update one row per thread.  Ends
// with hv[0..nc) = the coefficients; caller syncs before reading wv.
__device__ void cgs_project(const double* Q, int kq, int k, int nc, double* wv, double* hv) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c = warp; c < nc; c += LT / 32) {
    const double* qc = Q + (size_t)c * kq;
    double h = 0.0;
    for (int a = lane; a < k; a += 32) h = fma(qc[a], wv[a], h);
    h = mdsx::warp_sum(h);
    if (lane == 0) hv[c] = h;
  }
  __syncthreads();
  const int tid = threadIdx.x;
  if (tid < k) {
    double s0 = wv[tid], s1 = 0.0;
    int c = 0;
    for (; c + 1 < nc; c += 2) {
      s0 = fma(-Q[(size_t)c * kq + tid], hv[c], s0);
      s1 = fma(-Q[(size_t)(c + 1) * kq + tid], hv[c + 1], s1);
    }
    if (c < nc) s0 = fma(-Q[(size_t)c * kq + tid], hv[c], s0);
    wv[tid] = s0 + s1;
  }
}

template <int QMAX>
__global__ void __launch_bounds__(LT, QMAX <= QCAP_PIECES ? 2 : 1)
lanczos_smem_kernel(const PieceDesc* __restrict__ pd, int r, const double* __restrict__ Aall,
                    double* __restrict__ Uout, double* __restrict__ lam_out,
                    double* __restrict__ estimates, double* __restrict__ gof,
                    mdsx_piece_status* __restrict__ status, int qform_trivial) {
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
  const int qcap = min(QMAX, k);

  double fro = 0.0, tr = 0.0;
  for (int i = 0; i < k; ++i) {                // packed copy, coalesced per row
    const int off = i * k - i * (i - 1) / 2;
    for (int a = i + tid; a < k; a += LT) {
      const double v = Ag[(int64_t)i * k + a];
      A[off + a - i] = v;
      fro = fma((a == i ? 1.0 : 2.0) * v, v, fro);   // off-diagonal entries count twice
      if (a == i) tr += v;
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
  const int row_off = tid < k ? tid * k - tid * (tid - 1) / 2 - tid : 0;   // packed row base

  int m = 0;                 // current Krylov dimension (columns 0..m-1 of Q valid)
  bool done = false, broke = false, capped = false;
  const int first_check = max(2 * r + 4, 24);
  while (!done) {
    const double* q = Q + (size_t)m * kq;
    // w = A q with the packed symmetric A: row i = sum_{a<i} A[a][i] q_a + sum_{a>=i} A[i][a] q_a
    if (tid < k) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int off = 0;
      int a = 0;
      for (; a < tid; ++a) {                   // column part (coalesced across threads)
        a1 = fma(A[off + tid - a], q[a], a1);
        off += k - a;
      }
      const double* rowp = A + row_off;
      for (; a + 1 < k; a += 2) {              // own row part
        a0 = fma(rowp[a], q[a], a0);
        a2 = fma(rowp[a + 1], q[a + 1], a2);
      }
      if (a < k) a3 = fma(rowp[a], q[a], a3);
      wv[tid] = (a0 + a1) + (a2 + a3);
    }
    __syncthreads();
    double al = 0.0;
    for (int pass = 0; pass < 2; ++pass) {     // CGS2 against Q[:, 0..m]
      cgs_project(Q, kq, k, m + 1, wv, hv);
      al += hv[m];
      __syncthreads();
    }
    const double b = sqrt(block_sum(tid < k ? wv[tid] * wv[tid] : 0.0, red));
    if (tid == 0) {
      alpha[m] = al;
      beta[m] = b;
      beta2[m] = b * b;
    }
    m += 1;
    const bool full = (m >= k);
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
    for (int it = 0; it < 14; ++it) {              // 17^14 > 1e17: interval at fp resolution
      const bool active = grp < rr;
      double lo = 0.0, hi = 0.0;
      bool below_ok = false;
      if (active) {
        lo = lo_s[grp];
        hi = hi_s[grp];
        const double x = lo + (hi - lo) * (double)(sl + 1) / (double)(MS + 1);
        below_ok = sturm_below(alpha, beta2, m, x, pivmin) <= m - 1 - grp;   // grp-th largest
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
    if (tid < rr) theta[tid] = 0.5 * (lo_s[tid] + hi_s[tid]);
    __syncthreads();
    // eigenvectors of T_m (one thread per eigenvalue), S[c*RMAX + i]
    if (tid < rr) {
      double z[QMAX];
      tri_twisted_vector<QMAX>(alpha, beta, m, theta[tid], pivmin + 1e-300, z);
      for (int c = 0; c < m; ++c) S[c * RMAX + tid] = z[c];
    }
    __syncthreads();
    if (tid < 32) {            // MGS inside eigenvalue clusters only (fixed order, warp 0)
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
  }
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
  return ((size_t)kmax * (kmax + 1) / 2 + (size_t)qmax * (kmax | 1) + (size_t)qmax * RMAX) *
         sizeof(double);
}

size_t lanczos_smem_bytes(int kmax) { return lanczos_bytes(kmax, LMAX); }

// full_basis: Krylov capacity = LMAX (one CTA / SM, never flags -2; used for
// the Rayleigh-Ritz matrices of the block-Krylov solver); otherwise
// QCAP_PIECES (two CTAs / SM, capacity overflow -> Jacobi fallback).
int launch_lanczos_smem(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r,
                        const double* A, double* U, double* lam, double* estimates, double* gof,
                        mdsx_piece_status* status, int full_basis, cudaStream_t st) {
  if (npieces == 0) return MDSX_OK;
  auto go = [&](auto kern, int qmax) {
    const size_t smem = lanczos_bytes(kmax, qmax);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mdsx::pre(h, st);
    kern<<<npieces, LT, smem, st>>>(pd, r, A, U, lam, estimates, gof, status, 1);
    return launched(h, "lanczos_smem_kernel", st);
  };
  return full_basis ? go(lanczos_smem_kernel<LMAX>, LMAX)
                    : go(lanczos_smem_kernel<QCAP_PIECES>, QCAP_PIECES);
}

}  // namespace mdsx
