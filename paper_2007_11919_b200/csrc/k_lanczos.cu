// K3 top-r eigensolver for the per-piece k x k PSD Gram matrices (k <= 104):
// Krylov subspace iteration (Lanczos) with full re-orthogonalisation, one CTA
// per piece, the matrix A and the Krylov basis Q resident in shared memory.
//
//   step j:  w = A q_j ;  w -= Q (Q^T w) twice (CGS2) ;  alpha_j = q_j^T A q_j ;
//            beta_j = |w| ;  q_{j+1} = w / beta_j
//
// With full re-orthogonalisation Q stays orthonormal to working precision
// and T_j = Q^T A Q is tridiagonal (alpha, beta): this is Householder
// tridiagonalisation restricted to the Krylov space, so it reaches the exact
// answer at j = k at the latest.  Every 8 steps the top-r eigenpairs of T_j
// are computed in parallel — eigenvalues by 16-way multisection on Sturm
// counts (one half-warp per eigenvalue), vectors by inverse iteration with a
// pivoted tridiagonal LU — and the Lanczos residual |beta_j s_i(j)|, which
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

// inverse iteration for the eigenvector of tridiagonal T (al, be) at theta:
// LU of (T - theta I) with partial pivoting (dgttrf layout), two solves.
__device__ void tri_inverse_iteration(const double* al, const double* be, int m, double theta,
                                      double tiny, double* x /* m, out */) {
  double d[LMAX], du[LMAX], du2[LMAX], dl[LMAX];
  int piv[LMAX];
  for (int i = 0; i < m; ++i) {
    d[i] = al[i] - theta;
    du[i] = i + 1 < m ? be[i] : 0.0;
    dl[i] = i + 1 < m ? be[i] : 0.0;
    du2[i] = 0.0;
  }
  for (int i = 0; i + 1 < m; ++i) {
    if (fabs(d[i]) >= fabs(dl[i])) {           // no interchange
      piv[i] = 0;
      if (d[i] == 0.0) d[i] = tiny;
      const double f = dl[i] / d[i];
      dl[i] = f;
      d[i + 1] -= f * du[i];
    } else {                                   // interchange rows i, i+1
      piv[i] = 1;
      const double f = d[i] / dl[i];
      d[i] = dl[i];
      dl[i] = f;
      const double t = du[i];
      du[i] = d[i + 1];
      d[i + 1] = t - f * d[i + 1];
      if (i + 2 < m) {
        du2[i] = du[i + 1];
        du[i + 1] = -f * du[i + 1];
      }
    }
  }
  if (d[m - 1] == 0.0) d[m - 1] = tiny;
  for (int i = 0; i < m; ++i) x[i] = 1.0;
  for (int it = 0; it < 3; ++it) {
    for (int i = 0; i + 1 < m; ++i) {          // apply L^-1 (with interchanges)
      if (piv[i]) {
        const double t = x[i];
        x[i] = x[i + 1];
        x[i + 1] = t - dl[i] * x[i + 1];
      } else {
        x[i + 1] -= dl[i] * x[i];
      }
    }
    x[m - 1] /= d[m - 1];                      // U^-1
    if (m > 1) x[m - 2] = (x[m - 2] - du[m - 2] * x[m - 1]) / d[m - 2];
    for (int i = m - 3; i >= 0; --i) x[i] = (x[i] - du[i] * x[i + 1] - du2[i] * x[i + 2]) / d[i];
    double nrm = 0.0;
    for (int i = 0; i < m; ++i) nrm = fma(x[i], x[i], nrm);
    nrm = sqrt(nrm);
    for (int i = 0; i < m; ++i) x[i] /= nrm;
  }
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

__global__ void __launch_bounds__(LT)
lanczos_smem_kernel(const PieceDesc* __restrict__ pd, int r, const double* __restrict__ Aall,
                    double* __restrict__ Uout, double* __restrict__ lam_out,
                    double* __restrict__ estimates, double* __restrict__ gof,
                    mdsx_piece_status* __restrict__ status, int qform_trivial) {
  extern __shared__ double sm[];
  __shared__ mdsx::PieceScratch ps;
  __shared__ double alpha[LMAX], beta[LMAX], beta2[LMAX];
  __shared__ double wv[LMAX], hv[LMAX + 1], part[2][LMAX];
  __shared__ double theta[RMAX], lo_s[RMAX], hi_s[RMAX];
  __shared__ double red[LT / 32];
  __shared__ double trace_s, anorm_s;
  __shared__ int conv_s;

  const PieceDesc d = pd[blockIdx.x];
  const int pid = d.id, k = d.k;
  const int kq = k | 1;                        // odd leading dim of Q (conflict-free columns)
  const int tid = threadIdx.x;
  const double* Ag = Aall + d.a_off;
  double* A = sm;                              // k x k
  double* Q = A + (size_t)k * k;               // column j at Q + j*kq
  double* S = Q + (size_t)k * kq;              // m x r Ritz coefficients (column i at S + i*k)

  double fro = 0.0, tr = 0.0;
  for (int e = tid; e < k * k; e += LT) {
    const double v = Ag[e];
    A[e] = v;
    fro = fma(v, v, fro);
    if (e / k == e % k) tr += v;
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

  // matvec mapping: two halves of the reduction index, thread -> (row, half)
  const int half = tid >> 7, row = tid & 127;
  const int a_lo = half ? k / 2 : 0, a_hi = half ? k : k / 2;

  int m = 0;                 // current Krylov dimension (columns 0..m-1 of Q valid)
  bool done = false;
  bool broke = false;        // last step hit an invariant subspace (restarted)
  int nconv_checks = 0;
  // Krylov dimension of the first convergence test (earlier tests never pass)
  const int first_check = max(2 * r + 4, 24);
  while (!done) {
    const double* q = Q + (size_t)m * kq;
    // w = A q  (A symmetric: read A[a][row] across threads; 4 independent chains)
    if (row < k) {
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int a = a_lo;
      for (; a + 3 < a_hi; a += 4) {
        a0 = fma(A[a * k + row], q[a], a0);
        a1 = fma(A[(a + 1) * k + row], q[a + 1], a1);
        a2 = fma(A[(a + 2) * k + row], q[a + 2], a2);
        a3 = fma(A[(a + 3) * k + row], q[a + 3], a3);
      }
      for (; a < a_hi; ++a) a0 = fma(A[a * k + row], q[a], a0);
      part[half][row] = (a0 + a1) + (a2 + a3);
    }
    __syncthreads();
    if (tid < k) wv[tid] = part[0][tid] + part[1][tid];
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
    if (!full) {
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
    if (!(full || (!broke && m >= first_check && m % CHECK_EVERY == 0))) continue;

    // ---- top-r eigenpairs of T_m: multisection (16 threads per eigenvalue)
    ++nconv_checks;
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
    // eigenvectors of T_m by inverse iteration (one thread per eigenvalue)
    if (tid < rr) {
      double x[LMAX];
      tri_inverse_iteration(alpha, beta, m, theta[tid], 1e-300 + 1e-16 * anorm, x);
      for (int i = 0; i < m; ++i) S[(size_t)tid * k + i] = x[i];
    }
    __syncthreads();
    if (tid < 32) {            // MGS across the r vectors (clusters), fixed order, warp 0
      const int lane = tid;
      for (int i = 1; i < rr; ++i) {
        double* si = S + (size_t)i * k;
        for (int j = 0; j < i; ++j) {
          const double* sj = S + (size_t)j * k;
          double dt = 0.0;
          for (int t = lane; t < m; t += 32) dt = fma(si[t], sj[t], dt);
          dt = mdsx::warp_sum(dt);
          for (int t = lane; t < m; t += 32) si[t] = fma(-dt, sj[t], si[t]);
          __syncwarp();
        }
        double nr = 0.0;
        for (int t = lane; t < m; t += 32) nr = fma(si[t], si[t], nr);
        nr = sqrt(mdsx::warp_sum(nr));
        for (int t = lane; t < m; t += 32) si[t] /= nr;
        __syncwarp();
      }
    }
    __syncthreads();
    if (tid == 0) {
      int ok = rr == r;
      const double bm = full ? 0.0 : beta[m - 1];
      for (int i = 0; i < rr && ok; ++i)
        if (!(fabs(bm * S[(size_t)i * k + m - 1]) <= 1e-12 * fabs(theta[0]))) ok = 0;
      conv_s = ok || full;
    }
    __syncthreads();
    done = conv_s != 0;
  }

  // Ritz vectors y_i = Q s_i  (k x r) and outputs
  for (int e = tid; e < k * r; e += LT) {
    const int a = e / r, i = e % r;
    double u = 0.0;
    if (i < m) {
      const double* si = S + (size_t)i * k;
      for (int c = 0; c < m; ++c) u = fma(Q[(size_t)c * kq + a], si[c], u);
    }
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

size_t lanczos_smem_bytes(int kmax) {
  return ((size_t)kmax * kmax + (size_t)kmax * (kmax | 1) + (size_t)kmax * RMAX) * sizeof(double);
}

int launch_lanczos_smem(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r,
                        const double* A, double* U, double* lam, double* estimates, double* gof,
                        mdsx_piece_status* status, int qform_trivial, cudaStream_t st) {
  if (npieces == 0) return MDSX_OK;
  const size_t smem = lanczos_smem_bytes(kmax);
  cudaFuncSetAttribute(lanczos_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mdsx::pre(h, st);
  lanczos_smem_kernel<<<npieces, LT, smem, st>>>(pd, r, A, U, lam, estimates, gof, status,
                                                 qform_trivial);
  return launched(h, "lanczos_smem_kernel", st);
}

}  // namespace mdsx
