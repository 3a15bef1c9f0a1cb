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
#include "points_stream.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

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
constexpr int QCAP_PIECES = 48;  // Krylov basis capacity for plan pieces (2 CTAs / SM)
constexpr int CHECK_EVERY = 4;
#ifdef MDSX_LZ_PROF
#define LZT(v) long long v = clock64()
#else
#define LZT(v)
#endif
__device__ __forceinline__ int sturm_scaled(const double* as, const double* bs, int m, double x);
__device__ __noinline__ void tw_charpoly(const double* as, const double* bs, const double* ar,
                                         const double* br, const double* bq, int m, double th,
                                         double* zc, double* Dc, double* Uc, bool act, int sl,
                                         int src0, double& gamma, double& nrm2);

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

// index of the stored upper tile (I, J), I <= J, of an nbk x nbk block grid
__device__ __forceinline__ int lz_tile(int I, int J, int nbk) {
  return I * nbk - (I * (I - 1)) / 2 + (J - I);
}

// three sums over the CTA at once (fixed order), results in every thread
__device__ void block_sum3(double (&v)[3], double* red3) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < 3; ++c) v[c] = mdsx::warp_sum(v[c]);
  if (lane == 0)
#pragma unroll
    for (int c = 0; c < 3; ++c) red3[c * (LT / 32) + warp] = v[c];
  __syncthreads();
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    double s = 0.0;
    for (int w = 0; w < LT / 32; ++w) s += red3[c * (LT / 32) + w];
    v[c] = s;
  }
  __syncthreads();
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

template <typename T>
__device__ __noinline__ void lz_points(const PtsEpi& epi, const PieceDesc& d, int r,
                                       const double* Uout, unsigned char* smem) {
  auto go = [&](auto rm) {
    constexpr int RM = decltype(rm)::value;
    mdsx::PieceStream<T, RM> ps(smem, (const T*)epi.X, epi.ld, epi.row_idx + d.row_off, epi.p, d.m);
    ps.prologue();
    mdsx::ps_load_records<RM>(smem, Uout + d.u_off, epi.mu + (int64_t)d.id * epi.p, epi.p, r);
    __syncthreads();
    ps.run(smem, r, epi.points + d.pt_off * r);
  };
  if (r <= 4) go(std::integral_constant<int, 4>{});
  else if (r <= 8) go(std::integral_constant<int, 8>{});
  else go(std::integral_constant<int, 10>{});
}

// The Lanczos solve of piece `pidx` by the calling CTA (LT threads); `sm` is
// the dynamic shared memory (lanczos_bytes).
template <int QMAX>
__device__ __forceinline__ void lanczos_piece(const PieceDesc* __restrict__ pd, int pidx, int r,
                                              const double* __restrict__ Aall,
                                              double* __restrict__ Uout, double* __restrict__ lam_out,
                                              double* __restrict__ estimates, double* __restrict__ gof,
                                              mdsx_piece_status* __restrict__ status, int only_flagged,
                                              const PtsEpi& epi, int getenv_first_check, double* sm) {
  __shared__ double alpha[QMAX], beta[QMAX], beta2[QMAX];
  __shared__ double wv[LMAX], hv[QMAX + 1];
  __shared__ double theta[RMAX], lo_s[RMAX], hi_s[RMAX], thp[RMAX], rhp[RMAX], res_s[RMAX];
  __shared__ double as_[QMAX + 8], bs_[QMAX + 8], bq_[QMAX + 8], ar_[QMAX + 8], br_[QMAX + 8];
  __shared__ double gl_s, gu_s;
  __shared__ int rounds_s;
  __shared__ double red[LT / 32], red3[3 * (LT / 32)];
  __shared__ double trace_s, anorm_s;
  __shared__ int conv_s;

  const PieceDesc d = pd[pidx];
  const int pid = d.id, k = d.k;
  const int kq = (8 * ((k + 7) >> 3)) | 1;    // odd leading dim of Q, >= the tiled width (zero rows past k)
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
    if (epi.pending && tid == 0) epi.pending[pid] = 1;
    for (int e = tid; e < k * r; e += LT) Uout[d.u_off + e] = 0.0;
    if (tid < r) {
      estimates[(int64_t)pid * r + tid] = 0.0;
      lam_out[(int64_t)pid * r + tid] = 0.0;
    }
    if (tid < 2) gof[2 * (int64_t)pid + tid] = 0.0;
    return;
  }
  // A in 8x8 tiles of its upper block triangle: tile (I, J), I <= J < nbk, at
  // At + 64 * tidx(I, J), row-major inside the tile, zero-padded past k
  // (diagonal tiles hold both triangles).  One LDS.128 per lane reads a whole
  // tile, and the matvec needs no per-element index arithmetic.
  const int nbk = (k + 7) >> 3;
  const int ntile = nbk * (nbk + 1) / 2;
  double* At = sm;
  double* Q = At + (size_t)64 * ntile;         // column j at Q + j*kq, j < QMAX
  double* S = Q + (size_t)QMAX * kq;           // Ritz coefficients, S[c*RMAX + i]
  double* U2 = S + (size_t)QMAX * RMAX;        // twisted-factorisation pivots, same layout
  double* U3 = U2 + (size_t)QMAX * RMAX;
  const int qcap = min(QMAX, k);

  double fro = 0.0, tr = 0.0;
  for (int e = tid; e < 64 * ntile; e += LT) At[e] = 0.0;
  for (int e = tid; e < QMAX * kq; e += LT) Q[e] = 0.0;     // rows past k stay zero
  __syncthreads();
  if ((k & 1) == 0 && (reinterpret_cast<uintptr_t>(Ag) & 15) == 0) {
    // tiled copy, 16-byte loads, 8 in flight per thread (the matrix is read once
    // per piece; with 4 scalar loads in flight this phase was ~6% of the kernel)
    const int kk2 = k * k;
    const double2* Ag2 = reinterpret_cast<const double2*>(Ag);
    for (int e0 = tid; 2 * e0 < kk2; e0 += 8 * LT) {
      double2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * LT;
        v[u] = 2 * e < kk2 ? Ag2[e] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = 2 * (e0 + u * LT);
        if (e < kk2) {
          const int i = e / k, a = e - i * k;              // a even: a, a + 1 share the row
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double val = h ? v[u].y : v[u].x;
            const int ah = a + h;
            const int I = i >> 3, J = ah >> 3;
            if (I <= J) At[64 * lz_tile(I, J, nbk) + 8 * (i & 7) + (ah & 7)] = val;
            if (ah >= i) {
              fro = fma((ah == i ? 1.0 : 2.0) * val, val, fro);
              if (ah == i) tr += val;
            }
          }
        }
      }
    }
  } else {                                     // tiled copy: 4 independent loads in flight
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
          const int I = i >> 3, J = a >> 3;
          if (I <= J) At[64 * lz_tile(I, J, nbk) + 8 * (i & 7) + (a & 7)] = v[u];
          if (a >= i) {
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
  bool done = false, broke = false, capped = false, have_prev = false;
  // first check at 28 (r = 10): measured on dc2 / fast3, a check (~30k cycles) costs about
  // as much as four steps, and about half the pieces are not converged at 24
  const int first_check = getenv_first_check > 0 ? getenv_first_check : max(2 * r + 8, 28);
#ifdef MDSX_LZ_PROF
  long long lzp[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  LZ_T0(t_all);
#endif
  while (!done) {
    const double* q = Q + (size_t)m * kq;
    LZ_T0(t_mv);
    // w = A q over the tiles: warp w owns block rows I = w, w + 8; lane (i =
    // lane / 4, c = lane % 4) reads A_IJ[i][2c..2c+1] of the stored tile (I, J)
    // (J >= I: direct, y_I[i] += A_IJ[i][.] q_J[.]) or of tile (J, I) (J < I:
    // transposed, y_I[2c+v] += A_JI[i][2c+v] q_J[i]); both partial sums stay
    // in registers over the block row and are reduced once (4 and 8 lanes).
    {
      const int lane = tid & 31, warp = tid >> 5;
      const int ti = lane >> 2, tc = lane & 3;
      for (int I = warp; I < nbk; I += LT / 32) {
        double dsum = 0.0, t0 = 0.0, t1 = 0.0;
        const int lofs = 8 * ti + 2 * tc;
        // transposed part, J < I: tile (J, I); its index grows by nbk - J - 1 per J
        const double* tp = At + 64 * (I) + lofs;           // tile (0, I)
#pragma unroll 4
        for (int J = 0; J < I; ++J) {
          const double2 a2 = *reinterpret_cast<const double2*>(tp);
          const double qi = q[8 * J + ti];
          t0 = fma(a2.x, qi, t0);
          t1 = fma(a2.y, qi, t1);
          tp += 64 * (nbk - J - 1);
        }
        // direct part, J >= I: tiles (I, I), (I, I+1), ... are consecutive
        const double* dp = At + 64 * lz_tile(I, I, nbk) + lofs;
        const double* qd = q + 8 * I + 2 * tc;
#pragma unroll 4
        for (int J = I; J < nbk; ++J) {
          const double2 a2 = *reinterpret_cast<const double2*>(dp);
          dsum = fma(a2.x, qd[0], dsum);
          dsum = fma(a2.y, qd[1], dsum);
          dp += 64;
          qd += 8;
        }
        dsum += __shfl_xor_sync(0xffffffffu, dsum, 1);
        dsum += __shfl_xor_sync(0xffffffffu, dsum, 2);
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          t0 += __shfl_xor_sync(0xffffffffu, t0, o);
          t1 += __shfl_xor_sync(0xffffffffu, t1, o);
        }
        // lane (ti, 0) owns row 8I + ti of the direct part; lane (0, tc) rows 8I + 2tc, +1
        // of the transposed part: gather both into row-owner lanes, one store each
        const double tt0 = __shfl_sync(0xffffffffu, t0, (ti >> 1) & 3);   // lane (0, ti/2)
        const double tt1 = __shfl_sync(0xffffffffu, t1, (ti >> 1) & 3);
        if (tc == 0 && 8 * I + ti < k) wv[8 * I + ti] = dsum + ((ti & 1) ? tt1 : tt0);
      }
    }
    __syncthreads();
    LZ_ACC(0, t_mv);
    LZ_T0(t_cgs);
    // three-term part first (alpha = q_j.y, gamma = q_{j-1}.y, |y|^2 in one
    // reduction), then ONE classical Gram-Schmidt pass against Q[:, 0..m];
    // a second pass only when the first removed more than half of the norm
    // (DGKS, "twice is enough") or the three-term estimate is unreliable.
    // Barriers: partial sums (1), w (1), CGS coefficients (1), projected w and
    // its norm (1), next basis vector (1); each reduction buffer is written
    // once per step, so one barrier per reduction suffices.
    const int lane = tid & 31, wrp = tid >> 5;
    double al, nw0;
    {
      const double yv = tid < k ? wv[tid] : 0.0;
      const double qv = tid < k ? q[tid] : 0.0;
      const double pv = (tid < k && m > 0) ? Q[(size_t)(m - 1) * kq + tid] : 0.0;
      double s3[3] = {qv * yv, pv * yv, yv * yv};
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        s3[c] = mdsx::warp_sum(s3[c]);
        if (lane == 0) red3[c * (LT / 32) + wrp] = s3[c];
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        double t = 0.0;
        for (int w2 = 0; w2 < LT / 32; ++w2) t += red3[c * (LT / 32) + w2];   // fixed order
        s3[c] = t;
      }
      al = s3[0];
      const double ga = s3[1];
      nw0 = s3[2] - al * al - ga * ga;
      if (!(nw0 > 1e-4 * s3[2])) nw0 = 1e308;        // cancellation: force the second pass
      if (tid < k) wv[tid] = fma(-al, qv, fma(-ga, pv, yv));
      __syncthreads();
    }
    // one CGS pass: coefficients h = Q^T w (4 threads per column), then
    // w -= Q h by row pairs with the squared norm of the result reduced in the
    // same phase; the row owner keeps its projected entry in wreg
    const int nc = m + 1;
    double wreg = 0.0, nw = 0.0;
    for (int pass = 0; pass < 2; ++pass) {
      {
        // 8 threads per column (k split in 8 contiguous parts), 3-level shuffle
        const int part = tid & 7;
        const int seg = (k + 7) >> 3;
        for (int c = tid >> 3; c < ((nc + 3) & ~3); c += LT / 8) {     // warp-uniform trip count
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
          h += __shfl_xor_sync(0xffffffffu, h, 4);
          if (c < nc && part == 0) hv[c] = h;
        }
      }
      __syncthreads();
      al += hv[m];
      {
        const int hf = tid & 1;
        const int cmid = (nc + 1) >> 1;
        double sq = 0.0;
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
          if (a < k && hf == 0) {
            wreg = wv[a] - t;                        // LT / 2 >= k: one row per pair
            sq = wreg * wreg;
          }
        }
        sq = mdsx::warp_sum(sq);
        if (lane == 0) red[wrp] = sq;
        // the projected entries go back to wv only after everyone has read the
        // old ones (the barrier below): kept in wreg meanwhile
        __syncthreads();
        nw = 0.0;
        for (int w2 = 0; w2 < LT / 32; ++w2) nw += red[w2];                  // fixed order
        if ((tid >> 1) < k && (tid & 1) == 0) wv[tid >> 1] = wreg;
      }
      if (!(nw < 0.5 * nw0) || pass == 1) break;
      __syncthreads();                              // second pass reads the new wv
    }
    LZ_ACC(1, t_cgs);
    LZ_T0(t_b);
    const double b = sqrt(nw);
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
        if ((tid >> 1) < k && (tid & 1) == 0) Q[(size_t)m * kq + (tid >> 1)] = wreg / b;
      } else {
        // invariant subspace: continue from a fresh direction orthogonal to Q
        // (finds further copies of repeated eigenvalues)
        broke = true;
        __syncthreads();
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
    // ---- top-r eigenpairs of T_m: all 256 threads, one half-warp (MS = 16
    // lanes) per eigenvalue.  Division-free passes on an exactly scaled copy
    // of T (sturm_scaled, tw_charpoly), brackets from the previous check
    // (Cauchy interlacing lower bound, verified upper guess), 16-way
    // multisection to 1e-7 of the Gershgorin width, one Rayleigh-quotient
    // step from the twisted factorisation, eigenvectors and residuals from a
    // second twisted pass.  Clusters / a quotient outside its bracket: full
    // precision multisection from Gershgorin.
    const int rr = r < m ? r : m;
    if (tid < 32) {
      double gl = 1e308, gu = -1e308;
      for (int i = tid; i < m; i += 32) {
        const double off = (i > 0 ? fabs(beta[i - 1]) : 0.0) + (i + 1 < m ? fabs(beta[i]) : 0.0);
        gl = fmin(gl, alpha[i] - off);
        gu = fmax(gu, alpha[i] + off);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
        gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
      }
      if (tid == 0) { gl_s = gl; gu_s = gu; }
    }
    __syncthreads();
    int ex;
    frexp(fmax(fmax(fabs(gl_s), fabs(gu_s)), 1e-300), &ex);
    const double isc = ldexp(1.0, -ex), sc = ldexp(1.0, ex);
    for (int i = tid; i < m + 4; i += LT) {
      as_[i] = i < m ? alpha[i] * isc : 0.0;
      bs_[i] = (i > 0 && i < m) ? fmax(beta2[i - 1] * isc * isc, 1e-300) : 0.0;
      bq_[i] = i + 1 < m ? beta[i] * isc : 0.0;
      ar_[i] = i < m ? alpha[m - 1 - i] * isc : 0.0;
      br_[i] = (i > 0 && i < m) ? fmax(beta2[m - 1 - i] * isc * isc, 1e-300) : 0.0;
    }
    if (tid == 0) rounds_s = 0;
    __syncthreads();
    const double gls = gl_s * isc, gus = gu_s * isc, gw = gus - gls;
    const int grp = tid / MS, sl = tid % MS;
    const bool active = grp < rr;
    const int gbase = threadIdx.x & 16;                  // group's first lane in the warp
    constexpr double RS = 1.0 / (MS + 1);
    double lo = gls, hi = gus;
    if (have_prev) {
      const double tp = active ? thp[grp] * isc : 0.0, rp = active ? rhp[grp] * isc : 0.0;
      const double lo2 = tp - 1e-14 * gw, hi2 = fmin(gus, tp + 2.0 * rp + 1e-12 * gw);
      const bool below = active && sl < 2 &&
                         sturm_scaled(as_, bs_, m, sl == 0 ? lo2 : hi2) <= m - 1 - grp;
      const unsigned bal = __ballot_sync(0xffffffffu, below);
      if (active) {
        if ((bal >> gbase) & 1u) lo = lo2;               // theta_grp >= lo2
        if (!((bal >> (gbase + 1)) & 1u)) hi = hi2;      // theta_grp < hi2
        if (!(lo < hi)) { lo = gls; hi = gus; }
      }
    }
    auto msect = [&](int rounds) {
      for (int it = 0; it < rounds; ++it) {
        const double x = lo + (hi - lo) * ((double)(sl + 1) * RS);
        const int cntb = sturm_scaled(as_, bs_, m, x);          // all threads (uniform)
        const bool below_ok = active && cntb <= m - 1 - grp;
        const unsigned okm = __ballot_sync(0xffffffffu, below_ok);
        const int c = __popc((okm >> gbase) & 0xFFFFu);
        if (active) {
          const double lo0 = lo, w = hi - lo;
          lo = c > 0 ? lo0 + w * ((double)c * RS) : lo0;
          hi = c < MS ? lo0 + w * ((double)(c + 1) * RS) : hi;
        }
      }
    };
    auto rounds_to = [&](double target) {               // CTA-uniform round count
      int n = 0;
      for (double w = active ? hi - lo : 0.0; w > target * gw && n < 200; w *= RS) ++n;
      n = __reduce_max_sync(0xffffffffu, n);
      if ((threadIdx.x & 31) == 0) atomicMax(&rounds_s, n);
      __syncthreads();
      const int nr = rounds_s;
      __syncthreads();
      if (tid == 0) rounds_s = 0;
      return nr;
    };
    LZ_T0(t_ms6);
    msect(rounds_to(1e-7));
    LZ_ACC(5, t_ms6);
    LZ_T0(t_rq);
    int bad = 0;
    {
      double gam, n2;
      const double t0 = 0.5 * (lo + hi);
      tw_charpoly(as_, bs_, ar_, br_, bq_, m, t0, S + grp, U2 + grp, U3 + grp, active, sl, gbase,
                  gam, n2);
      const double t1 = t0 + gam / n2;
      if (active && sl == 0) {
        if (t1 >= lo && t1 <= hi) theta[grp] = t1;
        else bad = 1;
        lo_s[grp] = lo;
        hi_s[grp] = hi;
      }
    }
    __syncthreads();
    if (active && sl == 0 && grp + 1 < rr && !(hi_s[grp + 1] < lo_s[grp])) bad = 1;   // cluster
    const int any_bad = __syncthreads_or(bad);
    LZ_ACC(6, t_rq);
    if (any_bad) {
      lo = gls;
      hi = gus;
      msect(rounds_to(1e-17));
      if (active && sl == 0) theta[grp] = 0.5 * (lo + hi);
    }
    __syncthreads();
    {
      double gam, n2;
      const double tq = active ? theta[grp] : 0.0;
      tw_charpoly(as_, bs_, ar_, br_, bq_, m, tq, S + grp, U2 + grp, U3 + grp, active, sl, gbase,
                  gam, n2);
      if (active && sl == 0) {
        const double inv = 1.0 / sqrt(n2);
        const double bm = full ? 0.0 : beta[m - 1];
        res_s[grp] = fabs(bm * S[(m - 1) * RMAX + grp]) * inv;
        for (int c = 0; c < m; ++c) S[c * RMAX + grp] *= inv;
        theta[grp] = tq * sc;
      }
    }
    __syncthreads();
    if (active && sl == 0) { thp[grp] = theta[grp]; rhp[grp] = res_s[grp]; }
    have_prev = !any_bad;
    LZ_ACC(3, t_ck);
    LZ_T0(t_mgs);
    if (tid == 0) {
      int ok = rr == r;
      for (int i = 0; i < rr && ok; ++i)
        if (!(res_s[i] <= 1e-12 * fabs(theta[0]))) ok = 0;
      conv_s = ok || full ? 1 : (capped ? 2 : 0);
    }
    __syncthreads();
    done = conv_s != 0;
    if (conv_s == 1) {
      // clusters are runs of adjacent Ritz values (theta is descending): MGS
      // inside eigenvalue clusters only (fixed order, warp 0)
      const int adj = tid >= 1 && tid < rr && fabs(theta[tid - 1] - theta[tid]) <= 1e-3 * fabs(theta[0]);
      if (__syncthreads_or(adj) && tid < 32) {
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
    }
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
    if (epi.pending && tid == 0) epi.pending[pid] = 1;
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
  if (epi.points) {
    // points epilogue: the CTA streams its piece's rows while the SM's other
    // CTA is (typically) still in its latency-bound Krylov phase
    __syncthreads();                          // U in global (L1-hot), A / Q smem free
    if (tid == 0) epi.pending[pid] = 0;
    if (epi.f32) lz_points<float>(epi, d, r, Uout, reinterpret_cast<unsigned char*>(sm));
    else lz_points<double>(epi, d, r, Uout, reinterpret_cast<unsigned char*>(sm));
  }
}

template <int QMAX>
__global__ void __launch_bounds__(LT, QMAX <= QCAP_PIECES ? 2 : 1)
lanczos_smem_kernel(const PieceDesc* __restrict__ pd, int r, const double* __restrict__ Aall,
                    double* __restrict__ Uout, double* __restrict__ lam_out,
                    double* __restrict__ estimates, double* __restrict__ gof,
                    mdsx_piece_status* __restrict__ status, int only_flagged, const PtsEpi epi,
                    int getenv_first_check) {
  extern __shared__ double sm[];
  lanczos_piece<QMAX>(pd, blockIdx.x, r, Aall, Uout, lam_out, estimates, gof, status, only_flagged,
                      epi, getenv_first_check, sm);
}



// ---------------------------------------------------------------------------
// Tridiagonal helpers of the convergence checks (declared at the top).
// Branch-free reciprocal (MUFU seed + two Newton steps, ~1 ulp): unlike the
// IEEE division it has no slow-path branch, so independent reciprocals
// overlap with the recurrences instead of serialising them.
__device__ __forceinline__ double rcp_nr(double d) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
  double e = fma(-d, r, 1.0);
  r = fma(r, e, r);
  e = fma(-d, r, 1.0);
  return fma(r, e, r);
}

// Sturm count of the SCALED tridiagonal (as[i] = a_i / s, bs[i] = b_{i-1}^2 / s^2,
// bs[0] = 0, couplings >= 1e-300, |entries| <= 1) below x: the division-free
// leading-minor recurrence, one DFMA per step on the chain; the sign
// bookkeeping runs on the integer pipe (the fp64 pipe is shared with the
// stepper warps).  An exact zero minor needs no special case: with a nonzero
// coupling the next minor has the opposite sign of the previous one, so
// either sign of the zero gives exactly one change.  Exact power-of-two
// rescale every four steps (growth is at most 3x per step after scaling).
// Whole chunks of four with no per-step branches: steps past m only feed the
// masked-out tail (the arrays are zero-padded).
__device__ __forceinline__ int sturm_scaled(const double* as, const double* bs, int m, double x) {
  double pm = 1.0, pc = as[0] - x;
  int cnt = __double2hiint(pc) < 0;
  for (int i0 = 1; i0 < m; i0 += 4) {
    double a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { a[u] = as[i0 + u] - x; b[u] = bs[i0 + u]; }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double pn = fma(a[u], pc, -b[u] * pm);
      const unsigned ch = (unsigned)(__double2hiint(pn) ^ __double2hiint(pc)) >> 31;
      cnt += (int)(ch & (unsigned)(i0 + u < m));
      pm = pc;
      pc = pn;
    }
    const int e = (__double2hiint(pc) >> 20) & 0x7ff;
    const double f = e > 1023 + 300 ? 0x1p-300 : (e < 1023 - 300 ? 0x1p300 : 1.0);
    pc *= f;
    pm *= f;
  }
  return cnt;
}

// Twisted factorisation of T - theta I (SCALED T) with the pivots taken as
// ratios of consecutive principal minors: the minors come from the
// division-free three-term recurrences (one DFMA per step on the chain,
// exact power-of-two rescaling) and the pivots d_i = p_{i+1} / p_i from
// branch-free reciprocals off the chain (a zero minor becomes -pivmin times
// its predecessor, LAPACK's pivmin rule).  Lane sl == 0 of the group runs the
// leading (LDL^T) pass over (as, bs) and lane sl == 1 the trailing (UDU^T)
// pass over the reversed copies (ar, br) through the SAME instruction stream
// (no divergence, no per-step branches); the twist k = argmin |gamma_k| is
// scanned by both lanes (halves); the vector outward from the twist (z_k = 1)
// goes to column zc (stride RMAX), upward by sl 0 and downward by sl 1, again
// in one instruction stream.  Returns gamma_k and |z|^2 on the sl == 0 lane:
// theta + gamma_k / |z|^2 is the Rayleigh quotient of z.  All lanes of the
// warp must call it.
#ifdef MDSX_LZ_PROF
__device__ long long sh_prof[4];
#endif
__device__ __noinline__ void tw_charpoly(const double* as, const double* bs, const double* ar, const double* br,
                           const double* bq, int m, double th, double* zc, double* Dc, double* Uc,
                           bool act, int sl, int src0, double& gamma, double& nrm2) {
  constexpr double PIVMIN = 1e-290;
  LZT(tw0);
  const bool mine = act && sl < 2;
  const bool fw = sl == 0;
  {
    // forward: row s of (as, bs) -> Dc[s];  backward: row s of the reversed
    // copies = row m-1-s -> Uc[m-1-s]
    const double* A = fw ? as : ar;
    const double* B = fw ? bs : br;
    double* P = fw ? Dc : Uc + (m - 1) * RMAX;
    const int stp = fw ? RMAX : -RMAX;
    double pm = 1.0, pc = A[0] - th;
    if (mine) P[0] = fabs(pc) < PIVMIN ? -PIVMIN : pc;
    for (int s0 = 1; s0 < m; s0 += 4) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { a[u] = A[s0 + u] - th; b[u] = B[s0 + u]; }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double pn = fma(a[u], pc, -b[u] * pm);
        const double den = pc != 0.0 ? pc : -PIVMIN * pm;
        const double dv = pn * rcp_nr(den);
        if (mine && s0 + u < m) P[(s0 + u) * stp] = fabs(dv) < PIVMIN ? -PIVMIN : dv;
        pm = pc;
        pc = pn;
      }
      const int e = (__double2hiint(pc) >> 20) & 0x7ff;
      const double f = e > 1023 + 300 ? 0x1p-300 : (e < 1023 - 300 ? 0x1p300 : 1.0);
      pc *= f;
      pm *= f;
    }
  }
  __syncwarp();
  LZT(tw1);
  // twist: argmin |gamma_i|, gamma_i = d_i + u_i - (a_i - theta); ties -> larger i
  int kt = -1;
  double best = 1e308, gk = 0.0;
  for (int i = m - 1 - (sl & 1); i >= 0; i -= 2) {  // all lanes (uniform); only sl 0/1 are used
    const double g = Dc[i * RMAX] + Uc[i * RMAX] - (as[i] - th);
    const bool take = mine && fabs(g) < best;
    best = take ? fabs(g) : best;
    gk = take ? g : gk;
    kt = take ? i : kt;
  }
  {
    const double best_o = __shfl_sync(0xffffffffu, best, src0 + 1);
    const double gk_o = __shfl_sync(0xffffffffu, gk, src0 + 1);
    const int kt_o = __shfl_sync(0xffffffffu, kt, src0 + 1);
    if (best_o < best || (best_o == best && kt_o > kt)) { best = best_o; gk = gk_o; kt = kt_o; }
  }
  kt = __shfl_sync(0xffffffffu, kt, src0);
  LZT(tw2);
  double part = 0.0;
  {
    // upward (sl 0): z_i = -(b_i / d_i) z_{i+1}, i = kt-1 .. 0;
    // downward (sl 1): z_i = -(b_{i-1} / u_i) z_{i-1}, i = kt+1 .. m-1
    const int cnt = mine ? (fw ? kt : m - 1 - kt) : 0;
    const int steps = __reduce_max_sync(0xffffffffu, cnt);
    const int sg = fw ? -1 : 1;
    const double* P = fw ? Dc : Uc;
    const double* Bq = fw ? bq : bq - 1;
    if (mine && fw) zc[kt * RMAX] = 1.0;
    double z = 1.0;
    for (int s0 = 1; s0 <= steps; s0 += 4) {      // ratios (reciprocals) off the product chain
      double f[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = min(max(kt + sg * (s0 + u), 0), m - 1);
        f[u] = -Bq[i + (fw ? 0 : (i == 0))] * rcp_nr(P[i * RMAX]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool ok = s0 + u <= cnt;
        z *= ok ? f[u] : 1.0;
        if (ok) zc[(kt + sg * (s0 + u)) * RMAX] = z;
        part = ok ? fma(z, z, part) : part;
      }
    }
  }
  const double other = __shfl_sync(0xffffffffu, part, src0 + 1);
  gamma = gk;
  nrm2 = 1.0 + part + other;
  __syncwarp();
#ifdef MDSX_LZ_PROF
  if (blockIdx.x == 0 && threadIdx.x == 224) {
    sh_prof[0] += tw1 - tw0; sh_prof[1] += tw2 - tw1; sh_prof[2] += clock64() - tw2;
  }
#endif
}


}  // namespace

namespace mdsx {

int lanczos_kmax() { return LMAX; }
int lanczos_rmax() { return RMAX; }

static size_t lanczos_bytes(int kmax, int qmax) {
  const size_t nbk = (size_t)(kmax + 7) / 8;
  return (64 * nbk * (nbk + 1) / 2 + (size_t)qmax * ((8 * nbk) | 1) + 3 * (size_t)qmax * RMAX) *
         sizeof(double);
}

size_t lanczos_smem_bytes(int kmax) { return lanczos_bytes(kmax, LMAX); }

// full_basis: Krylov capacity = LMAX (one CTA / SM, never flags -2; used for
// the Rayleigh-Ritz matrices of the block-Krylov solver); otherwise
// QCAP_PIECES (two CTAs / SM, capacity overflow -> Jacobi fallback).
int launch_lanczos_smem(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r,
                        const double* A, double* U, double* lam, double* estimates, double* gof,
                        mdsx_piece_status* status, int full_basis, int only_flagged,
                        cudaStream_t st, const PtsEpi* epi) {
  if (epi && (full_basis || only_flagged || r > 10)) epi = nullptr;
  if (npieces == 0) return MDSX_OK;
  PtsEpi e{};
  if (epi) e = *epi;
  auto go = [&](auto kern, int qmax) {
    size_t smem = lanczos_bytes(kmax, qmax);
    if (epi) smem = std::max(smem, mdsx::ps_smem_bytes<10>(epi->p));
    if (getenv("MDSX_LZ_ONE")) smem = std::max<size_t>(smem, 120 * 1024);   // experiment: 1 CTA/SM
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mdsx::pre(h, st);
    const char* fc = getenv("MDSX_LZ_FIRST");
    kern<<<npieces, LT, smem, st>>>(pd, r, A, U, lam, estimates, gof, status, only_flagged, e,
                                    fc ? atoi(fc) : 0);
    return launched(h, "lanczos_smem_kernel", st);
  };
  return full_basis ? go(lanczos_smem_kernel<LMAX>, LMAX)
                    : go(lanczos_smem_kernel<QCAP_PIECES>, QCAP_PIECES);
}


}  // namespace mdsx
