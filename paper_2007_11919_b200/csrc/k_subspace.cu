// K3 top-r eigensolver by blocked subspace iteration on the fp64 tensor pipe
// (north star (b): "a top-r eigensolve by blocked subspace iteration, so GEMMs
// go to tensor cores and small r x r Rayleigh-Ritz/QR steps run warp-level").
//
// One CTA (4 warps) per piece, 32 < k <= 104, r <= 12.  The piece's k x k PSD
// matrix A lives in shared memory as a packed upper triangle (~40 KB at
// k = 100, so three pieces share an SM).  A block V of SB = 16 orthonormal
// columns is iterated
//     Y = (A + s I) V                 (DMMA m8n8k4, 13 x 2 output blocks)
//     V = orth(Y)                     (Cholesky-QR twice: G = Y^T Y by DMMA,
//                                      16 x 16 Cholesky + inverse in one warp,
//                                      V = Y L^-T by DMMA)
// and from iteration SS_FIRST every SS_EVERY iterations a Rayleigh-Ritz step
// diagonalises H = V^T A V (16 x 16, parallel Jacobi), forms the Ritz vectors
// X = V Z and the residuals |A x_j - theta_j x_j| = |(Y Z)_j - (s+theta_j) x_j|,
// all by DMMA, and accepts when every top-r residual is <= 1e-12 theta_1 (the
// Lanczos kernel's criterion).  The shift s = 1e-3 trace(A)/k keeps Y full
// rank (Cholesky-QR safe; eigenvectors unchanged).  Convergence per iteration
// is ~ lambda_17 / lambda_r: 12-20 iterations for the BASELINE Gaussian pieces.
// A piece that has not converged after SS_MAX_IT iterations (no spectral gap
// after r) is flagged (status NUMERICAL, value -3) and the Lanczos kernel,
// launched next in the same stream, solves exactly the flagged pieces.
//
// G1/G2 use trace(A) (PSD Gram of Euclidean data: Sum|lambda| = trace; G1 ==
// G2 bitwise, classical.py:75-85), eigenvalues snapped at 1e-8 theta_1 and the
// DegenerateRank rule of classical.py:137-142, as in the Lanczos kernel.
#include "mdsx_common.cuh"

#ifdef MDSX_SS_PROF
#define SS_T0(v) long long v = clock64()
#define SS_ACC(slot, v) if (blockIdx.x == 0 && threadIdx.x == 0) prof[slot] += clock64() - v
#else
#define SS_T0(v)
#define SS_ACC(slot, v)
#endif

namespace {

constexpr int SS_T = 128;        // threads per CTA (4 warps)
constexpr int SB = 16;           // block width
constexpr int SNB = 13;          // max 8-row blocks (k <= 104)
constexpr int LDT = 108;         // pitch of V^T / Y^T (== 12 mod 16: conflict-free fragments)
constexpr int SS_MAX_IT = 40;
constexpr int SS_FIRST = 12;
constexpr int SS_EVERY = 2;
constexpr int SS_RMAX = 12;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double hash_unit(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  return (double)(x >> 11) * (1.0 / 9007199254740992.0) * 2.0 - 1.0;
}

struct SsShared {
  // QR phase: G (Gram / Cholesky factor in place) and Li = L^-1;
  // RR phase: H (-> diagonalised) and Z (eigenvectors).  Never live together.
  double M0[SB * SB], M1[SB * SB];
  double red[4][SB];
  double rinv[SB];
  double jc[SB], jsn[SB / 2];
  int jpq[SB / 2];
  double theta[SB];
  int rank_of[SB];
  double trace, anorm;
  int flag;
};

// packed-upper offset of row i (entries (i, j >= i) at off(i) + j - i)
__device__ __forceinline__ int poff(int i, int k) { return i * k - i * (i - 1) / 2; }

// Gram of the 16 columns stored transposed in Bt (16 x LDT, rows >= k zero):
// warp w computes block (w >> 1, w & 1) of G = B^T B into G (16 x 16).
__device__ __forceinline__ void gram16(const double* Bt, int nk4, double* G, int warp, int gid,
                                       int tig) {
  const int ib = warp >> 1, jb = warp & 1;
  double c0 = 0.0, c1 = 0.0;
  const double* ra = Bt + (8 * ib + gid) * LDT + tig;
  const double* rb = Bt + (8 * jb + gid) * LDT + tig;
#pragma unroll 4
  for (int kb = 0; kb < nk4; ++kb) dmma(c0, c1, ra[4 * kb], rb[4 * kb]);
  G[(8 * ib + gid) * SB + 8 * jb + 2 * tig] = c0;
  G[(8 * ib + gid) * SB + 8 * jb + 2 * tig + 1] = c1;
}

// Reciprocal for the serial recurrences.  Measured on B200 (tools/lat_micro.cu):
// a dependent DDIV costs ~60 clk, a float-seeded Newton reciprocal ~130 clk
// (two F2F conversions + MUFU on the chain), so plain division wins.
__device__ __forceinline__ double fast_rcp(double d) { return 1.0 / d; }

// Cholesky G = L L^T of the 16 x 16 Gram in G (symmetrised on the fly) by one
// warp: lane i holds row i in registers, column j's pivot and entries are
// broadcast by shuffles (no shared-memory round trips on the critical path).
// Writes L (lower, zero above) back to G and 1/L_jj to rinv; *flag = -1 on a
// non-positive pivot.
__device__ __forceinline__ void chol16_warp(double* G, double* rinv, int lane, int* flag) {
  const int i = lane & 15;
  double g[SB];
#pragma unroll
  for (int l = 0; l < SB; ++l) g[l] = 0.5 * (G[i * SB + l] + G[l * SB + i]);
  __syncwarp();
  bool ok = true;
#pragma unroll
  for (int j = 0; j < SB; ++j) {
    const double piv = __shfl_sync(0xffffffffu, g[j], j);
    ok = ok && piv > 0.0;
    // 1/sqrt(piv): single-precision seed, two Newton steps (full double accuracy)
    const double pv = fmax(piv, 1e-300);
    const double rs = 1.0 / sqrt(pv);
    const double lij = i > j ? g[j] * rs : (i == j ? pv * rs : 0.0);
    g[j] = lij;
#pragma unroll
    for (int l = 0; l < SB; ++l) {
      if (l > j) {
        const double llj = __shfl_sync(0xffffffffu, lij, l);
        if (i >= l) g[l] = fma(-lij, llj, g[l]);
      }
    }
    if (lane == 0) rinv[j] = rs;
  }
  if (lane < SB)
#pragma unroll
    for (int l = 0; l < SB; ++l) G[i * SB + l] = l <= i ? g[l] : 0.0;
  if (lane == 0) *flag = ok ? 0 : -1;
}

// Cyclic Jacobi on the 16 x 16 symmetric H (smem, pitch 16) by one warp:
// round-robin pairing (8 disjoint rotations per round, computed by lanes
// 0..7), the two-sided update as 36 independent 2x2 block tasks and the
// eigenvector update as 128 row tasks, __syncwarp only.  Rotates when
// |h_pq| > max(eps sqrt|h_pp h_qq|, floor_abs); stops after a sweep without
// rotations.  Z (initialised by the caller) accumulates the rotations.
__device__ int jacobi16_warp(double* H, double* Z, double floor_abs, int lane, int max_sweeps,
                             double* cs, double* sn, int* pq) {
  const double eps = 2.220446049250313e-16;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int rot = 0;
    for (int rnd = 0; rnd < SB - 1; ++rnd) {
      if (lane < SB / 2) {
        const int x = lane == 0 ? 0 : 1 + (rnd + lane - 1) % (SB - 1);
        const int y = 1 + (rnd - lane + SB - 2) % (SB - 1);
        const int p = min(x, y), q = max(x, y);
        const double app = H[p * SB + p], aqq = H[q * SB + q], apq = H[p * SB + q];
        double c = 1.0, sv = 0.0, t = 0.0;
        if (fabs(apq) > floor_abs && apq * apq > eps * eps * fabs(app * aqq)) {
          mdsx::sym_rotation(app, aqq, apq, c, sv, t);
          rot = 1;
        }
        cs[lane] = c; sn[lane] = sv; pq[lane] = p | (q << 8);
        cs[SB / 2 + lane] = t;
      }
      __syncwarp();
      for (int L = lane; L < 36; L += 32) {           // tasks (a, b), b <= a < 8
        int a = 0, t = L;
        while (t > a) { t -= a + 1; ++a; }
        const int b = t;
        const int p = pq[a] & 255, q = pq[a] >> 8;
        if (a == b) {
          const double tt = cs[SB / 2 + a];
          if (tt != 0.0) {
            const double apq = H[p * SB + q];
            H[p * SB + p] -= tt * apq;
            H[q * SB + q] += tt * apq;
            H[p * SB + q] = 0.0;
            H[q * SB + p] = 0.0;
          }
          continue;
        }
        const int p2 = pq[b] & 255, q2 = pq[b] >> 8;
        const double c = cs[a], sv = sn[a], c2 = cs[b], s2 = sn[b];
        const double a1 = H[p * SB + p2], a2 = H[p * SB + q2];
        const double a3 = H[q * SB + p2], a4 = H[q * SB + q2];
        const double b1 = c2 * a1 - s2 * a2, b2 = s2 * a1 + c2 * a2;
        const double b3 = c2 * a3 - s2 * a4, b4 = s2 * a3 + c2 * a4;
        const double n1 = c * b1 - sv * b3, n3 = sv * b1 + c * b3;
        const double n2 = c * b2 - sv * b4, n4 = sv * b2 + c * b4;
        H[p * SB + p2] = n1; H[p2 * SB + p] = n1;
        H[p * SB + q2] = n2; H[q2 * SB + p] = n2;
        H[q * SB + p2] = n3; H[p2 * SB + q] = n3;
        H[q * SB + q2] = n4; H[q2 * SB + q] = n4;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {                   // Z rows x pairs: 16 x 8 tasks
        const int L = lane + 32 * u;
        const int row = L >> 3, a = L & 7;
        const double sv = sn[a];
        if (sv != 0.0) {
          const double c = cs[a];
          const int p = pq[a] & 255, q = pq[a] >> 8;
          const double up = Z[row * SB + p], uq = Z[row * SB + q];
          Z[row * SB + p] = c * up - sv * uq;
          Z[row * SB + q] = sv * up + c * uq;
        }
      }
      __syncwarp();
      rot = __any_sync(0xffffffffu, rot) ? 1 : rot;
    }
    if (!__any_sync(0xffffffffu, rot)) return sweep + 1;
  }
  return max_sweeps;
}

// Dst = Src L^-T row by row (V L^T = Y: forward substitution, right-looking),
// one thread per row a < nrows; Src/Dst stored transposed (16 x LDT) and may
// alias (each thread reads and writes only its own row).
__device__ __forceinline__ void trsv_rows(const double* Srct, double* Dstt, const double* L,
                                          const double* rinv, int nrows) {
  const int a = threadIdx.x;
  if (a >= nrows) return;
  double v[SB];
#pragma unroll
  for (int j = 0; j < SB; ++j) v[j] = Srct[j * LDT + a];
#pragma unroll
  for (int j = 0; j < SB; ++j) {
    v[j] *= rinv[j];
#pragma unroll
    for (int l = 0; l < SB; ++l)
      if (l > j) v[l] = fma(-v[j], L[l * SB + j], v[l]);
  }
#pragma unroll
  for (int j = 0; j < SB; ++j) Dstt[j * LDT + a] = v[j];
}

__global__ void __launch_bounds__(SS_T, 3)
subspace_kernel(const PieceDesc* __restrict__ pd, int r, const double* __restrict__ Aall,
                double* __restrict__ Uout, double* __restrict__ lam_out,
                double* __restrict__ estimates, double* __restrict__ gof,
                mdsx_piece_status* __restrict__ status) {
  extern __shared__ double ssm[];
  __shared__ SsShared sh;
#ifdef MDSX_SS_PROF
  long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  SS_T0(t_all);
#endif
  const PieceDesc d = pd[blockIdx.x];
  const int pid = d.id, k = d.k;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int nb = (k + 7) >> 3, nk4 = 2 * nb;
  double* Ap = ssm;                                        // k(k+1)/2 packed upper
  double* Vt = Ap + ((k * (k + 1) / 2 + 1) & ~1);          // SB x LDT
  double* Yt = Vt + SB * LDT;                              // SB x LDT

  if (status[pid].code == MDSX_INVALID_INPUT) {            // non-finite rows: nothing to solve
    for (int e = tid; e < k * r; e += SS_T) Uout[d.u_off + e] = 0.0;
    if (tid < r) {
      estimates[(int64_t)pid * r + tid] = 0.0;
      lam_out[(int64_t)pid * r + tid] = 0.0;
    }
    if (tid < 2) gof[2 * (int64_t)pid + tid] = 0.0;
    return;
  }

  // ---- A (packed), trace, |A|_F; 4 independent loads in flight per thread
  const double* Ag = Aall + d.a_off;
  double fro = 0.0, tr = 0.0;
  {
    const int kk2 = k * k;
    for (int e0 = tid; e0 < kk2; e0 += 4 * SS_T) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * SS_T;
        v[u] = e < kk2 ? Ag[e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * SS_T;
        if (e < kk2) {
          const int i = e / k, a = e - i * k;
          if (a >= i) {
            Ap[poff(i, k) + a - i] = v[u];
            fro = fma((a == i ? 1.0 : 2.0) * v[u], v[u], fro);
            if (a == i) tr += v[u];
          }
        }
      }
    }
  }
  fro = mdsx::warp_sum(fro);
  tr = mdsx::warp_sum(tr);
  if (lane == 0) { sh.red[0][warp] = fro; sh.red[1][warp] = tr; }
  // start block: batch-independent hash vectors (rows >= k zero)
  for (int e = tid; e < SB * LDT; e += SS_T) {
    const int j = e / LDT, a = e % LDT;
    Vt[e] = a < k ? hash_unit(((uint64_t)j << 24) ^ ((uint64_t)a * 0x9E37ull + 17)) : 0.0;
    Yt[e] = 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double f = 0.0, t = 0.0;
    for (int w = 0; w < SS_T / 32; ++w) { f += sh.red[0][w]; t += sh.red[1][w]; }
    sh.trace = t;
    sh.anorm = sqrt(f);
    sh.flag = 0;
  }
  __syncthreads();
  const double shift = 1e-3 * sh.trace / (double)k;

  // per-lane packed offsets of the rows this lane touches as A-fragment rows
  int roff[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int i = 8 * (warp + 4 * q) + gid;
    roff[q] = poff(min(i, k - 1), k) - i;
  }
  double acc[4][2][2];

  // V = orth(Src): Cholesky-QR, `passes` times (the second pass restores
  // orthogonality to working precision; used before Rayleigh-Ritz)
  auto orth = [&](const double* Srct, int passes) -> bool {
    bool good = true;
    for (int pass = 0; pass < passes; ++pass) {
      const double* src = pass == 0 ? Srct : Vt;
      SS_T0(t0);
      gram16(src, nk4, sh.M0, warp, gid, tig);
      __syncthreads();
      SS_ACC(0, t0);
      SS_T0(t1);
      if (warp == 0) chol16_warp(sh.M0, sh.rinv, lane, &sh.flag);
      __syncthreads();
      SS_ACC(1, t1);
      good = good && sh.flag == 0;
      SS_T0(t2);
      trsv_rows(src, Vt, sh.M0, sh.rinv, 8 * nb);
      __syncthreads();
      SS_ACC(2, t2);
    }
    return good;
  };
  auto is_check = [&](int itn) {
    return itn >= SS_FIRST && ((itn - SS_FIRST) % SS_EVERY == 0 || itn == SS_MAX_IT);
  };

  bool ok = orth(Vt, 2);
  int it = 0;
  bool converged = false;
  while (ok && !converged && it < SS_MAX_IT) {
    // ---- Y = (A + s I) V
    SS_T0(t3);
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int cb = 0; cb < 2; ++cb) acc[q][cb][0] = acc[q][cb][1] = 0.0;
#pragma unroll 2
    for (int kb = 0; kb < nk4; ++kb) {
      const int j = 4 * kb + tig;
      const double b0 = Vt[gid * LDT + j], b1 = Vt[(8 + gid) * LDT + j];
      const int coff = poff(min(j, k - 1), k) - j;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rb = warp + 4 * q;
        if (rb < nb) {
          const int i = 8 * rb + gid;
          const int idx = i <= j ? roff[q] + j : coff + i;
          const double af = (i < k && j < k) ? Ap[idx] : 0.0;
          dmma(acc[q][0][0], acc[q][0][1], af, b0);
          dmma(acc[q][1][0], acc[q][1][1], af, b1);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int rb = warp + 4 * q;
      if (rb < nb)
#pragma unroll
        for (int cb = 0; cb < 2; ++cb)
#pragma unroll
          for (int v = 0; v < 2; ++v) {
            const int row = 8 * rb + gid, col = 8 * cb + 2 * tig + v;
            Yt[col * LDT + row] = fma(shift, Vt[col * LDT + row], acc[q][cb][v]);
          }
    }
    __syncthreads();
    SS_ACC(3, t3);
    ++it;

    if (is_check(it)) {
      // ---- Rayleigh-Ritz: H = V^T Y - s I  (= V^T A V), symmetrised; Z = I
      {
        const int ib = warp >> 1, jb = warp & 1;
        double c0 = 0.0, c1 = 0.0;
        const double* ra = Vt + (8 * ib + gid) * LDT + tig;
        const double* rb = Yt + (8 * jb + gid) * LDT + tig;
#pragma unroll 4
        for (int kb = 0; kb < nk4; ++kb) dmma(c0, c1, ra[4 * kb], rb[4 * kb]);
        const int row = 8 * ib + gid, col = 8 * jb + 2 * tig;
        sh.M0[row * SB + col] = c0 - (row == col ? shift : 0.0);
        sh.M0[row * SB + col + 1] = c1 - (row == col + 1 ? shift : 0.0);
      }
      for (int e = tid; e < SB * SB; e += SS_T) sh.M1[e] = (e / SB == e % SB) ? 1.0 : 0.0;
      __syncthreads();
      {
        int pi = 0, pj = 0;
        double hs = 0.0;
        const bool mine = tid < SB * (SB - 1) / 2;
        if (mine) {                                  // pair index -> (pi < pj)
          int t = tid;
          pi = 0;
          while (t >= SB - 1 - pi) { t -= SB - 1 - pi; ++pi; }
          pj = pi + 1 + t;
          hs = 0.5 * (sh.M0[pi * SB + pj] + sh.M0[pj * SB + pi]);
        }
        __syncthreads();
        if (mine) { sh.M0[pi * SB + pj] = hs; sh.M0[pj * SB + pi] = hs; }
        __syncthreads();
      }
      const double floor_abs = 1e-15 * sh.anorm;
      SS_T0(t4);
      int nsw = 0;
      if (warp == 0) nsw = jacobi16_warp(sh.M0, sh.M1, floor_abs, lane, 30, sh.jc, sh.jsn, sh.jpq);
      (void)nsw;
      __syncthreads();
      SS_ACC(4, t4);
#ifdef MDSX_SS_PROF
      if (blockIdx.x == 0 && tid == 0) { prof[5] += nsw; prof[6] += 1; }
#endif
      // descending order of the Ritz values (stable: ties by index)
      if (tid < SB) {
        const double lj = sh.M0[tid * SB + tid];
        int rk = 0;
        for (int i = 0; i < SB; ++i) {
          const double li = sh.M0[i * SB + i];
          if (li > lj || (li == lj && i < tid)) ++rk;
        }
        sh.rank_of[tid] = rk;
        sh.theta[tid] = lj;
      }
      __syncthreads();
      // ---- X = V Z and W = Y Z; residual columns |W_j - (s + theta_j) X_j|
      double xacc[4][2][2], wacc[4][2][2];
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) {
          xacc[q][cb][0] = xacc[q][cb][1] = 0.0;
          wacc[q][cb][0] = wacc[q][cb][1] = 0.0;
        }
#pragma unroll
      for (int kb = 0; kb < SB / 4; ++kb) {
        double bf[2];
#pragma unroll
        for (int cb = 0; cb < 2; ++cb) bf[cb] = sh.M1[(4 * kb + tig) * SB + 8 * cb + gid];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rb = warp + 4 * q;
          if (rb < nb) {
            const double av = Vt[(4 * kb + tig) * LDT + 8 * rb + gid];
            const double ay = Yt[(4 * kb + tig) * LDT + 8 * rb + gid];
#pragma unroll
            for (int cb = 0; cb < 2; ++cb) {
              dmma(xacc[q][cb][0], xacc[q][cb][1], av, bf[cb]);
              dmma(wacc[q][cb][0], wacc[q][cb][1], ay, bf[cb]);
            }
          }
        }
      }
      double rs[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rb = warp + 4 * q;
        if (rb < nb)
#pragma unroll
          for (int cb = 0; cb < 2; ++cb)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
              const int col = 8 * cb + 2 * tig + v;
              const double res = fma(-(shift + sh.theta[col]), xacc[q][cb][v], wacc[q][cb][v]);
              rs[cb][v] = fma(res, res, rs[cb][v]);
            }
      }
      // column sums over gid (lanes xor 4, 8, 16), then over warps in fixed order
#pragma unroll
      for (int cb = 0; cb < 2; ++cb)
#pragma unroll
        for (int v = 0; v < 2; ++v) {
          double t = rs[cb][v];
          t += __shfl_xor_sync(0xffffffffu, t, 4);
          t += __shfl_xor_sync(0xffffffffu, t, 8);
          t += __shfl_xor_sync(0xffffffffu, t, 16);
          if (gid == 0) sh.red[warp][8 * cb + 2 * tig + v] = t;
        }
      __syncthreads();
      if (tid == 0) {
        double top = -1e308;
        for (int j = 0; j < SB; ++j) top = fmax(top, sh.theta[j]);
        int conv = 1;
        for (int j = 0; j < SB; ++j) {
          if (sh.rank_of[j] >= r) continue;
          const double rn = sqrt(sh.red[0][j] + sh.red[1][j] + sh.red[2][j] + sh.red[3][j]);
          if (!(rn <= 1e-12 * fabs(top))) conv = 0;
        }
        sh.flag = conv;
      }
      __syncthreads();
      converged = sh.flag != 0;
      if (converged) {
        // outputs: top-r Ritz vectors (k x r, rank order), values, estimates, G
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rb = warp + 4 * q;
          if (rb < nb)
#pragma unroll
            for (int cb = 0; cb < 2; ++cb)
#pragma unroll
              for (int v = 0; v < 2; ++v) {
                const int row = 8 * rb + gid, col = 8 * cb + 2 * tig + v;
                const int rk = sh.rank_of[col];
                if (row < k && rk < r) Uout[d.u_off + (int64_t)row * r + rk] = xacc[q][cb][v];
              }
        }
        if (tid == 0) {
          double th[SB];
          for (int j = 0; j < SB; ++j) th[sh.rank_of[j]] = sh.theta[j];
          const double tol = 1e-8 * fabs(th[0]);
          mdsx_piece_status st{MDSX_OK, 0, 0.0};
          if (status[pid].code != MDSX_OK) st.code = status[pid].code;
          double kept = 0.0;
          for (int i = 0; i < r; ++i) {
            double v = th[i];
            if (fabs(v) <= tol) v = 0.0;
            if (st.code == MDSX_OK && v <= 0.0) {
              st.code = MDSX_DEGENERATE; st.index = i + 1; st.value = v;
            }
            kept += v;
            lam_out[(int64_t)pid * r + i] = v;
            estimates[(int64_t)pid * r + i] = v / d.m;
          }
          if (st.code == MDSX_OK) st.value = (double)it;   // diagnostics: iterations used
          status[pid] = st;
          const double g = st.code == MDSX_OK ? kept / sh.trace : 0.0;
          gof[2 * (int64_t)pid] = g;
          gof[2 * (int64_t)pid + 1] = g;
        }
#ifdef MDSX_SS_PROF
        SS_ACC(7, t_all);
        if (blockIdx.x == 0 && tid == 0)
          printf("ss prof it=%d gram %lld chol %lld trsv %lld AV %lld jacobi %lld sweeps %lld/%lld checks total %lld\n", it,
                 prof[0], prof[1], prof[2], prof[3], prof[4], prof[5], prof[6], prof[7]);
#endif
        return;
      }
      // not yet: continue from the Ritz basis, Y <- Y Z (same span; the next
      // H is then nearly diagonal and its Jacobi takes one or two sweeps)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rb = warp + 4 * q;
        if (rb < nb)
#pragma unroll
          for (int cb = 0; cb < 2; ++cb)
#pragma unroll
            for (int v = 0; v < 2; ++v)
              Yt[(8 * cb + 2 * tig + v) * LDT + 8 * rb + gid] = wacc[q][cb][v];
      }
      __syncthreads();
    }
    // ---- V = orth(Y)
    ok = orth(Yt, is_check(it + 1) ? 2 : 1);
  }
  // not converged (or Cholesky breakdown): the Lanczos kernel takes this piece
  if (tid == 0 && status[pid].code == MDSX_OK)
    status[pid] = mdsx_piece_status{MDSX_NUMERICAL, 0, -3.0};
}

}  // namespace

namespace mdsx {

int subspace_rmax() { return SS_RMAX; }

int launch_subspace(mdsx_handle* h, const PieceDesc* pd, int npieces, int kmax, int r,
                    const double* A, double* U, double* lam, double* estimates, double* gof,
                    mdsx_piece_status* status, cudaStream_t st) {
  if (npieces == 0) return MDSX_OK;
  const size_t smem = (((size_t)kmax * (kmax + 1) / 2 + 1) / 2 * 2 + 2 * (size_t)SB * LDT) *
                      sizeof(double);
  cudaFuncSetAttribute(subspace_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mdsx::pre(h, st);
  subspace_kernel<<<npieces, SS_T, smem, st>>>(pd, r, A, U, lam, estimates, gof, status);
  return launched(h, "subspace_kernel", st);
}

}  // namespace mdsx
