// Parallel-order cyclic Jacobi eigen-solver core for a symmetric k x k matrix
// held in shared memory (used by the per-piece solver and by the
// Rayleigh-Ritz step of the subspace solver).
#pragma once
#include "mdsx_common.cuh"

namespace mdsx {

struct JacobiShared {
  double cs[MDSX_JACOBI_KMAX / 2], sn[MDSX_JACOBI_KMAX / 2], tn[MDSX_JACOBI_KMAX / 2];
  int pp[MDSX_JACOBI_KMAX / 2], qq[MDSX_JACOBI_KMAX / 2];
  int nrot;
};

// A (kk x kk, row-major, rows/cols >= k zero) is diagonalised in place and
// the rotations accumulated into U (initialised by the caller).  Rounds pair
// the kk indices round-robin; each pair (p,q) is rotated when
// |a_pq| > max(eps sqrt|a_pp a_qq|, floor_abs) (relative criterion, plus an
// absolute floor ~1e-15 |A|_F, the round-off level of the rotations themselves).  The two-sided update of a round is a set of
// independent 2x2 block tasks.  Returns true when a sweep did no rotation.
__device__ inline bool jacobi_sweeps(double* A, double* U, int k, int kk, double floor_abs,
                                     JacobiShared& js, int max_sweeps) {
  const int tid = threadIdx.x, nt = blockDim.x, P = kk / 2;
  const double eps = 2.220446049250313e-16;
  double* cs = js.cs; double* sn = js.sn; double* tn = js.tn;
  int* pp = js.pp; int* qq = js.qq;
  int& nrot = js.nrot;
  int sweep = 0;
  bool converged = (k <= 1);
  for (; sweep < max_sweeps && !converged; ++sweep) {
    __syncthreads();
    if (tid == 0) nrot = 0;
    __syncthreads();
    for (int rnd = 0; rnd < kk - 1; ++rnd) {
      if (tid < P) {
        const int x = (tid == 0) ? 0 : 1 + (rnd + tid - 1) % (kk - 1);
        const int y = 1 + (rnd - tid + kk - 2) % (kk - 1);
        const int p_ = min(x, y), q_ = max(x, y);
        const double app = A[p_ * kk + p_], aqq = A[q_ * kk + q_], apq = A[p_ * kk + q_];
        double c = 1.0, s = 0.0, t = 0.0;
        if (fabs(apq) > fmax(eps * sqrt(fabs(app) * fabs(aqq)), floor_abs)) {
          mdsx::sym_rotation(app, aqq, apq, c, s, t);
          atomicAdd(&nrot, 1);
        }
        cs[tid] = c; sn[tid] = s; tn[tid] = t; pp[tid] = p_; qq[tid] = q_;
      }
      __syncthreads();
      for (int L = tid; L < P * P; L += nt) {
        const int i = L / P, i2 = L % P;
        if (i2 > i) continue;
        const int p = pp[i], q = qq[i];
        if (i == i2) {
          const double t = tn[i];
          if (t != 0.0) {
            const double apq = A[p * kk + q];
            A[p * kk + p] -= t * apq;
            A[q * kk + q] += t * apq;
            A[p * kk + q] = 0.0;
            A[q * kk + p] = 0.0;
          }
          continue;
        }
        const int p2 = pp[i2], q2 = qq[i2];
        const double c = cs[i], s = sn[i], c2 = cs[i2], s2 = sn[i2];
        const double a1 = A[p * kk + p2], a2 = A[p * kk + q2];
        const double a3 = A[q * kk + p2], a4 = A[q * kk + q2];
        const double b1 = c2 * a1 - s2 * a2, b2 = s2 * a1 + c2 * a2;
        const double b3 = c2 * a3 - s2 * a4, b4 = s2 * a3 + c2 * a4;
        const double n1 = c * b1 - s * b3, n3 = s * b1 + c * b3;
        const double n2 = c * b2 - s * b4, n4 = s * b2 + c * b4;
        A[p * kk + p2] = n1; A[p2 * kk + p] = n1;
        A[p * kk + q2] = n2; A[q2 * kk + p] = n2;
        A[q * kk + p2] = n3; A[p2 * kk + q] = n3;
        A[q * kk + q2] = n4; A[q2 * kk + q] = n4;
      }
      for (int L = tid; L < kk * P; L += nt) {
        const int row = L / P, i = L % P;
        const double s = sn[i];
        if (s == 0.0) continue;
        const double c = cs[i];
        const int p = pp[i], q = qq[i];
        const double up = U[row * kk + p], uq = U[row * kk + q];
        U[row * kk + p] = c * up - s * uq;
        U[row * kk + q] = s * up + c * uq;
      }
      __syncthreads();
    }
    converged = (nrot == 0);
  }
  __syncthreads();
  return converged;
}

}  // namespace mdsx
