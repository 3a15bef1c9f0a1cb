// Per-piece eigen-solvers shared by the classical-MDS kernels.
#pragma once
#include "jacobi_core.cuh"

namespace mdsx {

constexpr int JAC_THREADS = 512;
constexpr int JAC_MAX_SWEEPS = 40;

struct PieceScratch {
  JacobiShared js;
  double red[JAC_THREADS];
  int order[MDSX_JACOBI_KMAX];
  double lam[MDSX_JACOBI_KMAX];
  int trivial;
  int flag;
};

// K3 full solver.  Parallel cyclic Jacobi (round-robin pairing) on the piece's
// k x k symmetric matrix in shared memory `sm` (needs 2 kk^2 doubles), then
// the spectrum post-processing of classical.py:88-106,137-150: trivial-mode
// removal (Q-form), stable descending order, 1e-8 relative zero snap,
// degenerate check, G1/G2 over the full spectrum, variance-scale estimates,
// and the top-r eigenvectors (k x r) into Uout.
// Parallel cyclic Jacobi (round-robin pairing) on a k x k symmetric matrix in
// shared memory.  Each round rotates kk/2 disjoint pairs; the two-sided
// update is done as independent 2x2 block tasks (one writer per block).
__device__ inline void full_jacobi_piece(const PieceDesc& d, int r, const double* __restrict__ Aall,
                                         double* __restrict__ Uout, double* __restrict__ lam_out,
                                         double* __restrict__ estimates, double* __restrict__ gof,
                                         mdsx_piece_status* __restrict__ status, int qform_trivial,
                                         double* sm, PieceScratch& ps) {
  JacobiShared& js = ps.js;
  double* red = ps.red;
  int* order = ps.order;
  double* lam = ps.lam;
  int& trivial = ps.trivial;
  const int pid = d.id;
  const int k = d.k, kk = k + (k & 1);
  const int tid = threadIdx.x, nt = blockDim.x;
  double* A = sm;
  double* U = sm + kk * kk;
  const double* Ag = Aall + d.a_off;

  if (status[pid].code == MDSX_INVALID_INPUT) {   // non-finite rows: nothing to solve
    for (int e = tid; e < k * r; e += nt) Uout[d.u_off + e] = 0.0;
    if (tid < r) {
      estimates[(int64_t)pid * r + tid] = 0.0;
      lam_out[(int64_t)pid * r + tid] = 0.0;
    }
    if (tid < 2) gof[2 * (int64_t)pid + tid] = 0.0;
    return;
  }

  double fro = 0.0;
  for (int e = tid; e < kk * kk; e += nt) {
    const int i = e / kk, j = e % kk;
    const double v = (i < k && j < k) ? Ag[(int64_t)i * k + j] : 0.0;
    A[e] = v;
    U[e] = (i == j) ? 1.0 : 0.0;
    fro += v * v;
  }
  red[tid] = fro;
  __syncthreads();
  for (int s = nt / 2; s > 0; s >>= 1) {
    if (tid < s) red[tid] += red[tid + s];
    __syncthreads();
  }
  // rotations below ~eps |A|_F only stir round-off noise (LAPACK-level backward error)
  const double floor_abs = 1e-15 * sqrt(red[0]);

  const bool converged = jacobi_sweeps(A, U, k, kk, floor_abs, js, JAC_MAX_SWEEPS);


  // ---- spectrum post-processing (classical.py:88-106, 137-150)
  if (tid == 0) trivial = -1;
  __syncthreads();
  if (qform_trivial && d.form == 1) {
    // eigenvector with the largest |V^T 1| carries the structural zero
    if (tid < k) {
      double s = 0.0;
      for (int i = 0; i < k; ++i) s += U[i * kk + tid];
      red[tid] = fabs(s);
    }
    __syncthreads();
    if (tid == 0) {
      int best = 0;
      for (int j = 1; j < k; ++j)
        if (red[j] > red[best]) best = j;
      trivial = best;
    }
    __syncthreads();
  }
  const int triv = trivial;
  for (int i = tid; i < k; i += nt) order[i] = i;   // valid indices even for NaN spectra
  __syncthreads();
  if (tid < k && tid != triv) {
    const double lj = A[tid * kk + tid];
    int rank = 0;
    for (int i = 0; i < k; ++i) {
      if (i == triv || i == tid) continue;
      const double li = A[i * kk + i];
      if (li > lj || (li == lj && i < tid)) ++rank;
    }
    order[rank] = tid;
  }
  __syncthreads();
  if (tid == 0) {
    const int nv = k - (triv >= 0 ? 1 : 0);
    double mx = 0.0;
    for (int i = 0; i < nv; ++i) mx = fmax(mx, fabs(A[order[i] * kk + order[i]]));
    const double tol = 1e-8 * mx;
    double sum_abs = 0.0, sum_pos = 0.0, kept = 0.0;
    for (int i = 0; i < nv; ++i) {
      double v = A[order[i] * kk + order[i]];
      if (fabs(v) <= tol) v = 0.0;
      lam[i] = v;
      sum_abs += fabs(v);
      sum_pos += fmax(v, 0.0);
      if (i < r) kept += v;
    }
    mdsx_piece_status st{MDSX_OK, 0, 0.0};
    if (status[pid].code != MDSX_OK) st.code = status[pid].code;
    else if (!converged) st.code = MDSX_NUMERICAL;
    for (int i = 0; i < r && st.code == MDSX_OK; ++i) {
      const double v = i < nv ? lam[i] : 0.0;
      if (v <= 0.0) { st.code = MDSX_DEGENERATE; st.index = i + 1; st.value = v; }
    }
    if (st.code == MDSX_OK && sum_abs == 0.0) st.code = MDSX_DEGENERATE;
    status[pid] = st;
    double* g = gof + 2 * (int64_t)pid;
    g[0] = st.code == MDSX_OK ? kept / sum_abs : 0.0;
    g[1] = st.code == MDSX_OK ? kept / sum_pos : 0.0;
    for (int i = 0; i < r; ++i) {
      const double v = i < nv ? lam[i] : 0.0;
      estimates[(int64_t)pid * r + i] = v / d.m;
      lam_out[(int64_t)pid * r + i] = v;
    }
  }
  __syncthreads();
  const int nv = k - (triv >= 0 ? 1 : 0);
  for (int e = tid; e < k * r; e += nt) {
    const int a = e / r, c = e % r;
    Uout[d.u_off + e] = c < nv ? U[a * kk + order[c]] : 0.0;
  }
}


}  // namespace mdsx
