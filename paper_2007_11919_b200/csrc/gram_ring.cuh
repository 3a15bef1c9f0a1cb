// Ring-fed Gram of one k <= 104 piece (the body of gram_piece_kernel and of
// the fused piece solver in k_lanczos.cu).  See gram_piece_kernel in
// k_gram_dmma.cu for the design.
#pragma once
#include "mdsx_common.cuh"
#include "bulk.cuh"

namespace gring {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr int GP_THREADS = 128;                 // compute warps (standalone kernel)
// Producer-side warps.  fp64 stages are shifted in place before the compute
// warps see them, and one warp doing that for 32 rows x p columns per stage
// (its DADDs queue behind the DMMAs of the same scheduler) paced the whole CTA:
// with two, each shifting and summing 16 rows of every stage, the Gram of dc2
// went 0.569 -> 0.519 ms (W = 6 / 8 compute warps, an unrolled shift loop and
// column sums through a ones column on the tensor pipe did not help).
constexpr int GP_NPROD = 2;
constexpr int GP_CTA = GP_THREADS + 32 * GP_NPROD;
constexpr int GP_KC = 32;                       // rows per stage (one per producer lane)
constexpr int GP_HDR = 2048;                    // mbarriers, x0, column sums, flag

__host__ __device__ constexpr int pair_i(int t) {
  int i = 0;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  return i;
}
__host__ __device__ constexpr int pair_j(int t) { return t - pair_i(t) * (pair_i(t) + 1) / 2; }

// the NP = NB (NB + 1) / 2 block pairs split over W compute warps
template <int NB, int W, int Q>
struct GpPart {
  static constexpr int NP = NB * (NB + 1) / 2;
  static constexpr int QS = (NP + W - 1) / W;           // pairs per warp (max)
  static constexpr int LO = Q * QS;
  static constexpr int CNT = (NP - LO) < QS ? ((NP - LO) > 0 ? NP - LO : 0) : QS;
};

// PRE: the stage holds x - x0 already (fp64 stages, shifted by the producer)
template <typename T, int NB, int W, int Q, bool PRE>
__device__ __forceinline__ void gp_chunk(const T* __restrict__ stg, int P, int nk4, const double* x0r,
                                         bool lastmask, int gid, int tig, double (*acc)[2]) {
  using QQ = GpPart<NB, W, Q>;
  const T* src = stg + (size_t)tig * P + gid;
#pragma unroll 2
  for (int k4 = 0; k4 < nk4; ++k4) {
    double f[NB];
#pragma unroll
    for (int b = 0; b < NB; ++b) f[b] = PRE ? (double)src[8 * b] : (double)src[8 * b] - x0r[b];
    if (lastmask) f[NB - 1] = 0.0;             // features >= P of the last block
#pragma unroll
    for (int u = 0; u < QQ::CNT; ++u) {
      const int t = QQ::LO + u;
      dmma(acc[u][0], acc[u][1], f[pair_i(t)], f[pair_j(t)]);
    }
    src += 4 * P;
  }
}

template <int NB, int W, int Q>
__device__ __forceinline__ void gp_store(double (*acc)[2], const double* s, double inv_m, int k,
                                         int gid, int tig, double* out) {
  using QQ = GpPart<NB, W, Q>;
#pragma unroll
  for (int u = 0; u < QQ::CNT; ++u) {
    const int t = QQ::LO + u;
    const int bi = pair_i(t), bj = pair_j(t);
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      const int gi = 8 * bi + gid, gj = 8 * bj + 2 * tig + v;
      if (gi < k && gj < k && gi >= gj) {
        const double c = fma(-s[gi] * inv_m, s[gj], acc[u][v]);
        out[(int64_t)gi * k + gj] = c;
        out[(int64_t)gj * k + gi] = c;
      }
    }
  }
}

// compile-time dispatch of warp q's pair range
template <typename T, int NB, int W, bool PRE, int Q = 0>
__device__ __forceinline__ void gp_chunk_w(int warp, const T* stg, int P, int nk4, const double* x0r,
                                           bool lastmask, int gid, int tig, double (*acc)[2]) {
  if constexpr (Q < W) {
    if (warp == Q) gp_chunk<T, NB, W, Q, PRE>(stg, P, nk4, x0r, lastmask, gid, tig, acc);
    else gp_chunk_w<T, NB, W, PRE, Q + 1>(warp, stg, P, nk4, x0r, lastmask, gid, tig, acc);
  }
}
template <int NB, int W, int Q = 0>
__device__ __forceinline__ void gp_store_w(int warp, double (*acc)[2], const double* s, double inv_m,
                                           int k, int gid, int tig, double* out) {
  if constexpr (Q < W) {
    if (warp == Q) gp_store<NB, W, Q>(acc, s, inv_m, k, gid, tig, out);
    else gp_store_w<NB, W, Q + 1>(warp, acc, s, inv_m, k, gid, tig, out);
  }
}

// The Gram of piece `pidx` by the calling CTA: warps 0 .. W-1 compute, warp W
// produces, later warps only take the first barrier.  Smem: GP_HDR + NS stages.
// fp64 stages are shifted in place by the producer (two stages ahead of the
// compute warps, on the `ready` mbarrier): one subtraction per element instead
// of one per compute warp, and no shift row in the compute warps' registers.
template <typename T, int NB, int NS, int W>
__device__ __forceinline__ void gram_piece_body(const T* __restrict__ X, int64_t ld, int p, int P,
                                                const int64_t* __restrict__ row_idx,
                                                const PieceDesc* __restrict__ pd, int pidx,
                                                double* __restrict__ A, double* __restrict__ mu_all,
                                                mdsx_piece_status* __restrict__ status,
                                                unsigned char* gp_smem) {
  constexpr bool PRE = sizeof(T) == 8;
  constexpr int NPR = PRE ? GP_NPROD : 1;          // warps sharing the shift + sums of a stage
  constexpr int NTH = 32 * (W + NPR);              // threads of the Gram roles
  uint64_t* full = reinterpret_cast<uint64_t*>(gp_smem);
  uint64_t* empty = full + NS;
  uint64_t* ready = empty + NS;
  double* x0s = reinterpret_cast<double*>(gp_smem + 128);          // 8 NB <= 104
  double* ssum = x0s + 104;
  int* bad = reinterpret_cast<int*>(ssum + 104);
  T* stage = reinterpret_cast<T*>(gp_smem + GP_HDR);                // NS x GP_KC x P
  const PieceDesc d = pd[pidx];
  const int k = d.k, m = d.m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int64_t* ridx = row_idx + d.row_off;
  const size_t stage_elems = (size_t)GP_KC * P;
  const int nchunks = (m + GP_KC - 1) / GP_KC;

  // zero padding columns [p, P) of every stage row (never written by the copies)
  for (int e = tid; P > p && e < NS * GP_KC * (P - p); e += blockDim.x) {
    const int row = e / (P - p), c = p + e % (P - p);
    stage[(size_t)row * P + c] = T(0);
  }
  if (tid < 8 * NB) x0s[tid] = tid < k ? (double)X[ridx[0] * ld + tid] : 0.0;
  if (tid == 0) {
    *bad = 0;
    for (int s = 0; s < NS; ++s) {
      bulk::bar_init(&full[s], 1);
      bulk::bar_init(&empty[s], W);
      bulk::bar_init(&ready[s], NPR);
    }
    bulk::bar_fence();
  }
  __syncthreads();
  if (warp >= W + NPR) return;

  if (warp >= W) {
    const int pw = warp - W;                       // 0: copies + its share of the rows; others: rows only
    // ---- producer: gather rows, shift (fp64) and sum the columns of the
    // stages handed over
    const unsigned row_bytes = (unsigned)((size_t)p * sizeof(T));
    double cs[4] = {0.0, 0.0, 0.0, 0.0};       // features lane + 32 q
    double x0l[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x0l[q] = lane + 32 * q < 8 * NB ? x0s[lane + 32 * q] : 0.0;
    auto colsums = [&](int c) {
      const int s = c % NS;
      bulk::wait(&full[s], (unsigned)((c / NS) & 1));
      T* stg = stage + (size_t)s * stage_elems;
      const int nr = min(GP_KC, m - c * GP_KC);
      const int i0 = pw * (GP_KC / NPR), i1 = min(nr, (pw + 1) * (GP_KC / NPR));
      for (int i = i0; i < i1; ++i)
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (lane + 32 * q < p) {
            const double v = (double)stg[(size_t)i * P + lane + 32 * q] - x0l[q];
            if constexpr (PRE) stg[(size_t)i * P + lane + 32 * q] = (T)v;
            cs[q] += v;
          }
      if constexpr (PRE) {
        __syncwarp();
        if (lane == 0) bulk::arrive(&ready[s]);
      }
    };
    constexpr int LAG = PRE ? 2 : NS - 1;          // stages between issue and the sums
    if (pw == 0) {
      int64_t nidx = lane < m ? ridx[lane] : 0;
      int64_t nidx2 = GP_KC + lane < m ? ridx[GP_KC + lane] : 0;
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % NS;
        const int r0 = c * GP_KC, nr = min(GP_KC, m - r0);
        const int64_t idx = nidx;
        nidx = nidx2;
        if (r0 + 2 * GP_KC + lane < m) nidx2 = ridx[r0 + 2 * GP_KC + lane];
        if (PRE && c >= LAG) colsums(c - LAG);      // ahead of the compute warps
        if (c >= NS) bulk::wait(&empty[s], (unsigned)((c / NS - 1) & 1));
        T* dst = stage + (size_t)s * stage_elems;
        const int npad = ((nr + 3) & ~3) - nr;     // rows that complete the last k4 group
        for (int e = lane; e < npad * p; e += 32)  // shifted value exactly 0 there
          dst[(size_t)(nr + e / p) * P + e % p] = PRE ? T(0) : (T)x0s[e % p];
        __syncwarp();
        if (lane == 0) bulk::arrive_expect(&full[s], (unsigned)nr * row_bytes);
        __syncwarp();
        if (lane < nr) bulk::copy(dst + (size_t)lane * P, X + idx * ld, row_bytes, &full[s]);
        if (!PRE && c >= LAG) colsums(c - LAG);
      }
      for (int c = max(0, nchunks - LAG); c < nchunks; ++c) colsums(c);
    } else {
      for (int c = 0; c < nchunks; ++c) colsums(c);   // its rows of every stage, as they land
    }
    // column sums: producer 0's partial first, then the others in warp order
    for (int w2 = 0; w2 < NPR; ++w2) {
      if (pw == w2) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int a = lane + 32 * q;
          if (a < 8 * NB) ssum[a] = (w2 ? ssum[a] : 0.0) + (a < p ? cs[q] : 0.0);
          if (a < k && !isfinite(cs[q])) *bad = 1;
        }
      }
      if (NPR > 1) asm volatile("bar.sync 2, %0;\n" ::"r"(32 * NPR));
    }
    asm volatile("bar.sync 1, %0;\n" ::"r"(NTH));
    return;
  }
  // ---- compute warps
  double x0r[PRE ? 1 : NB];
  if constexpr (!PRE) {
#pragma unroll
    for (int b = 0; b < NB; ++b) x0r[b] = x0s[8 * b + gid];
  }
  const bool lastmask = 8 * (NB - 1) + gid >= P;    // the stage pitch may be < 8 NB
  constexpr int QS = GpPart<NB, W, 0>::QS;
  double acc[QS][2];
#pragma unroll
  for (int u = 0; u < QS; ++u) acc[u][0] = acc[u][1] = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const int s = c % NS;
    bulk::wait(PRE ? &ready[s] : &full[s], (unsigned)((c / NS) & 1));
    const T* stg = stage + (size_t)s * stage_elems;
    const int nk4 = (min(GP_KC, m - c * GP_KC) + 3) / 4;
    gp_chunk_w<T, NB, W, PRE>(warp, stg, P, nk4, x0r, lastmask, gid, tig, acc);
    __syncwarp();
    if (lane == 0) bulk::arrive(&empty[s]);
  }
  asm volatile("bar.sync 1, %0;\n" ::"r"(NTH));          // column sums ready
  const double inv_m = 1.0 / (double)m;
  double* out = A + d.a_off;
  gp_store_w<NB, W>(warp, acc, ssum, inv_m, k, gid, tig, out);
  if (tid < k) mu_all[(int64_t)d.id * p + tid] = x0s[tid] + ssum[tid] * inv_m;
  if (tid == 0 && *bad) status[d.id].code = MDSX_INVALID_INPUT;
}

}  // namespace gring
