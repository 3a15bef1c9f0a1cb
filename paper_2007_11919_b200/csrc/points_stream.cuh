// Piece points X~ U_r for one form-0 piece by one CTA of PS_T threads, and the
// canonical column signs (linalg.py:139-146).  Shared by points_piece_kernel
// (k_points.cu) and the points epilogue of the Lanczos kernel (k_lanczos.cu).
//
// Thread t owns rows t, t+PS_T, ... of the piece and streams them back to back
// through a private PS_NS-deep cp.async ring of 64-byte feature blocks in
// shared memory (its own cp.async groups: no block barrier in the loop, and
// the ring never drains between rows).  The per-feature records (U row pairs,
// mean) are read as warp broadcasts; all r outputs accumulate in registers.
// The column signs (largest |value| positive, lowest row on ties) are reduced
// in the CTA and applied to the rows the thread wrote (L1/L2-hot).
#pragma once
#include "mdsx_common.cuh"

namespace mdsx {

constexpr int PS_T = 256;         // threads
constexpr int PS_NS = 4;          // ring depth (64-byte blocks in flight per thread)
constexpr int PS_PITCH = 80;      // bytes per ring slot (64 + 16: conflict-free 16-byte reads)

template <int RM>
__host__ __device__ constexpr int ps_rec_width() { return RM / 2 + 1; }

// shared-memory bytes: records p x W double2 + the ring + the sign scratch
constexpr size_t PS_SCRATCH = (size_t)(PS_T / 32) * MDSX_MAX_R * 12 + MDSX_MAX_R * 8;
template <int RM>
__host__ __device__ constexpr size_t ps_smem_bytes(int p) {
  return (size_t)p * ps_rec_width<RM>() * 16 + (size_t)PS_T * PS_NS * PS_PITCH + PS_SCRATCH;
}

// Records from U (k x r, row-major, global or shared) and the piece mean.
template <int RM>
__device__ void ps_load_records(unsigned char* smem, const double* U, const double* mu, int p, int r) {
  constexpr int W = ps_rec_width<RM>();
  double2* rec = reinterpret_cast<double2*>(smem);
  for (int e = threadIdx.x; e < p * W; e += PS_T) {
    const int a = e / W, w = e % W;
    double2 v = make_double2(0.0, 0.0);
    if (w < RM / 2) {
      v.x = 2 * w < r ? U[(int64_t)a * r + 2 * w] : 0.0;
      v.y = 2 * w + 1 < r ? U[(int64_t)a * r + 2 * w + 1] : 0.0;
    } else {
      v.x = mu[a];
    }
    rec[e] = v;
  }
}

// Streams the piece; the records must be in smem (and a barrier passed) before
// the first wait, i.e. call ps_load_records, __syncthreads, then this.  The
// ring prologue is issued by ps_prologue so it overlaps the record loads.
template <typename T, int RM>
struct PieceStream {
  static constexpr int FB = 64 / (int)sizeof(T);
  unsigned char* ring;
  const T* X;
  int64_t ld;
  const int64_t* ridx;
  int p, nblk, my_rows, nstream;
  int iq, ib, is, issued;
  const char* src_cur;
  int64_t nxt_idx;

  // rows [0, m) of ridx_ (callers offset ridx_ to a chunk of the piece)
  __device__ PieceStream(unsigned char* smem, const T* X_, int64_t ld_, const int64_t* ridx_, int p_,
                         int m)
      : X(X_), ld(ld_), ridx(ridx_), p(p_) {
    const int tid = threadIdx.x;
    ring = smem + (size_t)p * ps_rec_width<RM>() * 16 + (size_t)tid * PS_PITCH;
    nblk = (p + FB - 1) / FB;
    my_rows = tid < m ? (m - 1 - tid) / PS_T + 1 : 0;
    nstream = my_rows * nblk;
    iq = ib = is = issued = 0;
    src_cur = my_rows > 0 ? reinterpret_cast<const char*>(X + ridx[tid] * ld) : nullptr;
    nxt_idx = my_rows > 1 ? ridx[tid + PS_T] : 0;
  }

  // one 64-byte block of the cursor (row iq, block ib); the next row's base
  // address is loaded one row ahead
  __device__ __forceinline__ void issue() {
    if (issued < nstream) {
      const int nbytes = min(64, (int)((p - ib * FB) * (int)sizeof(T)));
      unsigned char* dst = ring + (size_t)is * PS_T * PS_PITCH;
      for (int o = 0; o < nbytes; o += 16) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + o);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src_cur + 64 * ib + o));
      }
      ++issued;
      if (++is == PS_NS) is = 0;
      if (++ib == nblk) {
        ib = 0;
        ++iq;
        src_cur = reinterpret_cast<const char*>(X + nxt_idx * ld);
        if (iq + 1 < my_rows) nxt_idx = ridx[threadIdx.x + (iq + 1) * PS_T];
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }

  __device__ void prologue() {
#pragma unroll
    for (int b = 0; b < PS_NS - 1; ++b) issue();
  }

  // points of the rows into out (m x r, row-major).  cand == nullptr: the rows
  // are the whole piece and the column signs are applied here; otherwise the
  // per-column (signed value, row0 + row) of the largest |value| go to
  // cand[0..r) for sign_chunk_kernel.
  __device__ void run(const unsigned char* smem, int r, double* out, double2* cand = nullptr,
                      int row0 = 0) {
    constexpr int W = ps_rec_width<RM>();
    const double2* rec = reinterpret_cast<const double2*>(smem);
    const int tid = threadIdx.x;
    double best[RM];                                        // signed value of largest |.|
    int bi[RM];
    double acc[RM];
#pragma unroll
    for (int c = 0; c < RM; ++c) { best[c] = 0.0; bi[c] = 0x7fffffff; acc[c] = 0.0; }
    int q = 0, b = 0, cs = 0;
    const unsigned char* ring0 = ring;
    for (int sidx = 0; sidx < nstream; ++sidx) {
      issue();
      asm volatile("cp.async.wait_group %0;\n" ::"n"(PS_NS - 1));
      const unsigned char* xb = ring0 + (size_t)cs * PS_T * PS_PITCH;
      if (++cs == PS_NS) cs = 0;
      const int a0 = b * FB;
      const int nf = min(FB, p - a0);
      constexpr int VW = 16 / (int)sizeof(T);
#pragma unroll
      for (int v4 = 0; v4 < 4; ++v4) {
        if (v4 * VW >= nf) break;                     // the last block may be short
        double xv[VW];
        if constexpr (sizeof(T) == 4) {
          const float4 f = *reinterpret_cast<const float4*>(xb + 16 * v4);
          xv[0] = f.x; xv[1] = f.y; xv[2] = f.z; xv[3] = f.w;
        } else {
          const double2 f = *reinterpret_cast<const double2*>(xb + 16 * v4);
          xv[0] = f.x; xv[1] = f.y;
        }
#pragma unroll
        for (int u = 0; u < VW; ++u) {
          const double2* rp = rec + (size_t)(a0 + v4 * VW + u) * W;
          const double y = xv[u] - rp[W - 1].x;
#pragma unroll
          for (int w = 0; w < RM / 2; ++w) {
            const double2 uu = rp[w];
            acc[2 * w] = fma(y, uu.x, acc[2 * w]);
            acc[2 * w + 1] = fma(y, uu.y, acc[2 * w + 1]);
          }
        }
      }
      if (++b == nblk) {                               // row done: store, candidates, next row
        const int i = tid + q * PS_T;
#pragma unroll
        for (int c = 0; c < RM; ++c) {
          if (c < r) {
            out[(int64_t)i * r + c] = acc[c];
            if (fabs(acc[c]) > fabs(best[c]) || bi[c] == 0x7fffffff) { best[c] = acc[c]; bi[c] = i; }
          }
          acc[c] = 0.0;
        }
        b = 0;
        ++q;
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    // column signs: (|value|, lowest row) maxima over the CTA in fixed order
    // (scratch in the dynamic allocation after the ring: no static shared memory,
    // so the Lanczos kernel that embeds this keeps its two CTAs per SM)
    unsigned char* scr = const_cast<unsigned char*>(smem) + (size_t)p * W * 16 +
                         (size_t)PS_T * PS_NS * PS_PITCH;
    double (*ps_wv)[MDSX_MAX_R] = reinterpret_cast<double (*)[MDSX_MAX_R]>(scr);
    double* ps_sgn = reinterpret_cast<double*>(scr + (size_t)(PS_T / 32) * MDSX_MAX_R * 8);
    int (*ps_wi)[MDSX_MAX_R] = reinterpret_cast<int (*)[MDSX_MAX_R]>(
        scr + (size_t)(PS_T / 32) * MDSX_MAX_R * 8 + MDSX_MAX_R * 8);
    const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
    for (int c = 0; c < RM; ++c) {
      if (c >= r) break;
      double v = best[c];
      int ix = bi[c];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, ix, o);
        if (i2 != 0x7fffffff &&
            (ix == 0x7fffffff || fabs(v2) > fabs(v) || (fabs(v2) == fabs(v) && i2 < ix))) {
          v = v2;
          ix = i2;
        }
      }
      if (lane == 0) { ps_wv[warp][c] = v; ps_wi[warp][c] = ix; }
    }
    __syncthreads();
    if (tid < r) {
      double v = 0.0;
      int ix = 0x7fffffff;
      for (int w = 0; w < PS_T / 32; ++w) {
        const double v2 = ps_wv[w][tid];
        const int i2 = ps_wi[w][tid];
        if (i2 != 0x7fffffff &&
            (ix == 0x7fffffff || fabs(v2) > fabs(v) || (fabs(v2) == fabs(v) && i2 < ix))) {
          v = v2;
          ix = i2;
        }
      }
      ps_sgn[tid] = v < 0.0 ? -1.0 : 1.0;
      if (cand) cand[tid] = make_double2(v, (double)(ix == 0x7fffffff ? ix : row0 + ix));
    }
    if (cand) return;
    __syncthreads();
    bool any = false;
    double sg[RM];
#pragma unroll
    for (int c = 0; c < RM; ++c) {
      sg[c] = c < r ? ps_sgn[c] : 1.0;
      any |= sg[c] < 0.0;
    }
    if (any)
      for (int qq = 0; qq < my_rows; ++qq) {
        double* row = out + (int64_t)(tid + qq * PS_T) * r;
#pragma unroll
        for (int c = 0; c < RM; ++c)
          if (c < r && sg[c] < 0.0) row[c] = -row[c];
      }
  }
};

}  // namespace mdsx
