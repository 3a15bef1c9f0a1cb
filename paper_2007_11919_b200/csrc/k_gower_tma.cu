// K4 streaming Gower interpolation through TMA tensor maps (sm_100a).
//
// Same arithmetic as gower_bulk_kernel (k_gower.cu): per row y,
//   out = y^T M - xbar^T M - |y - xbar|^2 v,
// with M, v, xbar from the Gower context (algorithms.py:193-242 restated).
//
// Data movement: a 2-D tensor map over the n x p input with a box of
// 256 rows x 128 bytes (32 fp32 / 16 fp64 features) and the hardware 128-byte
// swizzle.  A stage is one feature slab of one 512-row tile (two boxes,
// 64 KB); a producer warp streams (tile, slab) stages through a 3-deep
// mbarrier ring.  Rows past n and features past p arrive zero-filled.
//
// Compute: eight warps, lane l of warp w owns rows 64w + l and 64w + l + 32 of
// the tile for ALL features (no cross-lane reduction), so every lane of a warp
// reads the same per-feature record (M row, mean, mask) at the same time — a
// shared-memory broadcast feeding 64 rows — while the row reads of a lane are
// 16-byte chunks made conflict-free by the 128-byte swizzle (chunk c of row
// rho lives at chunk c ^ (rho & 7)).  Per-CTA column sums of the output are
// accumulated for the re-centring (fixed order).
//
// Opt-in (MDSX_GOWER_TMA=1): measured on config 4 at 1.63 ms against 1.18 ms
// for the 1-D bulk-copy kernel (gower_bulk_kernel) — the record broadcasts
// still cost two wavefronts per 128-bit load and the per-lane instruction
// count is higher (ncu: 842M vs 694M warp instructions).  Kept for the
// 4-rows-per-lane / 64-byte-slab variant.
#include "mdsx_common.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace {

constexpr int GT_THREADS = 256;            // consumer threads (8 warps)
constexpr int GT_CTA = GT_THREADS + 32;    // + producer warp
constexpr int GT_ROWS = 512;               // rows per tile (8 warps x 64)
constexpr int GT_BOX_ROWS = 256;           // rows per TMA box
constexpr int GT_STAGES = 3;
constexpr int GT_STAGE_BYTES = GT_ROWS * 128;   // 64 KB
constexpr int GT_HEADER = 1024;            // barriers, c0, v (1024 keeps the stages aligned)

__device__ __forceinline__ unsigned saddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void bar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(saddr(b)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, unsigned phase) {
  asm volatile(
      "{\n.reg .pred P;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
      "@!P bra WAIT_%=;\n}\n" ::"r"(saddr(b)), "r"(phase) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];\n" ::"r"(saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(saddr(b)) : "memory");
}

template <typename T, int RM, bool N32>
__global__ void __launch_bounds__(GT_CTA, 1)
gower_tma_kernel(const __grid_constant__ CUtensorMap tmap, const T* __restrict__ X, int64_t m,
                 int p, int r,
                 const double* __restrict__ ctx_mean, const double* __restrict__ ctx_M,
                 const double* __restrict__ ctx_v, double* __restrict__ out,
                 double* __restrict__ colpart, int32_t* __restrict__ nonfinite) {
  constexpr int FS = 128 / (int)sizeof(T);  // features per slab
  constexpr int VW = 16 / (int)sizeof(T);   // features per 16-byte chunk
  constexpr int W = RM / 2 + 1;             // record: M pairs, (mean, mask)
  extern __shared__ __align__(1024) unsigned char gsm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(gsm);
  uint64_t* empty = full + GT_STAGES;
  double* c0s = reinterpret_cast<double*>(gsm + 128);     // xbar^T M (16)
  double* vvs = c0s + 16;                                  // v (16)
  unsigned char* stages = gsm + GT_HEADER;
  const int nslab = (p + FS - 1) / FS;
  double2* rec = reinterpret_cast<double2*>(stages + (size_t)GT_STAGES * GT_STAGE_BYTES);
  const int tid = threadIdx.x;
  const int64_t ntiles = (m + GT_ROWS - 1) / GT_ROWS;
  const int64_t my_tiles = blockIdx.x < ntiles ? (ntiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int64_t nstage_total = my_tiles * nslab;

  if (tid == 0) {
    for (int s = 0; s < GT_STAGES; ++s) {
      bar_init(&full[s], 1);
      bar_init(&empty[s], GT_THREADS / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (tid >= GT_THREADS) {                  // ---- producer warp
    if (tid == GT_THREADS) {
      for (int64_t k = 0; k < nstage_total; ++k) {
        const int s = (int)(k % GT_STAGES);
        if (k >= GT_STAGES) bar_wait(&empty[s], (unsigned)((k / GT_STAGES - 1) & 1));
        const int64_t tile = blockIdx.x + (k / nslab) * gridDim.x;
        const int slab = (int)(k % nslab);
        unsigned char* dst = stages + (size_t)s * GT_STAGE_BYTES;
        bar_expect(&full[s], GT_STAGE_BYTES);
        tma_load_2d(dst, &tmap, slab * FS, (int)(tile * GT_ROWS), &full[s]);
        tma_load_2d(dst + GT_BOX_ROWS * 128, &tmap, slab * FS, (int)(tile * GT_ROWS + GT_BOX_ROWS),
                    &full[s]);
      }
    }
    return;
  }

  // ---- records: rec[f * W + w] for f < nslab * FS (zero, mask 0 past p)
  for (int e = tid; e < nslab * FS * W; e += GT_THREADS) {
    const int f = e / W, w = e % W;
    double2 v2 = make_double2(0.0, 0.0);
    if (f < p) {
      if (w < RM / 2) {
        const int c = 2 * w;
        v2.x = c < r ? ctx_M[(int64_t)f * r + c] : 0.0;
        v2.y = c + 1 < r ? ctx_M[(int64_t)f * r + c + 1] : 0.0;
      } else {
        v2.x = ctx_mean[f];
        v2.y = N32 ? __hiloint2double(__float_as_int(1.0f), __float_as_int((float)ctx_mean[f])) : 1.0;
      }
    }
    rec[e] = v2;
  }
  if (tid < 16) {                            // c0 = xbar^T M (fixed order), v
    double sacc = 0.0;
    if (tid < r)
      for (int a = 0; a < p; ++a) sacc = fma(ctx_mean[a], ctx_M[(int64_t)a * r + tid], sacc);
    c0s[tid] = sacc;
    vvs[tid] = tid < r ? ctx_v[tid] : 0.0;
  }
  asm volatile("bar.sync 1, %0;\n" ::"n"(GT_THREADS) : "memory");

  const int lane = tid & 31, warp = tid >> 5;
  const int rho0 = warp * 64 + lane, rho1 = rho0 + 32;    // rows of the tile (rho & 7 == lane & 7)
  const int sw = lane & 7;
  double csum[RM];
#pragma unroll
  for (int c = 0; c < RM; ++c) csum[c] = 0.0;
  double acc[2][RM], nrm[2];
  float nrm32[2];
  bool bad = false;
  for (int64_t k = 0; k < nstage_total; ++k) {
    const int s = (int)(k % GT_STAGES);
    const int slab = (int)(k % nslab);
    if (slab == 0) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        nrm[q] = 0.0;
        nrm32[q] = 0.0f;
#pragma unroll
        for (int c = 0; c < RM; ++c) acc[q][c] = 0.0;
      }
    }
    bar_wait(&full[s], (unsigned)((k / GT_STAGES) & 1));
    const unsigned char* st = stages + (size_t)s * GT_STAGE_BYTES;
    const unsigned char* row0 = st + rho0 * 128;
    const unsigned char* row1 = st + rho1 * 128;
    const double2* rbase = rec + (size_t)slab * FS * W;
#pragma unroll 2
    for (int ch = 0; ch < FS / VW; ++ch) {
      const int pc = (ch ^ sw) * 16;                       // 128-byte swizzle
      double xv[2][VW];
      if constexpr (sizeof(T) == 4) {
        const float4 f0 = *reinterpret_cast<const float4*>(row0 + pc);
        const float4 f1 = *reinterpret_cast<const float4*>(row1 + pc);
        xv[0][0] = f0.x; xv[0][1] = f0.y; xv[0][2] = f0.z; xv[0][3] = f0.w;
        xv[1][0] = f1.x; xv[1][1] = f1.y; xv[1][2] = f1.z; xv[1][3] = f1.w;
      } else {
        const double2 f0 = *reinterpret_cast<const double2*>(row0 + pc);
        const double2 f1 = *reinterpret_cast<const double2*>(row1 + pc);
        xv[0][0] = f0.x; xv[0][1] = f0.y;
        xv[1][0] = f1.x; xv[1][1] = f1.y;
      }
#pragma unroll
      for (int u = 0; u < VW; ++u) {
        const double2* rp = rbase + (size_t)(ch * VW + u) * W;
        double2 mw[W];
#pragma unroll
        for (int w = 0; w < W; ++w) mw[w] = rp[w];            // warp broadcast
        const double mu = mw[W - 1].x, msk = mw[W - 1].y;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double xq = xv[q][u];
          if constexpr (N32) {
            const float xf = (float)xq;
            const float y32 = (xf - __int_as_float(__double2loint(msk))) *
                              __int_as_float(__double2hiint(msk));
            nrm32[q] = fmaf(y32, y32, nrm32[q]);
          } else {
            const double y = fma(xq, msk, -mu);
            nrm[q] = fma(y, y, nrm[q]);
          }
#pragma unroll
          for (int w = 0; w < RM / 2; ++w) {
            acc[q][2 * w] = fma(xq, mw[w].x, acc[q][2 * w]);
            acc[q][2 * w + 1] = fma(xq, mw[w].y, acc[q][2 * w + 1]);
          }
        }
      }
    }
    const bool last = slab == nslab - 1;
    const int64_t tile = blockIdx.x + (k / nslab) * gridDim.x;
    if (last) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if constexpr (N32) nrm[q] = (double)nrm32[q];
        const int64_t row = tile * GT_ROWS + (q == 0 ? rho0 : rho1);
        if (row < m && !isfinite(nrm[q])) {
          // overflowed norm (fp64 data / fp32 norms of huge values) or a real
          // non-finite value: decide on the input row, recompute in fp64
          const T* xr = X + row * p;
          double s2 = 0.0;
          for (int a = 0; a < p; ++a) {
            const double xa = (double)xr[a];
            bad |= !isfinite(xa);
            const double ya = xa - ctx_mean[a];
            s2 = fma(ya, ya, s2);
          }
          nrm[q] = s2;
        }
      }
    }
    __syncwarp();
    if (lane == 0) bar_arrive(&empty[s]);
    if (last) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int64_t row = tile * GT_ROWS + (q == 0 ? rho0 : rho1);
        if (row >= m) continue;
        double* o = out + row * r;
#pragma unroll
        for (int c = 0; c < RM; ++c)
          if (c < r) {
            const double val = fma(-nrm[q], vvs[c], acc[q][c] - c0s[c]);
            o[c] = val;
            csum[c] += val;
          }
      }
    }
  }
  if (bad) atomicOr(nonfinite, 1);
  if (colpart != nullptr) {
    asm volatile("bar.sync 1, %0;\n" ::"n"(GT_THREADS) : "memory");   // all stages consumed
    double* red = reinterpret_cast<double*>(stages);
#pragma unroll
    for (int c = 0; c < RM; ++c) red[c * GT_THREADS + tid] = csum[c];
    asm volatile("bar.sync 1, %0;\n" ::"n"(GT_THREADS) : "memory");
    if (tid < r) {
      double sacc = 0.0;
      for (int i = 0; i < GT_THREADS; ++i) sacc += red[tid * GT_THREADS + i];
      colpart[(int64_t)blockIdx.x * r + tid] = sacc;
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

}  // namespace

namespace mdsx {

// TMA tensor-map Gower over m dense rows (row pitch p, 16-byte multiple).
// *nparts = column-sum partials written (one per CTA); 0 when not applicable
// (nothing launched).
int launch_gower_tma(mdsx_handle* h, const void* X, int dtype, int64_t m, int p, int r,
                     const double* mean, const double* M, const double* v, double* out,
                     double* colpart, int32_t* nonfinite, int* nparts, cudaStream_t st,
                     bool norm32) {
  *nparts = 0;
  const size_t es = dtype == MDSX_F32 ? 4 : 8;
  if (m == 0 || r > 16 || ((size_t)p * es) % 16 != 0 || m > ((int64_t)1 << 31) - GT_ROWS ||
      (reinterpret_cast<uintptr_t>(X) & 15) != 0 || !getenv("MDSX_GOWER_TMA"))
    return MDSX_OK;
  auto enc = encode_fn();
  if (!enc) return MDSX_OK;
  const int FS = (int)(128 / es);
  const int nslab = (p + FS - 1) / FS;
  const int RM = r <= 4 ? 4 : r <= 8 ? 8 : r <= 10 ? 10 : r <= 12 ? 12 : 16;
  const size_t smem = GT_HEADER + (size_t)GT_STAGES * GT_STAGE_BYTES +
                      (size_t)nslab * FS * (RM / 2 + 1) * 16;
  if (smem > (size_t)(h->max_smem_optin > 0 ? h->max_smem_optin : 227 * 1024)) return MDSX_OK;
  CUtensorMap tmap;
  const cuuint64_t dims[2] = {(cuuint64_t)p, (cuuint64_t)m};
  const cuuint64_t strides[1] = {(cuuint64_t)p * es};
  const cuuint32_t box[2] = {(cuuint32_t)FS, (cuuint32_t)GT_BOX_ROWS};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&tmap, dtype == MDSX_F32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
          2, const_cast<void*>(X), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return MDSX_OK;
  const int64_t ntiles = (m + GT_ROWS - 1) / GT_ROWS;
  const int blocks = (int)std::min<int64_t>(ntiles, (int64_t)h->num_sms);
  auto go = [&](auto tag, auto rm, auto n32) -> int {
    using T = decltype(tag);
    constexpr int RMc = decltype(rm)::value;
    constexpr bool N32c = decltype(n32)::value;
    auto kern = gower_tma_kernel<T, RMc, N32c>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    mdsx::pre(h, st);
    kern<<<blocks, GT_CTA, smem, st>>>(tmap, (const T*)X, m, p, r, mean, M, v, out, colpart,
                                       nonfinite);
    const int rc = launched(h, "gower_tma_kernel", st);
    if (!rc) *nparts = colpart ? blocks : -1;
    return rc;
  };
  using F = std::false_type;
  using Tr = std::true_type;
  auto by_rm = [&](auto tag, auto n32) -> int {
    switch (RM) {
      case 4: return go(tag, std::integral_constant<int, 4>{}, n32);
      case 8: return go(tag, std::integral_constant<int, 8>{}, n32);
      case 10: return go(tag, std::integral_constant<int, 10>{}, n32);
      case 12: return go(tag, std::integral_constant<int, 12>{}, n32);
      default: return go(tag, std::integral_constant<int, 16>{}, n32);
    }
  };
  if (dtype == MDSX_F32) return norm32 ? by_rm(float{}, Tr{}) : by_rm(float{}, F{});
  return by_rm(double{}, F{});
}

}  // namespace mdsx
