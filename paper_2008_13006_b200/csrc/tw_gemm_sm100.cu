// K2: persistent grouped tile-wise sparse GEMM for sm_100a.
//
// Replaces, in one launch, the reference's per-call pipeline
//   _plan_tasks + gather_rows   (engine.py:61-69, :126-149)  -> TMA gather4 of
//                                 the kept A^T rows straight into SW128 smem
//   group_by_shape + execute_batched + thread pool (engine.py:72-123)
//                               -> static LPT work list over persistent CTAs
//   mm_accum                    (_kernels.py:13-27) -> tcgen05.mma, fp32 TMEM
//   ct = zeros(N, M)            (engine.py:102) -> pruned C^T rows written as
//                                 zeros by the epilogue warps, interleaved
//                                 with the MMA work
//
// Orientation.  C = A * W per tile, with the MMA's M = tokens (128 per work
// unit), N = the tile's output columns (n_i <= 256), K = the tile's kept rows.
//   A operand (MN-major, SW128): kept rows of A^T (K x M, M contiguous).  Per
//     pipeline stage 64 kept k x 128 tokens: two 64-token halves (LBO = 8 KB),
//     each 64 rows of 128 B (8-row swizzle atoms, SBO = 1 KB).  Loaded with
//     16 x 2 TMA gather4 (4 kept k-rows each); padded k indices point past K
//     so TMA zero-fills them.
//   B operand (K-major, SW128): the packed weight image of the tile, one
//     1-D bulk copy per stage (wrows x 128 B, pre-swizzled on the host).
//   D (TMEM, fp32): lane = token, column = tile column.  Double buffered
//     (2 x BN columns) so the epilogue of unit i overlaps the mainloop of i+1.
// Epilogue.  tcgen05.ld 32x32b: thread t of epilogue warp q owns token
//   m0 + 32q + t; for each tile column n the warp stores 32 consecutive
//   tokens to C^T[col_ids[n], m0 + 32q ...] -- one 128 B coalesced line (fp32).
//
// Warp roles (192 threads): w0 = TMA producer, w1 = MMA issuer + TMEM owner,
// w2..w5 = epilogue (TMEM lane quadrant = warp % 4).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tw_internal.h"
#include "tw_ptx.cuh"

namespace tw {


namespace {

constexpr int kThreads = 192;
constexpr int kBlockM = 128;
constexpr int kBlockK = 64;
constexpr uint32_t kABytes = kBlockM * kBlockK * 2;  // 16 KB per stage

template <int BN>
struct Cfg {
  static constexpr int kStages = BN <= 128 ? 6 : 4;
  static constexpr uint32_t kBBytes = BN * 128;
  static constexpr uint32_t kTmemCols = 2 * BN;
  static constexpr uint32_t kSmem = 1024 /*align slack*/ + kStages * (kABytes + kBBytes) + 256;
};

template <typename T>
__device__ __forceinline__ T cvt_out(float v);
template <>
__device__ __forceinline__ float cvt_out<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ __half cvt_out<__half>(float v) { return __float2half_rn(v); }
template <typename T>
__device__ __forceinline__ float cvt_in(T v);
template <>
__device__ __forceinline__ float cvt_in<float>(float v) { return v; }
template <>
__device__ __forceinline__ float cvt_in<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ float cvt_in<__half>(__half v) { return __half2float(v); }

// zero rows [r0, r1) of the zero list, full M, by the 128 epilogue threads
template <typename OutT>
__device__ __forceinline__ void write_zero_rows(const GemmArgs &a, int r0, int r1, int et) {
  const int64_t row_bytes = (int64_t)a.M * sizeof(OutT);
  const bool vec = ((a.ldc * (int64_t)sizeof(OutT)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0);
  for (int r = r0; r < r1; ++r) {
    const int row = __ldg(a.zero_rows + r);
    char *base = reinterpret_cast<char *>(a.out) + (int64_t)row * a.ldc * sizeof(OutT);
    if (vec) {
      const int64_t n16 = row_bytes / 16;
      uint4 z = make_uint4(0, 0, 0, 0);
      for (int64_t i = et; i < n16; i += 128) reinterpret_cast<uint4 *>(base)[i] = z;
      for (int64_t i = n16 * 16 / sizeof(OutT) + et; i < a.M; i += 128) reinterpret_cast<OutT *>(base)[i] = cvt_out<OutT>(0.f);
    } else {
      for (int64_t i = et; i < a.M; i += 128) reinterpret_cast<OutT *>(base)[i] = cvt_out<OutT>(0.f);
    }
  }
}

template <int BN, typename OutT>
__global__ void __launch_bounds__(kThreads, 1)
    tw_gemm_sm100_kernel(const __grid_constant__ CUtensorMap tmap_at, const __grid_constant__ GemmArgs args) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sA = smem;
  uint8_t *sB = smem + C::kStages * kABytes;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + C::kStages * C::kBBytes);
  uint64_t *empty = full + C::kStages;
  uint64_t *tfull = empty + C::kStages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int total_units = args.n_live * args.mblocks;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 128);
    }
    ptx::fence_mbar_init();
    ptx::prefetch_tmap(&tmap_at);
  }
  if (warp == 1) ptx::tmem_alloc<C::kTmemCols>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      const uint64_t keep = ptx::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
        const TileMeta t = args.tiles[u / args.mblocks];
        const int m0 = (u % args.mblocks) * kBlockM;
        const int4 *ki = reinterpret_cast<const int4 *>(args.kidx + t.kidx_off);
        const uint8_t *wsrc = args.wimg + t.w_off;
        for (int kb = 0; kb < t.nkb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_arrive_expect_tx(&full[stage], kABytes + (uint32_t)args.wbytes);
          ptx::bulk_g2s(sB + stage * C::kBBytes, wsrc + (int64_t)kb * args.wbytes, (uint32_t)args.wbytes,
                        &full[stage], keep);
          uint8_t *a_dst = sA + stage * kABytes;
#pragma unroll 4
          for (int g = 0; g < kBlockK / 4; ++g) {
            const int4 rows = __ldg(ki + kb * (kBlockK / 4) + g);
            ptx::tma_gather4(a_dst + g * 512, &tmap_at, &full[stage], m0, rows, keep);
            ptx::tma_gather4(a_dst + 8192 + g * 512, &tmap_at, &full[stage], m0 + 64, rows, keep);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t a_base = ptx::smem_u32(sA);
    const uint32_t b_base = ptx::smem_u32(sB);
    for (int u = blockIdx.x; u < total_units; u += gridDim.x) {
      const TileMeta t = args.tiles[u / args.mblocks];
      const uint32_t n_mma = (uint32_t)((t.n_i + 15) & ~15);
      const uint32_t idesc = args.idesc | ((n_mma >> 3) << 17);
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
      ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      for (int kb = 0; kb < t.nkb; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const int nk = min(4, t.k16 - kb * 4);
        if (ptx::elect_one()) {
          for (int kk = 0; kk < nk; ++kk) {
            const uint64_t adesc = ptx::make_sw128_desc(a_base + stage * kABytes + kk * 2048, 8192, 1024);
            const uint64_t bdesc = ptx::make_sw128_desc(b_base + stage * C::kBBytes + kk * 32, 16, 1024);
            ptx::mma_f16_ss(d_tmem, adesc, bdesc, idesc, (kb | kk) != 0 ? 1u : 0u);
          }
          ptx::mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
      if (ptx::elect_one()) ptx::mma_commit(&tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    // ------------------------------------------------ epilogue (128 threads)
    const int et = threadIdx.x - 64;   // 0..127
    const int q = warp & 3;            // TMEM lane quadrant this warp may access
    // this CTA's share of the zero rows, interleaved with its MMA units
    int z0 = 0, z1 = 0;
    if (!args.accumulate && args.n_zero > 0) {
      z0 = (int)((int64_t)args.n_zero * blockIdx.x / gridDim.x);
      z1 = (int)((int64_t)args.n_zero * (blockIdx.x + 1) / gridDim.x);
    }
    const int my_units = blockIdx.x < total_units ? (total_units - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int i = 0;
    OutT *out = reinterpret_cast<OutT *>(args.out);
    for (int u = blockIdx.x; u < total_units; u += gridDim.x, ++i) {
      // zero part i of my_units (written while unit i's mainloop runs)
      write_zero_rows<OutT>(args, z0 + (z1 - z0) * i / my_units, z0 + (z1 - z0) * (i + 1) / my_units, et);
      const TileMeta t = args.tiles[u / args.mblocks];
      const int m = (u % args.mblocks) * kBlockM + q * 32 + lane;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
      for (int c0 = 0; c0 < t.n_i; c0 += 32) {
        uint32_t v[32];
        ptx::tmem_ld_32x32b_x32(t_row + (uint32_t)c0, v);
        const int cid = (c0 + lane < t.n_i) ? __ldg(args.colids + t.col_off + c0 + lane) : -1;
        ptx::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int row = __shfl_sync(0xffffffffu, cid, j);
          if (row >= 0 && m < args.M) {
            OutT *p = out + (int64_t)row * args.ldc + m;
            float val = __uint_as_float(v[j]);
            if (args.accumulate) val += cvt_in<OutT>(*p);
            *p = cvt_out<OutT>(val);
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (my_units == 0) write_zero_rows<OutT>(args, z0, z1, et);
  }

  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

template <int BN, typename OutT>
cudaError_t launch_bn(const CUtensorMap &tmap, const GemmArgs &args, int grid, cudaStream_t stream) {
  auto kern = tw_gemm_sm100_kernel<BN, OutT>;
  const int smem = (int)Cfg<BN>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, stream>>>(tmap, args);
  return cudaGetLastError();
}

template <typename OutT>
cudaError_t launch_out(const CUtensorMap &tmap, const GemmArgs &args, int grid, cudaStream_t stream) {
  return args.block_n <= 128 ? launch_bn<128, OutT>(tmap, args, grid, stream)
                             : launch_bn<256, OutT>(tmap, args, grid, stream);
}

}  // namespace

cudaError_t launch_tw_gemm_sm100(const CUtensorMap &tmap, const GemmArgs &args, int out_dtype, int grid,
                                 cudaStream_t stream) {
  switch (out_dtype) {
    case TW_F32: return launch_out<float>(tmap, args, grid, stream);
    case TW_BF16: return launch_out<__nv_bfloat16>(tmap, args, grid, stream);
    case TW_F16: return launch_out<__half>(tmap, args, grid, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tw
