// K2: persistent grouped tile-wise sparse GEMM for sm_100a.
//
// Replaces, in one launch, the reference's per-call pipeline
//   _plan_tasks + gather_rows   (engine.py:61-69, :126-149)  -> row gather of
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
//     each 64 rows of 128 B (8-row swizzle atoms, SBO = 1 KB).  Gathered by
//     the 4 producer warps with 16-byte cp.async (zero-fill for padded rows
//     and tokens >= M), or -- kGather == kGatherTma -- by TMA gather4.
//   B operand (K-major, SW128): the packed weight image of the tile, one
//     1-D TMA bulk copy per stage (wrows x 128 B, pre-swizzled on the host).
//   D (TMEM, fp32): lane = token, column = tile column.  Double buffered
//     (2 x BN columns) so the epilogue of unit i overlaps the mainloop of i+1.
// Epilogue.  tcgen05.ld 32x32b: thread t of epilogue warp q owns token
//   m0 + 32q + t; for each tile column n the warp stores 32 consecutive
//   tokens to C^T[col_ids[n], m0 + 32q ...] -- one 128 B coalesced line (fp32).
//
// Warp roles (288 threads): w0-3 = A gather + W bulk copy (producer),
// w4 = MMA issuer + TMEM owner, w5-8 = epilogue (TMEM lane quadrant w % 4).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "tw_internal.h"
#include "tw_ptx.cuh"

namespace tw {

namespace {

constexpr int kProducerWarps = 4;
constexpr int kMmaWarp = kProducerWarps;
constexpr int kEpiWarp0 = kProducerWarps + 1;
constexpr int kThreads = (kProducerWarps + 1 + 4) * 32;
constexpr int kBlockM = 128;
constexpr int kBlockK = 64;
constexpr uint32_t kABytes = kBlockM * kBlockK * 2;  // 16 KB per stage
constexpr int kGatherCpAsync = 0;
constexpr int kGatherTma = 1;

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

// streaming (evict-first) store of one output element
template <typename T>
__device__ __forceinline__ void st_cs(T *p, T v) {
  if constexpr (sizeof(T) == 4) {
    __stcs(reinterpret_cast<float *>(p), *reinterpret_cast<float *>(&v));
  } else {
    __stcs(reinterpret_cast<unsigned short *>(p), *reinterpret_cast<unsigned short *>(&v));
  }
}

// Zero rows [r0, r1) of the zero list (pruned columns of C), full M.  Called
// by the 4 epilogue warps; warp ew writes rows r0+ew, r0+ew+4, ... with
// coalesced 16-byte streaming stores (512 B per warp instruction).  The next
// row id is prefetched so the index load latency is paid once.
template <typename OutT>
__device__ __forceinline__ void write_zero_rows(const GemmArgs &a, int r0, int r1, int ew, int lane) {
  const bool vec = ((a.ldc * (int64_t)sizeof(OutT)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0);
  const int64_t n16 = vec ? (int64_t)a.M * (int64_t)sizeof(OutT) / 16 : 0;
  const int64_t tail0 = n16 * 16 / (int64_t)sizeof(OutT);
  int r = r0 + ew;
  int row = r < r1 ? __ldg(a.zero_rows + r) : 0;
  for (; r < r1; r += 4) {
    const int next = (r + 4 < r1) ? __ldg(a.zero_rows + r + 4) : 0;
    OutT *base = reinterpret_cast<OutT *>(a.out) + (int64_t)row * a.ldc;
    uint4 *b16 = reinterpret_cast<uint4 *>(base);
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (int64_t i = lane; i < n16; i += 32) __stcs(b16 + i, z);
    for (int64_t i = tail0 + lane; i < a.M; i += 32) base[i] = cvt_out<OutT>(0.f);
    row = next;
  }
}

// Profiling hook: globaltimer stamps per CTA and work unit (tw_gemm_traced).
// Slots: 0 producer unit start, 1 producer unit issued, 2 MMA start, 3 MMA
// committed, 4 epilogue zero rows done, 5 accumulator ready, 6 unit stored.
__device__ __forceinline__ void trace_evt(const GemmArgs &a, int unit_i, int slot) {
  if (a.trace != nullptr && unit_i < 8) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[((int64_t)blockIdx.x * 8 + unit_i) * 8 + slot] = (int64_t)t;
  }
}

// First zero-list row owned by CTA c: zero rows are dealt out so that every
// CTA writes about the same number of output bytes (its MMA units' columns
// plus its zero rows), i.e. CTAs with one unit fewer take more zero rows.
__device__ __forceinline__ int zero_split(const GemmArgs &a, int c, int G, int units, int64_t unit_bytes,
                                          int64_t row_bytes) {
  if (c >= G) return a.n_zero;
  const int64_t q = units / G, rem = units % G;
  const int64_t before = (int64_t)c * q + min((int64_t)c, rem);
  const int64_t total = (int64_t)units * unit_bytes + (int64_t)a.n_zero * row_bytes;
  const int64_t want = total / G * c - before * unit_bytes;
  int64_t z = want <= 0 ? 0 : want / row_bytes;
  return (int)min(z, (int64_t)a.n_zero);
}

template <int BN, typename OutT, int kGather>
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
    // full: W bulk-copy arrive(+tx) and, for the cp.async gather, one
    // deferred arrival per producer thread
    const uint32_t full_count = kGather == kGatherTma ? 1u : 1u + kProducerWarps * 32u;
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], full_count);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 128);
    }
    ptx::fence_mbar_init();
    if (kGather == kGatherTma) ptx::prefetch_tmap(&tmap_at);
  }
  if (warp == kMmaWarp) ptx::tmem_alloc<C::kTmemCols>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp < kProducerWarps) {
    // ------------------------------------------------ producer warps
    const uint64_t keep = ptx::policy_evict_last();
    int stage = 0;
    uint32_t phase = 0;
    int ui = 0;
    for (int u = blockIdx.x; u < total_units; u += gridDim.x, ++ui) {
      const TileMeta t = args.tiles[u / args.mblocks];
      if (threadIdx.x == 0) trace_evt(args, ui, 0);
      const int m0 = (u % args.mblocks) * kBlockM;
      const int32_t *ki = args.kidx + t.kidx_off;
      const uint8_t *wsrc = args.wimg + t.w_off;
      if (kGather == kGatherTma) {
        if (warp != 0) continue;
        // lane l < 16 issues the gather4 pair for kept rows 4l..4l+3 of each
        // stage, indices loaded one stage ahead
        int4 rows_next = lane < 16 ? __ldg(reinterpret_cast<const int4 *>(ki) + lane) : make_int4(0, 0, 0, 0);
        for (int kb = 0; kb < t.nkb; ++kb) {
          const int4 rows = rows_next;
          if (kb + 1 < t.nkb && lane < 16) rows_next = __ldg(reinterpret_cast<const int4 *>(ki) + (kb + 1) * 16 + lane);
          if (lane == 0) {
            ptx::mbar_wait(&empty[stage], phase ^ 1);
            ptx::mbar_arrive_expect_tx(&full[stage], kABytes + (uint32_t)args.wbytes);
            ptx::bulk_g2s(sB + stage * C::kBBytes, wsrc + (int64_t)kb * args.wbytes, (uint32_t)args.wbytes,
                          &full[stage], keep);
          }
          __syncwarp();
          if (lane < 16) {
            uint8_t *a_dst = sA + stage * kABytes + lane * 512;
            ptx::tma_gather4(a_dst, &tmap_at, &full[stage], m0, rows, keep);
            ptx::tma_gather4(a_dst + 8192, &tmap_at, &full[stage], m0 + 64, rows, keep);
          }
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
      } else {
        // cp.async gather: warp w fills kept rows 16w..16w+15 of the stage.
        // Per instruction lanes 0-15 copy one row's 256 B token span (both
        // 64-token halves), lanes 16-31 the next row; 8 instructions/stage.
        const int j = lane & 15;             // 16-byte chunk within the 256 B span
        const int half = j >> 3, c = j & 7;  // token half, chunk within the 128 B row
        const int mcol = m0 + half * 64 + c * 8;
        const uint32_t src_bytes_m = mcol + 8 <= args.M ? 16u : (mcol < args.M ? (uint32_t)(args.M - mcol) * 2u : 0u);
        const __nv_bfloat16 *at = reinterpret_cast<const __nv_bfloat16 *>(args.at);
        int idx_next = __ldg(ki + warp * 16 + j);
        for (int kb = 0; kb < t.nkb; ++kb) {
          const int idx_mine = idx_next;
          if (kb + 1 < t.nkb) idx_next = __ldg(ki + (kb + 1) * kBlockK + warp * 16 + j);
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (warp == 0 && lane == 0) {
            ptx::mbar_arrive_expect_tx(&full[stage], (uint32_t)args.wbytes);
            ptx::bulk_g2s(sB + stage * C::kBBytes, wsrc + (int64_t)kb * args.wbytes, (uint32_t)args.wbytes,
                          &full[stage], keep);
          }
          uint8_t *a_stage = sA + stage * kABytes + half * 8192;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int rl = it * 2 + (lane >> 4);  // row within this warp's 16
            const int r = warp * 16 + rl;         // kept row within the stage
            const int krow = __shfl_sync(0xffffffffu, idx_mine, rl);
            const bool row_ok = kb * kBlockK + r < t.k_i;
            const uint32_t nbytes = row_ok ? src_bytes_m : 0u;
            const __nv_bfloat16 *src = at + (row_ok ? (int64_t)krow * args.lda + (nbytes ? mcol : 0) : 0);
            ptx::cp_async_16(a_stage + r * 128 + ((c ^ (r & 7)) * 16), src, nbytes);
          }
          ptx::cp_async_mbar_arrive_noinc(&full[stage]);
          if (++stage == C::kStages) { stage = 0; phase ^= 1; }
        }
        if (threadIdx.x == 0) trace_evt(args, ui, 1);
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------ MMA issuer
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t a_base = ptx::smem_u32(sA);
    const uint32_t b_base = ptx::smem_u32(sB);
    int ui = 0;
    for (int u = blockIdx.x; u < total_units; u += gridDim.x, ++ui) {
      const TileMeta t = args.tiles[u / args.mblocks];
      const uint32_t n_mma = (uint32_t)((t.n_i + 15) & ~15);
      const uint32_t idesc = args.idesc | ((n_mma >> 3) << 17);
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
      ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      if (lane == 0) trace_evt(args, ui, 2);
      for (int kb = 0; kb < t.nkb; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        if (kGather == kGatherCpAsync) ptx::fence_proxy_async_smem();  // cp.async wrote via the generic proxy
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
      if (lane == 0) trace_evt(args, ui, 3);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    // ------------------------------------------------ epilogue (128 threads)
    const int q = warp & 3;   // TMEM lane quadrant this warp may access
    const int ew = warp - kEpiWarp0;  // 0..3
    const int G = gridDim.x;
    const int64_t row_bytes = (int64_t)args.M * sizeof(OutT);
    const int64_t unit_bytes = (int64_t)kBlockM * args.avg_cols * sizeof(OutT);
    int z0 = 0, z1 = 0;
    if (!args.accumulate && args.n_zero > 0) {
      z0 = zero_split(args, blockIdx.x, G, total_units, unit_bytes, row_bytes);
      z1 = max(z0, zero_split(args, blockIdx.x + 1, G, total_units, unit_bytes, row_bytes));
    }
    const int my_units = blockIdx.x < total_units ? (total_units - 1 - blockIdx.x) / G + 1 : 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int i = 0;
    OutT *out = reinterpret_cast<OutT *>(args.out);
    for (int u = blockIdx.x; u < total_units; u += G, ++i) {
      const TileMeta t = args.tiles[u / args.mblocks];
      int cid[BN / 32];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c)
        cid[c] = (c * 32 + lane < t.n_i) ? __ldg(args.colids + t.col_off + c * 32 + lane) : -1;
      // zero part i of my_units (written while unit i's mainloop runs)
      write_zero_rows<OutT>(args, z0 + (z1 - z0) * i / my_units, z0 + (z1 - z0) * (i + 1) / my_units, ew, lane);
      if (ew == 0 && lane == 0) trace_evt(args, i, 4);
      const int m = (u % args.mblocks) * kBlockM + q * 32 + lane;
      const bool m_ok = m < args.M;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      if (ew == 0 && lane == 0) trace_evt(args, i, 5);
      const uint32_t t_row = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        if (c * 32 < t.n_i) {
          uint32_t v[32];
          ptx::tmem_ld_32x32b_x32(t_row + (uint32_t)(c * 32), v);
          ptx::tmem_ld_wait();
#pragma unroll
          for (int jj = 0; jj < 32; ++jj) {
            const int row = __shfl_sync(0xffffffffu, cid[c], jj);
            if (row >= 0 && m_ok) {
              OutT *p = out + (int64_t)row * args.ldc + m;
              float val = __uint_as_float(v[jj]);
              if (args.accumulate) {
                val += cvt_in<OutT>(*p);
                *p = cvt_out<OutT>(val);
              } else {
                st_cs(p, cvt_out<OutT>(val));
              }
            }
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
      if (ew == 0 && lane == 0) trace_evt(args, i, 6);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (my_units == 0) write_zero_rows<OutT>(args, z0, z1, ew, lane);
  }

  __syncthreads();
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

template <int BN, typename OutT, int kGather>
cudaError_t launch_bn(const CUtensorMap &tmap, const GemmArgs &args, int grid, cudaStream_t stream) {
  auto kern = tw_gemm_sm100_kernel<BN, OutT, kGather>;
  const int smem = (int)Cfg<BN>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kern<<<grid, kThreads, smem, stream>>>(tmap, args);
  return cudaGetLastError();
}

template <typename OutT, int kGather>
cudaError_t launch_out(const CUtensorMap &tmap, const GemmArgs &args, int grid, cudaStream_t stream) {
  return args.block_n <= 128 ? launch_bn<128, OutT, kGather>(tmap, args, grid, stream)
                             : launch_bn<256, OutT, kGather>(tmap, args, grid, stream);
}

template <int kGather>
cudaError_t launch_gather(const CUtensorMap &tmap, const GemmArgs &args, int out_dtype, int grid,
                          cudaStream_t stream) {
  switch (out_dtype) {
    case TW_F32: return launch_out<float, kGather>(tmap, args, grid, stream);
    case TW_BF16: return launch_out<__nv_bfloat16, kGather>(tmap, args, grid, stream);
    case TW_F16: return launch_out<__half, kGather>(tmap, args, grid, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

bool use_tma_gather() {
  static const bool v = [] {
    const char *e = std::getenv("TW_B200_GATHER");
    return e && std::strcmp(e, "tma") == 0;
  }();
  return v;
}

cudaError_t launch_tw_gemm_sm100(const CUtensorMap &tmap, const GemmArgs &args, int out_dtype, int grid,
                                 cudaStream_t stream) {
  return use_tma_gather() ? launch_gather<kGatherTma>(tmap, args, out_dtype, grid, stream)
                          : launch_gather<kGatherCpAsync>(tmap, args, out_dtype, grid, stream);
}

}  // namespace tw
