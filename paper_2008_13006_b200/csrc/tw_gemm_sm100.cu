// K2: persistent grouped tile-wise sparse GEMM for sm_100a.
//
// Replaces, in one launch, the reference's per-call pipeline
//   _plan_tasks + gather_rows   (engine.py:61-69, :126-149)  -> cp.async row
//                                 gather of the kept A^T rows into SW128 smem
//   group_by_shape + execute_batched + thread pool (engine.py:72-123)
//                               -> static per-CTA unit lists (host LPT,
//                                  tw_schedule.cpp) over persistent CTAs
//   mm_accum                    (_kernels.py:13-27) -> tcgen05.mma, fp32 TMEM
//   ct = zeros(N, M)            (engine.py:102) -> pruned C^T rows written as
//                                 zeros by the epilogue while it waits for
//                                 accumulators
//
// Work unit = (live tile, token block of nh x 128 tokens).  For tiles of up
// to 128 columns a unit has up to 256 tokens (two M=128 MMAs per k-step share
// the weight operand); for G = 256 a unit is 128 tokens x up to 256 columns.
//   A operand (MN-major, SW128): kept rows of A^T (K x M, M contiguous).  Per
//     pipeline stage 64 kept k x TB tokens, stored as TB/64 blocks of
//     [64 rows x 128 B] (8-row swizzle atoms: SBO = 1 KB, blocks LBO = 8 KB).
//     Gathered by 4 producer warps with 16-byte cp.async (zero fill for
//     padded rows and tokens >= M); completion via cp.async.mbarrier.arrive.
//   B operand (K-major, SW128): the packed weight image of the tile, one
//     1-D TMA bulk copy per stage (wrows x 128 B, pre-swizzled on the host).
//   D (TMEM, fp32): 2 x 256 columns (double buffered accumulators).
// Epilogue (8 warps).  The output C^T has one row per output column, so a
// unit's results are token segments of scattered rows.  Storing straight from
// the TMEM register layout (one token per lane) makes every store
// instruction hit a different row (1.7-1.9 TB/s in tools/membench2.cu);
// instead each 32-column chunk is staged through shared memory and written
// row by row, 16 B per lane, 512 B of one row per warp instruction (4.8 TB/s).
//
// Warp roles (416 threads): w0-3 producer (A gather + W bulk copy), w4 MMA
// issuer + TMEM owner, w5-12 epilogue (TMEM lane quadrant = warp % 4).
#include <cuda.h>
#include <cstdlib>
#include <type_traits>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tw_internal.h"
#include "tw_ptx.cuh"

namespace tw {

namespace {

#ifndef TW_PRODUCER_WARPS
#define TW_PRODUCER_WARPS 4
#endif
constexpr int kProducerWarps = TW_PRODUCER_WARPS;
constexpr int kRowsPerWarp = 64 / kProducerWarps;  // kept rows of a 64-k stage per producer warp
constexpr int kIdxLanes = kRowsPerWarp / 4;        // lanes that prefetch this warp's row indices
constexpr int kMmaWarp = kProducerWarps;
constexpr int kEpiWarp0 = kProducerWarps + 1;
constexpr int kEpiWarps = 8;
constexpr int kEpiThreads = kEpiWarps * 32;
constexpr int kThreads = (kProducerWarps + 1 + kEpiWarps) * 32;
constexpr int kBlockK = 64;
constexpr int kEpiBarrier = 1;  // named barrier id for the epilogue warps
// Per-CTA stage stream (HostSchedule::stream): 64 kept-row indices + a
// 4-int record per 64-k stage.  Each producer warp prefetches its 16 indices
// and the record of stage i + kIdxLook into its own shared-memory ring with
// cp.async while issuing stage i: no register ever waits on an index load.
constexpr int kIdxInts = 68;
constexpr int kSlotInts = kRowsPerWarp + 4;  // this warp's row indices + the 4-int record
constexpr int kIdxSlots = 8;
constexpr int kIdxLook = 4;

template <int BN>
struct Cfg {
  static constexpr int TB = BN <= 128 ? 256 : 128;           // max tokens per unit
  static constexpr int kHalves = TB / 128;                    // max M=128 MMAs per k-step
  static constexpr uint32_t kABytes = TB * kBlockK * 2;       // 32 KB | 16 KB
  static constexpr uint32_t kBBytes = BN * 128;               // 16 KB | 32 KB
  static constexpr uint32_t kAccCols = 256;                   // TMEM columns per accumulator
  static constexpr uint32_t kTmemCols = 2 * kAccCols;
  static constexpr int kChunk = 32;                           // accumulator columns per epilogue chunk
  static constexpr int kStageCols = kHalves == 2 ? kChunk : 2 * kChunk;  // staged C^T rows per chunk
  static constexpr uint32_t kStageBytes = kStageCols * TB * 4;          // 16 KB; two are used
  static constexpr uint32_t kColBytes = 2 * BN * 4;                     // col-id table, double buffered
  static constexpr uint32_t kZeroBytes = 8192;  // zero source block for TMA zero-row stores
  static constexpr uint32_t kFixed = 1024 /*align slack*/ + 2 * kStageBytes + kColBytes + 256 /*barriers*/ +
                                     kProducerWarps * kIdxSlots * kSlotInts * 4 + kZeroBytes;
  // as many 64-k pipeline stages as fit next to the epilogue buffers (4 for
  // G <= 128): bytes in flight per SM set the gather throughput
  static constexpr int kStages = (int)((232448u - kFixed) / (kABytes + kBBytes)) > 4
                                     ? 4
                                     : (int)((232448u - kFixed) / (kABytes + kBBytes));
  static constexpr uint32_t kSmem = kFixed + kStages * (kABytes + kBBytes);
  static_assert(kStages >= 3, "pipeline too shallow");
  static_assert(kSmem <= 232448u, "shared memory budget");
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

__device__ __forceinline__ void epi_sync() {
  asm volatile("bar.sync %0, %1;" ::"n"(kEpiBarrier), "n"(kEpiThreads) : "memory");
}

// 16 bytes of output (16/sizeof(OutT) consecutive tokens) from fp32 values
template <typename OutT>
__device__ __forceinline__ uint4 pack16(const float *v) {
  uint4 r;
  if constexpr (sizeof(OutT) == 4) {
    r = make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]), __float_as_uint(v[3]));
  } else {
    // paired conversions (one F2FP.PACK_AB per two values; the scalar
    // F2F.F16.F32 form is a low-throughput instruction on the epilogue path)
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (std::is_same<OutT, __half>::value) {
        const __half2 p = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t *>(&p);
      } else {
        const __nv_bfloat162 p = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
        w[i] = *reinterpret_cast<const uint32_t *>(&p);
      }
    }
    r = make_uint4(w[0], w[1], w[2], w[3]);
  }
  return r;
}
template <typename OutT>
__device__ __forceinline__ void unpack16_add(uint4 old, float *v) {
  const uint32_t w[4] = {old.x, old.y, old.z, old.w};
  if constexpr (sizeof(OutT) == 4) {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] += __uint_as_float(w[i]);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint16_t bits = (uint16_t)(w[i >> 1] >> ((i & 1) * 16));
      v[i] += cvt_in<OutT>(*reinterpret_cast<OutT *>(&bits));
    }
  }
}

// Epilogue value of a pruned output column: 0, or relu?(0 + bias) when the
// bias/ReLU epilogue is fused (trainer.py:246-248 applies both to every
// column of the layer output, pruned ones included).
__device__ __forceinline__ float const_row_value(const GemmArgs &a, int row) {
  if (a.bias == nullptr) return 0.f;
  const float b = __fadd_rn(0.f, __ldg(a.bias + row));
  return a.relu ? fmaxf(b, 0.f) : b;
}

// One constant row (a pruned column of C) written by one warp: coalesced
// 16-byte streaming stores, 512 B per instruction.
template <typename OutT>
__device__ __forceinline__ void write_zero_row(const GemmArgs &a, int row, int lane, bool vec) {
  OutT *base = reinterpret_cast<OutT *>(a.out) + (int64_t)row * a.ldc;
  const int64_t n16 = vec ? (int64_t)a.M * (int64_t)sizeof(OutT) / 16 : 0;
  uint4 *b16 = reinterpret_cast<uint4 *>(base);
  const float c = const_row_value(a, row);
  float cv[8] = {c, c, c, c, c, c, c, c};
  const uint4 z = pack16<OutT>(cv);
  for (int64_t i = lane; i < n16; i += 32) __stcs(b16 + i, z);
  for (int64_t i = n16 * 16 / (int64_t)sizeof(OutT) + lane; i < a.M; i += 32) base[i] = cvt_out<OutT>(c);
}

// One zero row by 1-D TMA bulk stores (up to 8 KB each) from the zeroed smem
// block, issued by lane 0: zero rows never occupy the LSU that the gathers
// need (tools/membench7.cu: 8 KB bulk stores reach 5.4 TB/s chip-wide).
// Falls back to STG when the row is not 16-byte aligned / sized.
template <typename OutT>
__device__ __forceinline__ void zero_row_bulk(const GemmArgs &a, int row, int lane, bool bulk_ok, bool vec,
                                              const uint8_t *zero_buf, uint32_t zero_bytes) {
  if (!bulk_ok || (a.bias != nullptr && const_row_value(a, row) != 0.f)) {
    write_zero_row<OutT>(a, row, lane, vec);
    return;
  }
  if (lane == 0) {
    char *dst = reinterpret_cast<char *>(a.out) + (int64_t)row * a.ldc * (int64_t)sizeof(OutT);
    const int64_t bytes = (int64_t)a.M * (int64_t)sizeof(OutT);
    for (int64_t off = 0; off < bytes; off += zero_bytes) {
      const uint32_t n = (uint32_t)min((int64_t)zero_bytes, bytes - off);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                   "r"(ptx::smem_u32(zero_buf)), "r"(n)
                   : "memory");
    }
    ptx::bulk_commit();
  }
}

// Epilogue store phase: this warp's kRows staged rows (starting at staged
// row r0; staged row r holds tile column col_of(r)) -> their C^T rows, SEG
// tokens from token m0 (row stride RS floats in the staging buffer).
template <typename OutT, int kRows, int RS, typename ColOf>
__device__ __forceinline__ void store_rows(const GemmArgs &args, OutT *out, const float *buf, int r0, int lane, int m0,
                                           int seg, ColOf col_of, const int32_t *ucol, int n_i, bool vec) {
  constexpr int V = 16 / (int)sizeof(OutT);
  constexpr int NIT = (RS / V + 31) / 32;  // 16-byte pieces per lane per row
  constexpr int kBatch = kRows * NIT * V > 32 ? (32 / (NIT * V) > 0 ? 32 / (NIT * V) : 1) : kRows;
#pragma unroll
  for (int rb0 = 0; rb0 < kRows; rb0 += kBatch) {
    float vals[kBatch][NIT][V];
    int orows[kBatch];
#pragma unroll
    for (int rb = 0; rb < kBatch; ++rb) {
      const int srow = r0 + rb0 + rb;
      const int col = col_of(srow);
      orows[rb] = (col < n_i && !(args.debug & 2)) ? ucol[col] : -1;
      const float *srow_p = buf + srow * RS;
#pragma unroll
      for (int n = 0; n < NIT; ++n) {
        const int tk = (n * 32 + lane) * V;
#pragma unroll
        for (int x = 0; x < V; x += 4) {
          const float4 f = tk < seg ? *reinterpret_cast<const float4 *>(srow_p + tk + x) : make_float4(0.f, 0.f, 0.f, 0.f);
          vals[rb][n][x] = f.x; vals[rb][n][x + 1] = f.y; vals[rb][n][x + 2] = f.z; vals[rb][n][x + 3] = f.w;
        }
      }
    }
#pragma unroll
    for (int rb = 0; rb < kBatch; ++rb) {
      if (orows[rb] < 0) continue;
      OutT *grow = out + (int64_t)orows[rb] * args.ldc + m0;
      if (args.bias != nullptr) {  // fused bias (+ ReLU): fp32 add then max, as trainer.py:246-248
        const float bz = __ldg(args.bias + orows[rb]);
#pragma unroll
        for (int n = 0; n < NIT; ++n)
#pragma unroll
          for (int x = 0; x < V; ++x) {
            const float z = __fadd_rn(vals[rb][n][x], bz);
            vals[rb][n][x] = args.relu ? fmaxf(z, 0.f) : z;
          }
      }
#pragma unroll
      for (int n = 0; n < NIT; ++n) {
        const int tk = (n * 32 + lane) * V;
        if (tk >= seg) continue;
        float *v = vals[rb][n];
        if (vec && m0 + tk + V <= args.M) {
          uint4 *p = reinterpret_cast<uint4 *>(grow + tk);
          if (args.accumulate) unpack16_add<OutT>(*p, v);
          const uint4 pk = pack16<OutT>(v);
          if (args.debug & 16) {  // experiment: staging reads without the global store
            if ((pk.x ^ pk.y ^ pk.z ^ pk.w) == 0x7fc00001u) __stcs(p, pk);
          } else {
            __stcs(p, pk);
          }
        } else {
#pragma unroll
          for (int x = 0; x < V; ++x) {
            if (m0 + tk + x < args.M) {
              float r = v[x];
              if (args.accumulate) r += cvt_in<OutT>(grow[tk + x]);
              grow[tk + x] = cvt_out<OutT>(r);
            }
          }
        }
      }
    }
  }
}

// Store phase for 16-bit staging: staged row r already holds the rounded
// OutT values of tile column col_of(r) (RS tokens, row stride RS); each lane
// moves 16 bytes (8 tokens) straight from shared to global memory.
template <typename OutT, int kRows, int RS, typename ColOf>
__device__ __forceinline__ void store_rows16(const GemmArgs &args, OutT *out, const float *buf_f, int r0, int lane,
                                             int m0, ColOf col_of, const int32_t *ucol, int n_i, bool vec) {
  if constexpr (sizeof(OutT) != 2) return;  // only instantiated for 16-bit outputs
  const OutT *buf = reinterpret_cast<const OutT *>(buf_f);
  constexpr int PER_ROW = RS / 8;  // 16-byte pieces per staged row (32 | 16)
  if constexpr (PER_ROW == 16 && kRows % 2 == 0) {
    // 128-token rows are 256 B: two rows per instruction (lanes 0-15 row
    // 2j, 16-31 row 2j+1), so no lane idles and the unit's last-chunk drain
    // issues half as many stores
    const int half = lane >> 4, piece = lane & 15;
    uint4 vals2[kRows / 2];
    int orows2[kRows / 2];
#pragma unroll
    for (int j = 0; j < kRows / 2; ++j) {
      const int srow = r0 + 2 * j + half;
      const int col = col_of(srow);
      orows2[j] = (col < n_i && !(args.debug & 2)) ? ucol[col] : -1;
      vals2[j] = *reinterpret_cast<const uint4 *>(buf + srow * RS + piece * 8);
    }
#pragma unroll
    for (int j = 0; j < kRows / 2; ++j) {
      if (orows2[j] < 0) continue;
      OutT *grow = out + (int64_t)orows2[j] * args.ldc + m0 + piece * 8;
      if (vec && m0 + piece * 8 + 8 <= args.M) {
        __stcs(reinterpret_cast<uint4 *>(grow), vals2[j]);
      } else {
        const uint16_t *hv = reinterpret_cast<const uint16_t *>(&vals2[j]);
#pragma unroll
        for (int x = 0; x < 8; ++x)
          if (m0 + piece * 8 + x < args.M) reinterpret_cast<uint16_t *>(grow)[x] = hv[x];
      }
    }
    return;
  }
  uint4 vals[kRows];
  int orows[kRows];
  const bool on = lane < PER_ROW;
#pragma unroll
  for (int rb = 0; rb < kRows; ++rb) {
    const int srow = r0 + rb;
    const int col = col_of(srow);
    orows[rb] = (col < n_i && !(args.debug & 2)) ? ucol[col] : -1;
    vals[rb] = on ? *reinterpret_cast<const uint4 *>(buf + srow * RS + lane * 8) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int rb = 0; rb < kRows; ++rb) {
    if (orows[rb] < 0 || !on) continue;
    OutT *grow = out + (int64_t)orows[rb] * args.ldc + m0 + lane * 8;
    if (vec && m0 + lane * 8 + 8 <= args.M) {
      __stcs(reinterpret_cast<uint4 *>(grow), vals[rb]);
    } else {
      const uint16_t *h = reinterpret_cast<const uint16_t *>(&vals[rb]);
#pragma unroll
      for (int x = 0; x < 8; ++x)
        if (m0 + lane * 8 + x < args.M) reinterpret_cast<uint16_t *>(grow)[x] = h[x];
    }
  }
}

// Profiling hook: globaltimer stamps per CTA and work unit (tw_gemm_traced).
// Slots: 0 producer unit start, 1 producer unit issued, 2 MMA start, 3 MMA
// committed, 4 epilogue started waiting, 5 accumulator ready, 6 unit stored.
__device__ __forceinline__ void trace_evt(const GemmArgs &a, int unit_i, int slot) {
  if (a.trace != nullptr && unit_i < 8) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[((int64_t)blockIdx.x * 8 + unit_i) * 8 + slot] = (int64_t)t;
  }
}
// per pipeline stage (first 32 of each CTA), after the unit table:
// slot 0 producer issued, 1 MMA saw it full, 2 MMA committed
__device__ __forceinline__ void trace_stage(const GemmArgs &a, int s, int slot) {
  if (a.trace != nullptr && s < 32) {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.trace[(int64_t)gridDim.x * 64 + ((int64_t)blockIdx.x * 32 + s) * 4 + slot] = (int64_t)t;
  }
}

// epilogue chunk events of each CTA's first unit (after the stage table)
// (SM clock cycles, not globaltimer: the intervals are sub-microsecond)
__device__ __forceinline__ void trace_epi(const GemmArgs &a, int idx) {
  if (a.trace != nullptr && idx < 32) {
    a.trace[(int64_t)gridDim.x * 192 + (int64_t)blockIdx.x * 32 + idx] = (int64_t)clock64();
  }
}

template <int BN, typename OutT>
__global__ void __launch_bounds__(kThreads, 1) tw_gemm_sm100_kernel(const __grid_constant__ GemmArgs args) {
  using C = Cfg<BN>;
  constexpr int TB = C::TB;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KB alignment (SW128 atoms) by pointer arithmetic on the __shared__
  // array, NOT through an integer cast: the compiler must keep seeing a
  // shared-space pointer, or every access below becomes a generic LD/ST that
  // queues in the LSU behind this SM's outstanding gathers and stores.
  uint8_t *smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = smem;
  uint8_t *sB = smem + C::kStages * C::kABytes;
  float *sStage = reinterpret_cast<float *>(sB + C::kStages * C::kBBytes);
  int32_t *sCol = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(sStage) + 2 * C::kStageBytes);
  uint64_t *full = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(sCol) + C::kColBytes);
  uint64_t *empty = full + C::kStages;
  uint64_t *tfull = empty + C::kStages;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tempty + 2);
  int32_t *sIdx = reinterpret_cast<int32_t *>(reinterpret_cast<uint8_t *>(full) + 256);
  uint8_t *sZero = reinterpret_cast<uint8_t *>(sIdx + kProducerWarps * kIdxSlots * kSlotInts);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int u_begin = __ldg(args.sched_off + blockIdx.x);
  const int u_end = __ldg(args.sched_off + blockIdx.x + 1);
  const int s_begin = __ldg(args.stream_off + blockIdx.x);
  const int n_st = __ldg(args.stream_off + blockIdx.x + 1) - s_begin;

  if (threadIdx.x == 0) {
    trace_evt(args, 7, 0);  // CTA start
    if (args.trace != nullptr) args.trace[((int64_t)blockIdx.x * 8 + 7) * 8 + 2] = (int64_t)clock64();
  }
  // Programmatic dependent launch: let the next kernel in the stream start
  // its CTAs (they wait in griddepcontrol.wait until this grid completes).
  // This CTA itself only touches immutable plan data (schedule, weights)
  // until its own griddepcontrol.wait below.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      ptx::mbar_init(&full[s], 1u + kProducerWarps * 32u);  // W bulk arrive(+tx) + one cp.async arrival per thread
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], kEpiThreads);
    }
    ptx::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < (int)(C::kZeroBytes / 16); i += kThreads)
    reinterpret_cast<uint4 *>(sZero)[i] = make_uint4(0, 0, 0, 0);
  ptx::fence_proxy_async_smem();  // zero block is read by TMA (async proxy)
  if (warp == kMmaWarp) ptx::tmem_alloc<C::kTmemCols>(tmem_holder);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp < kProducerWarps) {
    // ------------------------------------------------ producer warps
    // Warp w fills kept rows w*R..w*R+R-1 (R = kRowsPerWarp) of each 64-row stage.  A row's TB
    // tokens are TB/8 16-byte chunks; one instruction covers 32/(TB/8) rows.
    // Address work per copy is one shuffle of the row's byte offset plus a
    // 64-bit add: the row offsets (kept index * row pitch) are computed once
    // per stage by 16 lanes, one stage ahead.
    constexpr int kChunks = TB / 8;
    constexpr int kRowsPerInst = 32 / kChunks;
    const int chunk = lane % kChunks;
    const int rsub = lane / kChunks;
    const int blk = chunk >> 3, cc = chunk & 7;  // 64-token block, 16 B chunk in the 128 B row
    const uint64_t keep = ptx::policy_evict_last();
    const char *at_bytes = reinterpret_cast<const char *>(args.at);
    const int64_t pitch = args.lda * 2;
    int stage = 0;
    uint32_t phase = 0;
    int32_t *ring = sIdx + warp * (kIdxSlots * kSlotInts);  // this warp's index ring
    // stage k's 16 row indices of this warp (lanes 0-3) + record (lane 4)
    auto prefetch = [&](int k) {
      if (lane <= kIdxLanes) {
        const int32_t *src =
            args.stream + (int64_t)(s_begin + k) * kIdxInts + (lane < kIdxLanes ? warp * kRowsPerWarp + lane * 4 : 64);
        ptx::cp_async_16(ring + (k % kIdxSlots) * kSlotInts + lane * 4, src, 16);
      }
    };
    for (int k = 0; k < kIdxLook; ++k) {  // one cp.async group per prefetched stage
      if (k < n_st) prefetch(k);
      ptx::cp_async_commit();
    }
    // A^T may be produced by the previous kernel in the stream (PDL)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const bool traced = args.trace != nullptr;
    for (int i = 0; i < n_st; ++i) {
      const int32_t *slot = ring + (i % kIdxSlots) * kSlotInts;
      const long long c0 = traced ? clock64() : 0;  // SM-clock reads only when tracing
      // 4096 (experiment, needs 4 = no MMA): no back-pressure from the consumer
      if (!(args.debug & 4096)) ptx::mbar_wait(&empty[stage], phase ^ 1);
      const long long c1 = traced ? clock64() : 0;  // SM-clock reads only when tracing
      // stage i's indices were the (kIdxLook)-th most recent group
      ptx::cp_async_wait_group<kIdxLook - 1>();
      __syncwarp();
      const long long c2 = traced ? clock64() : 0;  // SM-clock reads only when tracing
      const int4 rec = *reinterpret_cast<const int4 *>(slot + kRowsPerWarp);
      if (threadIdx.x == 0 && (rec.w & (1 << 16))) trace_evt(args, rec.w & 0xffff, 0);
      const int nh = rec.z & 0xf;
      const bool active = chunk < nh * 16;  // token half present in this unit
      const int mcol = rec.y + chunk * 8;
      const uint32_t src_bytes_m =
          !active ? 0u : (mcol + 8 <= args.M ? 16u : (mcol < args.M ? (uint32_t)(args.M - mcol) * 2u : 0u));
      const char *lane_base = at_bytes + (src_bytes_m ? (int64_t)mcol * 2 : 0);
      if (warp == 0 && lane == 0) {
        if (args.debug & 64) {  // experiment: no weight copy
          ptx::mbar_arrive(&full[stage]);
        } else {
          ptx::mbar_arrive_expect_tx(&full[stage], (uint32_t)args.wbytes);
          ptx::bulk_g2s(sB + stage * C::kBBytes, args.wimg + rec.x, (uint32_t)args.wbytes, &full[stage], keep);
        }
      }
      uint8_t *a_warp = sA + stage * C::kABytes + blk * 8192 + warp * kRowsPerWarp * 128;
      // all 16 row indices into registers BEFORE the first cp.async: a shared
      // load issued after a cp.async waits for it in the same (MIO) pipe
      int rows[kRowsPerWarp];
#pragma unroll
      for (int v4 = 0; v4 < kRowsPerWarp / 4; ++v4) {
        const int4 r4 = reinterpret_cast<const int4 *>(slot)[v4];
        rows[4 * v4] = r4.x; rows[4 * v4 + 1] = r4.y; rows[4 * v4 + 2] = r4.z; rows[4 * v4 + 3] = r4.w;
      }
      if (args.debug & 8192) {  // experiment: synthetic rows (random, in range) instead of the kept lists
#pragma unroll
        for (int r = 0; r < kRowsPerWarp; ++r) rows[r] = ((warp * kRowsPerWarp + r) * 389 + i * 13 + blockIdx.x * 7) % 768;
      }
      // Fast path (warp-uniform): every row real and the unit's full token
      // range inside M -> plain 16-byte cp.async.  The zero-fill form (with a
      // source-size operand) only for padded rows / ragged token blocks.
      int min_row = rows[0];
#pragma unroll
      for (int r = 1; r < kRowsPerWarp; ++r) min_row = min(min_row, rows[r]);
      const bool fast = min_row >= 0 && rec.y + nh * 128 <= args.M && !(args.debug & 256);
      if (TB == 256 && nh == 1 && fast && !(args.debug & 512)) {
        // one 128-token half: 256 B per row, so each instruction carries two
        // rows (lanes 0-15 row 2it, 16-31 row 2it+1) -- half the LDGSTS count
        // of the one-row form, whose upper 16 lanes would idle
        const int ch2 = lane & 15, rs2 = lane >> 4, cc2 = ch2 & 7;
        const char *lb2 = at_bytes + (int64_t)(rec.y + ch2 * 8) * 2;
        uint8_t *aw2 = sA + stage * C::kABytes + (ch2 >> 3) * 8192 + warp * kRowsPerWarp * 128;
#pragma unroll
        for (int it = 0; it < kRowsPerWarp / 2; ++it) {
          const int rl = it * 2 + rs2;
          const int row = rs2 ? rows[2 * it + 1] : rows[2 * it];
          ptx::cp_async_16_full(aw2 + rl * 128 + ((cc2 ^ (rl & 7)) * 16), lb2 + (int64_t)row * pitch);
        }
      } else if (fast) {
#pragma unroll
        for (int it = 0; it < kRowsPerWarp / kRowsPerInst; ++it) {
          const int rl = it * kRowsPerInst + rsub;
          const int row = kRowsPerInst == 1 ? rows[it] : (rsub ? rows[it * kRowsPerInst + 1] : rows[it * kRowsPerInst]);
          if (active) ptx::cp_async_16_full(a_warp + rl * 128 + ((cc ^ (rl & 7)) * 16), lane_base + (int64_t)row * pitch);
        }
      } else {
#pragma unroll
        for (int it = 0; it < kRowsPerWarp / kRowsPerInst; ++it) {
          const int rl = it * kRowsPerInst + rsub;  // row within this warp's kRowsPerWarp
          const int row = kRowsPerInst == 1 ? rows[it] : (rsub ? rows[it * kRowsPerInst + 1] : rows[it * kRowsPerInst]);
          const uint32_t nbytes = row >= 0 ? src_bytes_m : 0u;
          if (active)
            ptx::cp_async_16(a_warp + rl * 128 + ((cc ^ (rl & 7)) * 16),
                             nbytes ? lane_base + (int64_t)row * pitch : at_bytes, nbytes);
        }
      }
      // Slot (i + kIdxLook) % kIdxSlots last held stage i + kIdxLook - kIdxSlots,
      // which this warp has issued and the MMA warp has committed (we passed
      // empty[i], so stage i - kStages is consumed): free to overwrite.
      if (i + kIdxLook < n_st) prefetch(i + kIdxLook);
      ptx::cp_async_mbar_arrive_noinc(&full[stage]);  // also covers the prefetch
      ptx::cp_async_commit();
      if (threadIdx.x == 0) trace_stage(args, i, 0);
      if (threadIdx.x == 0 && args.trace != nullptr && i < 32) {
        const long long c3 = clock64();
        args.trace[(int64_t)gridDim.x * 64 + ((int64_t)blockIdx.x * 32 + i) * 4 + 3] =
            (min(c1 - c0, 0xfffffLL) << 40) | (min(c2 - c1, 0xfffffLL) << 20) | min(c3 - c2, 0xfffffLL);
      }
      if (threadIdx.x == 0 && (rec.w & (1 << 17))) trace_evt(args, rec.w & 0xffff, 1);
      if (++stage == C::kStages) { stage = 0; phase ^= 1; }
    }
    ptx::cp_async_wait_group<0>();
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------ MMA issuer
    // Walks the same stage stream (records from the shared index ring).
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint32_t a_base = ptx::smem_u32(sA);
    const uint32_t b_base = ptx::smem_u32(sB);
    uint32_t d_tmem = tmem_base;
    for (int i = 0; i < n_st; ++i) {
      // full[stage] includes producer warp 0's cp.async arrival for stage i,
      // which covers its prefetch of stage i's record into its ring
      ptx::mbar_wait(&full[stage], phase);
      if (lane == 0) trace_stage(args, i, 1);
      const int4 rec = *reinterpret_cast<const int4 *>(sIdx + (i % kIdxSlots) * kSlotInts + kRowsPerWarp);
      const int nh = rec.z & 0xf, nk = (rec.z >> 4) & 0xf;
      const uint32_t n_mma = (uint32_t)(rec.z >> 8);
      const uint32_t idesc = args.idesc | ((n_mma >> 3) << 17);
      const bool first = rec.w & (1 << 16), last = rec.w & (1 << 17);
      if (first) {
        d_tmem = tmem_base + (uint32_t)(acc * C::kAccCols);
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        if (lane == 0) trace_evt(args, rec.w & 0xffff, 2);
      }
      if (!(args.debug & 8)) ptx::fence_proxy_async_smem();  // cp.async data was written through the generic proxy
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
        for (int kk = 0; kk < nk; ++kk) {
          const uint64_t bdesc = ptx::make_sw128_desc(b_base + stage * C::kBBytes + kk * 32, 16, 1024);
          for (int h = 0; h < nh; ++h) {
            const uint64_t adesc =
                ptx::make_sw128_desc(a_base + stage * C::kABytes + h * 16384 + kk * 2048, 8192, 1024);
            if (!(args.debug & 4))
              ptx::mma_f16_ss(d_tmem + h * 128, adesc, bdesc, idesc, (first && kk == 0) ? 0u : 1u);
          }
        }
        if (args.debug & 16384) ptx::mbar_arrive(&empty[stage]);  // experiment (with 4): plain arrive, no commit
        else ptx::mma_commit(&empty[stage]);
      }
      __syncwarp();
      if (lane == 0) trace_stage(args, i, 2);
      if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      if (last) {
        if (ptx::elect_one()) ptx::mma_commit(&tfull[acc]);
        __syncwarp();
        if (lane == 0) trace_evt(args, rec.w & 0xffff, 3);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ------------------------------------------------ epilogue (8 warps)
    // Warp e reads TMEM lane quadrant q = warp % 4 (tokens 32q..32q+31 of a
    // 128-token half); the warp pairs (e, e + 4) split the rest by `h`:
    //   mode A (TB = 256, two token halves): h = token half, 32-column chunks;
    //   mode B (TB = 128, G = 256):          h = 128-column half, 32-col chunks;
    //   mode C (TB = 256, one token half):   h = which 32 columns of a 64-column
    //                                         chunk -- all 8 warps stay busy.
    // Per chunk: tcgen05.ld (issued one chunk ahead) -> staging [row][token]
    // in smem -> each warp stores whole C^T row segments with 16-byte
    // streaming stores (512 B of one row per instruction).
    const int e = warp - kEpiWarp0;   // 0..7
    const int et = e * 32 + lane;     // 0..255
    const int q = warp & 3;
    const int h = e >> 2;
    const bool vec = ((args.ldc * (int64_t)sizeof(OutT)) % 16 == 0) && ((reinterpret_cast<uintptr_t>(args.out) & 15) == 0);
    const bool bulk_ok = vec && ((int64_t)args.M * (int64_t)sizeof(OutT)) % 16 == 0 && !(args.debug & 32);
    // zero rows of this CTA: warp e writes rows z0+e, z0+e+8, ... (8 KB TMA
    // bulk stores) while it waits for an accumulator (policy 0: any unit; 1:
    // the CTA's last unit only; 2: none), and the rest at the end
    // Zero rows: while units are in flight only warp 0 writes them, with at
    // most 3 bulk stores in flight -- the TMA engine also carries the
    // producer's weight loads, and a burst of zero-row stores queued ahead
    // of them stalls the pipeline; the remainder is split over all 8 warps
    // once the CTA's last accumulator has been drained.
    int zr = __ldg(args.zero_off + blockIdx.x);
    volatile int32_t *s_zdone = reinterpret_cast<volatile int32_t *>(tmem_holder + 1);
    // the output may be read / written by the previous kernel (PDL)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int z1 = (args.accumulate || args.keep_pruned || (args.debug & 1)) ? 0 : __ldg(args.zero_off + blockIdx.x + 1);
    constexpr int CK = C::kChunk;              // 32 accumulator columns per TMEM load
    int acc = 0;
    uint32_t acc_phase = 0;
    OutT *out = reinterpret_cast<OutT *>(args.out);
    for (int j = u_begin; j < u_end; ++j) {
      const int4 su = __ldg(args.sched + j);
      const TileMeta t = args.tiles[su.x];
      const int m0 = su.y, nh = su.z;
      // col ids double-buffered by unit parity: a fast warp may fill the next
      // unit's table while others still store this unit's last chunk
      int32_t *ucol = sCol + ((j - u_begin) & 1) * BN;
      if (et < BN) ucol[et] = et < t.n_i ? __ldg(args.colids + t.col_off + et) : -1;
      if (e == 0 && lane == 0) trace_evt(args, j - u_begin, 4);
      // wait for the accumulator, writing zero rows meanwhile
      // (non-blocking test_wait while there is filler work: try_wait would
      // suspend the warp for up to its time limit between zero rows)
      const bool fill = args.zero_policy == 0 || (args.zero_policy == 1 && j == u_end - 1);
      while (e == 0 && fill && zr < z1 && !ptx::mbar_test_wait(&tfull[acc], acc_phase)) {
        if (lane == 0 && bulk_ok) {
          if (args.debug & 2048) ptx::bulk_wait_read<2>(); else ptx::bulk_wait_read<0>();
        }
        zero_row_bulk<OutT>(args, __ldg(args.zero_rows + zr), lane, bulk_ok, vec, sZero, C::kZeroBytes);
        ++zr;
      }
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      epi_sync();  // sCol visible; previous unit's staging reads done
      if (e == 0 && lane == 0) trace_evt(args, j - u_begin, 5);
      if (args.debug & 32768) {  // experiment: drop the accumulator unread
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        continue;
      }
      const bool mode_a = TB == 256 && nh == 2;
      // 16-bit outputs without accumulate / bias are rounded while staging
      const bool stage16 = sizeof(OutT) == 2 && !args.accumulate && args.bias == nullptr && !(args.debug & 1024);
      const bool mode_c = TB == 256 && nh == 1;
      const int ccols = mode_c ? 2 * CK : CK;  // tile columns per chunk
      const int n_chunks = (min(t.n_i, 128) + ccols - 1) / ccols;
      // first tile column this warp loads for chunk c, and its TMEM column
      auto warp_col = [&](int c) { return mode_a ? c * CK : (mode_c ? c * ccols + h * CK : h * 128 + c * CK); };
      auto tmem_col = [&](int c) { return mode_a ? h * 128 + c * CK : warp_col(c); };
      auto have_chunk = [&](int c) { return warp_col(c) < t.n_i && !(args.debug & 128); };
      const uint32_t t_base = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * C::kAccCols);
      uint32_t v[CK];  // TMEM chunk in flight: loaded one chunk ahead of its use
      if (have_chunk(0)) ptx::tmem_ld_32x32b_x32(t_base + (uint32_t)tmem_col(0), v);
      for (int ci = 0; ci < n_chunks; ++ci) {
        float *buf = sStage + (ci & 1) * (C::kStageBytes / 4);  // double-buffered staging
        // 1) TMEM -> registers -> staging: mode A [32 cols][256 tok], modes
        //    B/C [h][32 cols][128 tok] (conflict-free: consecutive tokens)
        const bool have = have_chunk(ci);
        if (have) {
          ptx::tmem_ld_wait();
          if (j == u_begin && e == 0 && lane == 0) trace_epi(args, ci * 4 + 0);
          const int rs = mode_a ? 256 : 128;
          const int so = mode_a ? h * 128 + q * 32 + lane : h * CK * 128 + q * 32 + lane;
          if (stage16) {  // 16-bit outputs: round once here, stage half the bytes
            OutT *dst = reinterpret_cast<OutT *>(buf) + so;
#pragma unroll
            for (int jj = 0; jj < CK; ++jj) dst[jj * rs] = cvt_out<OutT>(__uint_as_float(v[jj]));
          } else {
            float *dst = buf + so;
#pragma unroll
            for (int jj = 0; jj < CK; ++jj) dst[jj * rs] = __uint_as_float(v[jj]);
          }
        }
        if (ci == n_chunks - 1) {
          // all of this warp's TMEM reads for the unit are done: hand the
          // accumulator back to the MMA warp before storing the last chunk
          ptx::tc_fence_before();
          ptx::mbar_arrive(&tempty[acc]);
        }
        if (j == u_begin && e == 0 && lane == 0) trace_epi(args, ci * 4 + 1);
        // One barrier per chunk: it publishes buf[ci & 1] and (double
        // buffering) guarantees every warp finished storing chunk ci - 1,
        // whose buffer chunk ci + 1 will overwrite.
        epi_sync();
        // next chunk's TMEM load overlaps this chunk's global stores
        if (ci + 1 < n_chunks && have_chunk(ci + 1)) ptx::tmem_ld_32x32b_x32(t_base + (uint32_t)tmem_col(ci + 1), v);
        if (j == u_begin && e == 0 && lane == 0) trace_epi(args, ci * 4 + 2);
        // 2) staged rows -> global.  All shared-memory reads of a batch are
        // issued before its first global store: an LDS queued behind a
        // backpressured STG in the same pipe would wait for it.
        if (stage16) {
          if (mode_a)
            store_rows16<OutT, 4, 256>(args, out, buf, e * 4, lane, m0, [&](int r) { return ci * CK + r; }, ucol,
                                       t.n_i, vec);
          else
            store_rows16<OutT, 8, 128>(
                args, out, buf, e * 8, lane, m0,
                [&](int r) { return mode_c ? ci * ccols + r : (r < CK ? 0 : 128) + ci * CK + (r % CK); }, ucol,
                t.n_i, vec);
        } else if (mode_a) {
          store_rows<OutT, 4, 256>(args, out, buf, e * 4, lane, m0, 256, [&](int r) { return ci * CK + r; }, ucol,
                                   t.n_i, vec);
        } else {
          store_rows<OutT, 8, 128>(args, out, buf, e * 8, lane, m0, 128,
                                   [&](int r) { return mode_c ? ci * ccols + r : (r < CK ? 0 : 128) + ci * CK + (r % CK); },
                                   ucol, t.n_i, vec);
        }
        if (j == u_begin && e == 0 && lane == 0) trace_epi(args, ci * 4 + 3);
      }
      if (e == 0 && lane == 0) trace_evt(args, j - u_begin, 6);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    if (e == 0 && lane == 0) *s_zdone = zr;
    epi_sync();
    for (zr = *s_zdone + e; zr < z1; zr += kEpiWarps)
      zero_row_bulk<OutT>(args, __ldg(args.zero_rows + zr), lane, bulk_ok, vec, sZero, C::kZeroBytes);
    if (lane == 0) ptx::bulk_wait<0>();  // bulk stores performed (and smem read) before exit
    if (e == 0 && lane == 0) {
      trace_evt(args, 7, 1);  // last zero row issued
      if (args.trace != nullptr) args.trace[((int64_t)blockIdx.x * 8 + 7) * 8 + 3] = (int64_t)clock64();
    }
  }

  __syncthreads();
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<C::kTmemCols>(tmem_base);
  }
}

template <int BN, typename OutT>
cudaError_t launch_bn(const GemmArgs &args, int grid, cudaStream_t stream) {
  auto kern = tw_gemm_sm100_kernel<BN, OutT>;
  const int smem = (int)Cfg<BN>::kSmem;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  // programmatic dependent launch (TW_B200_PDL=0 disables): the next grid's
  // CTAs may start as SMs free up; griddepcontrol.wait orders memory
  static const bool pdl = [] {
    const char *e = std::getenv("TW_B200_PDL");
    return !(e && e[0] == '0');
  }();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = (size_t)smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, kern, args);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <typename OutT>
cudaError_t launch_out(const GemmArgs &args, int grid, cudaStream_t stream) {
  return args.block_n <= 128 ? launch_bn<128, OutT>(args, grid, stream) : launch_bn<256, OutT>(args, grid, stream);
}

}  // namespace

int tokens_per_unit(int block_n) { return block_n <= 128 ? Cfg<128>::TB : Cfg<256>::TB; }

cudaError_t launch_tw_gemm_sm100(const GemmArgs &args, int out_dtype, int grid, cudaStream_t stream) {
  switch (out_dtype) {
    case TW_F32: return launch_out<float>(args, grid, stream);
    case TW_BF16: return launch_out<__nv_bfloat16>(args, grid, stream);
    case TW_F16: return launch_out<__half>(args, grid, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace tw
