// Auxiliary sm_100a kernels of libtw_b200.so:
//   prep   : A (fp32, ROW_/COL_MAJOR) -> A^T in bf16/fp16/fp32  (engine.py:129)
//   spmm   : K3, TEW residual CSC SpMM into C^T rows            (engine.py:167-181,
//            _kernels.py:30-41), fp32 mul-then-add in ascending p
//   exact  : bit-exact CUDA-core TW GEMM over a packed plan      (_kernels.py:13-27)
#include <algorithm>
#include <type_traits>

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "tw_internal.h"

namespace tw {
namespace {

template <typename T>
__device__ __forceinline__ T to_t(float v);
template <>
__device__ __forceinline__ float to_t<float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 to_t<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ __half to_t<__half>(float v) { return __float2half_rn(v); }
template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }

// ---------------------------------------------------------------- prep
// A (fp32) -> A^T (K x M) in T, the reference's `at = a.array().T` copy
// (engine.py:129) with the cast fused.  kSplit (bf16 only): also the low
// parts, rows K..2K-1 = rn(a - rn(a)) -- the operand of TW_PLAN_SPLIT3.
template <typename T>
__device__ __forceinline__ void store8(T *dst, const float *v, bool vec) {
  if (vec) {
    if constexpr (sizeof(T) == 4) {
      reinterpret_cast<float4 *>(dst)[0] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4 *>(dst)[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else {
      uint32_t w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        T lo = to_t<T>(v[2 * i]), hi = to_t<T>(v[2 * i + 1]);
        w[i] = (uint32_t)*reinterpret_cast<uint16_t *>(&lo) | ((uint32_t)*reinterpret_cast<uint16_t *>(&hi) << 16);
      }
      *reinterpret_cast<uint4 *>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[i] = to_t<T>(v[i]);
  }
}

// ROW_MAJOR A (M x K): tiles of 128 tokens x 32 k through shared memory --
// 16-byte fp32 loads along K, 16-byte 16-bit stores along M (a 256 B run
// per A^T row per tile), conflict-free shared accesses (row stride 129).
template <typename T, bool kSplit>
__global__ void __launch_bounds__(256) prep_transpose_kernel(const float *__restrict__ a, int64_t m, int64_t k,
                                                             T *__restrict__ at, int64_t ldat) {
  __shared__ float tile[32][129];
  const int64_t m0 = (int64_t)blockIdx.x * 128, k0 = (int64_t)blockIdx.y * 32;
  const bool vin = (k % 4) == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int idx = threadIdx.x + it * 256;
    const int r = idx >> 3, c = idx & 7;  // token row r, k quad c
    const int64_t mm = m0 + r, kk = k0 + 4 * c;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    if (mm < m) {
      if (vin && kk + 4 <= k) {
        const float4 q = __ldg(reinterpret_cast<const float4 *>(a + mm * k + kk));
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (kk + i < k) v[i] = __ldg(a + mm * k + kk + i);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) tile[4 * c + i][r] = v[i];
  }
  __syncthreads();
  const bool vout = (ldat % 8) == 0 && (reinterpret_cast<uintptr_t>(at) & 15) == 0;
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int q = threadIdx.x + it * 256;
    const int kr = q >> 4, mc = (q & 15) * 8;  // k row, first of 8 tokens
    const int64_t kk = k0 + kr, mm = m0 + mc;
    if (kk >= k || mm >= m) continue;
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = tile[kr][mc + i];
    const bool full = mm + 8 <= m;
    if (full) {
      store8<T>(at + kk * ldat + mm, v, vout);
      if constexpr (kSplit) {
        float lo[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) lo[i] = v[i] - to_f<T>(to_t<T>(v[i]));
        store8<T>(at + (kk + k) * ldat + mm, lo, vout);
      }
    } else {
      for (int i = 0; i < 8 && mm + i < m; ++i) {
        at[kk * ldat + mm + i] = to_t<T>(v[i]);
        if constexpr (kSplit) at[(kk + k) * ldat + mm + i] = to_t<T>(v[i] - to_f<T>(to_t<T>(v[i])));
      }
    }
  }
}
// COL_MAJOR A (its buffer is already A^T, K x M with row stride M): cast copy,
// 8 tokens per thread (two 16-byte loads, one 16-byte store) when aligned
template <typename T, bool kSplit>
__global__ void __launch_bounds__(256) prep_cast_kernel(const float *__restrict__ a, int64_t m, int64_t k,
                                                        T *__restrict__ at, int64_t ldat) {
  const bool vec = (m % 8) == 0 && (ldat % 8) == 0 && (reinterpret_cast<uintptr_t>(a) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(at) & 15) == 0;
  const int64_t per_row = vec ? m / 8 : m;
  const int64_t total = per_row * k;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kk = i / per_row, j = i - kk * per_row;
    if (vec) {
      const float4 *src = reinterpret_cast<const float4 *>(a + kk * m + 8 * j);
      const float4 x0 = __ldg(src), x1 = __ldg(src + 1);
      float v[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      store8<T>(at + kk * ldat + 8 * j, v, true);
      if constexpr (kSplit) {
        float lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) lo[e] = v[e] - to_f<T>(to_t<T>(v[e]));
        store8<T>(at + (kk + k) * ldat + 8 * j, lo, true);
      }
    } else {
      const float v = __ldg(a + kk * m + j);
      at[kk * ldat + j] = to_t<T>(v);
      if constexpr (kSplit) at[(kk + k) * ldat + j] = to_t<T>(v - to_f<T>(to_t<T>(v)));
    }
  }
}

// ---------------------------------------------------------------- spmm (K3)
// One warp per (output row j, segment of 32*TOK tokens); j is a CSC column of
// S, i.e. a CSR row of S^T.  Lane l owns TOK = 16/sizeof(AT) consecutive
// tokens and reads them with one 16-byte load per stored entry.  The warp
// fetches 32 entries (row index, value) at a time into lanes and broadcasts
// them with shuffles; four entries' A^T loads are in flight at once.  Each
// entry p contributes v * at[row_idx[p], m] with a separately rounded
// multiply and add, in ascending p -- the exact operation sequence of
// spmm_accum (_kernels.py:30-41).
template <typename AT>
struct Vec16 {
  static constexpr int N = 16 / (int)sizeof(AT);
  __device__ __forceinline__ static void load(const AT *p, float (&o)[N]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4 *>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
    if constexpr (sizeof(AT) == 4) {
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = __uint_as_float(w[i]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint16_t b = (uint16_t)(w[i >> 1] >> ((i & 1) * 16));
        o[i] = to_f<AT>(*reinterpret_cast<const AT *>(&b));
      }
    }
  }
};

template <typename AT, typename OutT>
__global__ void __launch_bounds__(256) spmm_csc_kernel(const AT *__restrict__ at, int64_t m, int64_t lda,
                                                       int64_t col_begin, int64_t n_cols,
                                                       const int32_t *__restrict__ col_ptr,
                                                       const int32_t *__restrict__ row_idx,
                                                       const float *__restrict__ values, OutT *__restrict__ ct,
                                                       int64_t ldc, int accumulate, int vec_ok) {
  constexpr int TOK = Vec16<AT>::N;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t jr = (int64_t)blockIdx.y * 8 + warp;  // output row (re-based)
  if (jr >= n_cols) return;
  const int64_t j = jr + col_begin;
  const int64_t mbase = (int64_t)blockIdx.x * (32 * TOK) + lane * TOK;
  const bool full = vec_ok && mbase + TOK <= m;
  float acc[TOK];
#pragma unroll
  for (int x = 0; x < TOK; ++x) acc[x] = 0.f;
  const int p0 = __ldg(col_ptr + j), p1 = __ldg(col_ptr + j + 1);
  for (int pb = p0; pb < p1; pb += 32) {
    const int nb = min(32, p1 - pb);
    const int my_r = lane < nb ? __ldg(row_idx + pb + lane) : 0;
    const float my_v = lane < nb ? __ldg(values + pb + lane) : 0.f;
    int e = 0;
    for (; e + 4 <= nb; e += 4) {
      float a[4][TOK];
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t kr = __shfl_sync(0xffffffffu, my_r, e + u);
        v[u] = __shfl_sync(0xffffffffu, my_v, e + u);
        const AT *ap = at + kr * lda + mbase;
        if (full) {
          Vec16<AT>::load(ap, a[u]);
        } else {
#pragma unroll
          for (int x = 0; x < TOK; ++x) a[u][x] = mbase + x < m ? to_f<AT>(ap[x]) : 0.f;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int x = 0; x < TOK; ++x) acc[x] = __fadd_rn(acc[x], __fmul_rn(v[u], a[u][x]));
    }
    for (; e < nb; ++e) {
      const int64_t kr = __shfl_sync(0xffffffffu, my_r, e);
      const float v = __shfl_sync(0xffffffffu, my_v, e);
      const AT *ap = at + kr * lda + mbase;
      float a[TOK];
      if (full) {
        Vec16<AT>::load(ap, a);
      } else {
#pragma unroll
        for (int x = 0; x < TOK; ++x) a[x] = mbase + x < m ? to_f<AT>(ap[x]) : 0.f;
      }
#pragma unroll
      for (int x = 0; x < TOK; ++x) acc[x] = __fadd_rn(acc[x], __fmul_rn(v, a[x]));
    }
  }
  OutT *crow = ct + jr * ldc;
  constexpr int OV = 16 / (int)sizeof(OutT);  // outputs per 16-byte store
  if (full && (vec_ok & 2) && TOK % OV == 0) {
#pragma unroll
    for (int x0 = 0; x0 < TOK; x0 += OV) {
      uint4 *p = reinterpret_cast<uint4 *>(crow + mbase + x0);
      float r[OV];
#pragma unroll
      for (int x = 0; x < OV; ++x) r[x] = acc[x0 + x];
      if (accumulate) {
        const uint4 old = *p;
        const uint32_t w[4] = {old.x, old.y, old.z, old.w};
#pragma unroll
        for (int x = 0; x < OV; ++x) {
          float o;
          if constexpr (sizeof(OutT) == 4) {
            o = __uint_as_float(w[x]);
          } else {
            const uint16_t bits = (uint16_t)(w[x >> 1] >> ((x & 1) * 16));
            o = to_f<OutT>(*reinterpret_cast<const OutT *>(&bits));
          }
          r[x] = __fadd_rn(o, r[x]);
        }
      }
      uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
      for (int x = 0; x < OV; ++x) {
        if constexpr (sizeof(OutT) == 4) {
          w[x] = __float_as_uint(r[x]);
        } else {
          OutT o = to_t<OutT>(r[x]);
          w[x >> 1] |= (uint32_t)(*reinterpret_cast<uint16_t *>(&o)) << ((x & 1) * 16);
        }
      }
      *p = make_uint4(w[0], w[1], w[2], w[3]);
    }
    return;
  }
#pragma unroll
  for (int x = 0; x < TOK; ++x) {
    const int64_t mm = mbase + x;
    if (mm < m) {
      float r = acc[x];
      if (accumulate) r = __fadd_rn(to_f<OutT>(crow[mm]), r);
      crow[mm] = to_t<OutT>(r);
    }
  }
}

// acc + v * a for the tiled SpMM.  fp32 activations: a separately rounded
// multiply then add, the exact sequence of spmm_accum (_kernels.py:30-41);
// 16-bit activations (the TEW path, parity by rel-L2): one fused FMA.
template <typename AT>
__device__ __forceinline__ float spmm_madd(float acc, float v, float a) {
  if constexpr (sizeof(AT) == 4) {
    return __fadd_rn(acc, __fmul_rn(v, a));
  } else {
    return fmaf(v, a, acc);
  }
}

// PER consecutive activations from shared memory as fp32 (one vector load)
template <typename AT, int PER>
__device__ __forceinline__ void load_smem_vec(const AT *p, float (&o)[PER]) {
  if constexpr (std::is_same<AT, __nv_bfloat16>::value && PER == 4) {
    const uint2 u = *reinterpret_cast<const uint2 *>(p);  // bf16 -> fp32 is a 16-bit shift
    o[0] = __uint_as_float(u.x << 16);
    o[1] = __uint_as_float(u.x & 0xffff0000u);
    o[2] = __uint_as_float(u.y << 16);
    o[3] = __uint_as_float(u.y & 0xffff0000u);
  } else if constexpr (sizeof(AT) == 2 && PER == 4) {
    const uint2 u = *reinterpret_cast<const uint2 *>(p);
    const float2 lo = __half22float2(*reinterpret_cast<const __half2 *>(&u.x));
    const float2 hi = __half22float2(*reinterpret_cast<const __half2 *>(&u.y));
    o[0] = lo.x; o[1] = lo.y; o[2] = hi.x; o[3] = hi.y;
  } else if constexpr (sizeof(AT) == 4 && PER == 4) {
    const float4 f = *reinterpret_cast<const float4 *>(p);
    o[0] = f.x; o[1] = f.y; o[2] = f.z; o[3] = f.w;
  } else {
#pragma unroll
    for (int i = 0; i < PER; ++i) o[i] = to_f<AT>(p[i]);
  }
}
// PER consecutive outputs of row `crow` from token mt (accumulating if asked)
template <typename OutT, int PER>
__device__ __forceinline__ void store_vec(OutT *crow, int64_t mt, int64_t m, const float (&acc)[PER], int accumulate) {
#pragma unroll
  for (int x = 0; x < PER; ++x) {
    const int64_t mm = mt + x;
    if (mm < m) {
      float r = acc[x];
      if (accumulate) r = __fadd_rn(to_f<OutT>(crow[mm]), r);
      crow[mm] = to_t<OutT>(r);
    }
  }
}

// Shared-memory tiled variant (K3, default): the CTA copies the whole A^T
// token segment at[0:K, m0:m0+T] into shared memory once (cp.async), then
// its 8 warps walk columns j0, j0+1, ... of its column group: warp = column,
// lane = T/32 consecutive tokens, every stored entry read from smem.  A^T is
// read from L2 once per (segment, column group) instead of once per stored
// entry -- 2*nnz*M bytes of L2 traffic become ~groups*2*K*M.  Same exact
// multiply-then-add sequence in ascending p.
constexpr int kSpmmWarps = 32;
template <typename AT, typename OutT, int T>
__global__ void __launch_bounds__(kSpmmWarps * 32) spmm_tiled_kernel(const AT *__restrict__ at, int64_t m, int64_t k, int64_t lda,
                                                         int64_t col_begin, int64_t n_cols, int cols_per_cta,
                                                         const int32_t *__restrict__ col_ptr,
                                                         const int32_t *__restrict__ row_idx,
                                                         const float *__restrict__ values, OutT *__restrict__ ct,
                                                         int64_t ldc, int accumulate, int64_t smem_bytes) {
  extern __shared__ __align__(16) uint8_t sm_raw[];
  AT *sa = reinterpret_cast<AT *>(sm_raw);  // [K][T]
  constexpr int RB = T * (int)sizeof(AT);   // bytes per staged row
  constexpr int CPR = RB / 16;              // 16-byte chunks per row
  constexpr int PER = T / 32;               // tokens per lane
  const int64_t m0 = (int64_t)blockIdx.x * T;
  const int64_t j0 = (int64_t)blockIdx.y * cols_per_cta;
  const int64_t j1 = min(n_cols, j0 + cols_per_cta);
  // stage A^T[0:K, m0:m0+T] (zero-filled past M)
  for (int64_t c = threadIdx.x; c < k * CPR; c += blockDim.x) {
    const int64_t r = c / CPR, cc = c % CPR;
    const int64_t tok = m0 + cc * (16 / (int)sizeof(AT));
    const int64_t avail = m - tok;
    const uint32_t nbytes = avail >= 16 / (int)sizeof(AT) ? 16u : (avail > 0 ? (uint32_t)(avail * sizeof(AT)) : 0u);
    const AT *src = nbytes ? at + r * lda + tok : at;
    const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm_raw + r * RB + cc * 16);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(nbytes) : "memory");
  }
  // The column group's CSC slice (pointers, rows, values) is staged in the
  // shared memory left after the A^T segment when it fits; every warp then
  // reads its entries with broadcast shared loads instead of global loads
  // whose latency would sit on each column's critical path.
  // Entries are staged as interleaved (row, value) pairs -- one 8-byte
  // broadcast load per entry -- by 4-byte cp.async (no register round trip),
  // and converted to (row * T, value) once after the copy.
  const int64_t pg0 = __ldg(col_ptr + j0 + col_begin), pg1 = __ldg(col_ptr + j1 + col_begin);
  const int64_t ncg = j1 - j0;
  int32_t *s_ptr = reinterpret_cast<int32_t *>(sm_raw + k * RB);
  int2 *s_rv = reinterpret_cast<int2 *>(s_ptr + ((ncg + 2) & ~1));  // 8-byte aligned
  const bool staged = (int64_t)(k * RB) + (((ncg + 2) & ~1) + 2 * (pg1 - pg0)) * 4 <= smem_bytes;
  if (staged) {
    for (int64_t i = threadIdx.x; i <= ncg; i += blockDim.x)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(s_ptr + i)),
                   "l"(col_ptr + j0 + col_begin + i)
                   : "memory");
    for (int64_t i = threadIdx.x; i < pg1 - pg0; i += blockDim.x) {
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(s_rv + i);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(row_idx + pg0 + i) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d + 4), "l"(values + pg0 + i) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
  if (staged) {
    for (int64_t i = threadIdx.x; i <= ncg; i += blockDim.x) s_ptr[i] -= (int32_t)pg0;
    for (int64_t i = threadIdx.x; i < pg1 - pg0; i += blockDim.x) s_rv[i].x *= T;
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t mt = m0 + lane * PER;
  for (int64_t jr = j0 + warp; jr < j1; jr += kSpmmWarps) {
    // accumulating into an existing C^T (gemm_tew): a column without stored
    // entries leaves its row unchanged -- skip the read-modify-write
    if (accumulate && (staged ? s_ptr[jr - j0 + 1] == s_ptr[jr - j0]
                              : __ldg(col_ptr + jr + col_begin + 1) == __ldg(col_ptr + jr + col_begin)))
      continue;
    float acc[PER];
#pragma unroll
    for (int x = 0; x < PER; ++x) acc[x] = 0.f;
    if (staged) {
      const int q0 = s_ptr[jr - j0], q1 = s_ptr[jr - j0 + 1];
      int q = q0;
      const AT *sl = sa + lane * PER;
      for (; q + 4 <= q1; q += 4) {  // four entries' loads in flight, adds still in order
        float a[4][PER], v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int2 rv = s_rv[q + u];
          v[u] = __int_as_float(rv.y);
          load_smem_vec<AT, PER>(sl + rv.x, a[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int x = 0; x < PER; ++x) acc[x] = spmm_madd<AT>(acc[x], v[u], a[u][x]);
      }
      for (; q < q1; ++q) {
        float a[PER];
        const int2 rv = s_rv[q];
        load_smem_vec<AT, PER>(sl + rv.x, a);
#pragma unroll
        for (int x = 0; x < PER; ++x) acc[x] = spmm_madd<AT>(acc[x], __int_as_float(rv.y), a[x]);
      }
    } else {
      const int64_t j = jr + col_begin;
      const int p0 = __ldg(col_ptr + j), p1 = __ldg(col_ptr + j + 1);
      for (int pb = p0; pb < p1; pb += 32) {
        const int nb = min(32, p1 - pb);
        const int my_r = lane < nb ? __ldg(row_idx + pb + lane) : 0;
        const float my_v = lane < nb ? __ldg(values + pb + lane) : 0.f;
        for (int e = 0; e < nb; ++e) {
          const int r = __shfl_sync(0xffffffffu, my_r, e);
          const float v = __shfl_sync(0xffffffffu, my_v, e);
          float a[PER];
          load_smem_vec<AT, PER>(sa + (int64_t)r * T + lane * PER, a);
#pragma unroll
          for (int x = 0; x < PER; ++x) acc[x] = __fadd_rn(acc[x], __fmul_rn(v, a[x]));
        }
      }
    }
    store_vec<OutT, PER>(ct + jr * ldc, mt, m, acc, accumulate);
  }
}

// ---------------------------------------------------------------- exact GEMM
// Bit-exact TW GEMM: thread = token, 16 tile columns per block in registers,
// fp32 multiply then fp32 add in ascending kept-k order (mm_accum's
// sequence), weights read back from the swizzled plan image.
__global__ void __launch_bounds__(128) exact_gemm_kernel(const TileMeta *__restrict__ tiles,
                                                         const int32_t *__restrict__ kidx,
                                                         const int32_t *__restrict__ colids,
                                                         const uint8_t *__restrict__ wimg, int wbytes, int in_dtype,
                                                         const float *__restrict__ w32,
                                                         const int64_t *__restrict__ w32_off,
                                                         const float *__restrict__ at, int64_t m, int64_t lda,
                                                         float *__restrict__ ct, int64_t ldc) {
  const TileMeta t = tiles[blockIdx.y];
  const int n0 = blockIdx.z * 16;
  if (n0 >= t.n_i) return;
  const int64_t mm = (int64_t)blockIdx.x * 128 + threadIdx.x;
  float acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0.f;
  __shared__ float w_s[64][16];
  for (int kb = 0; kb < t.nkb; ++kb) {
    __syncthreads();
    for (int e = threadIdx.x; e < 64 * 16; e += 128) {
      const int r = e >> 4, j = e & 15, n = n0 + j, kk = kb * 64 + r;
      float w = 0.f;
      if (n < t.n_i && kk < t.k_i && w32 != nullptr) {  // TW_PLAN_F32_WEIGHTS: the reference's fp32 values
        w = __ldg(w32 + __ldg(w32_off + blockIdx.y) + (int64_t)kk * 128 + n);
      } else if (n < t.n_i && kk < t.k_i) {
        const int c = r >> 3, x = r & 7;
        const uint16_t bits = *reinterpret_cast<const uint16_t *>(
            wimg + t.w_off + (int64_t)kb * wbytes + n * 128 + ((c ^ (n & 7)) * 16) + x * 2);
        w = in_dtype == TW_BF16 ? __bfloat162float(__ushort_as_bfloat16(bits)) : __half2float(__ushort_as_half(bits));
      }
      w_s[r][j] = w;
    }
    __syncthreads();
    const int rend = min(64, t.k_i - kb * 64);
    if (mm < m) {
      for (int r = 0; r < rend; ++r) {
        const float a = __ldg(at + (int64_t)__ldg(kidx + t.kidx_off + kb * 64 + r) * lda + mm);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = __fadd_rn(acc[j], __fmul_rn(w_s[r][j], a));
      }
    }
  }
  if (mm < m) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int n = n0 + j;
      if (n < t.n_i) ct[(int64_t)colids[t.col_off + n] * ldc + mm] = acc[j];
    }
  }
}

__global__ void zero_rows_f32_kernel(const int32_t *__restrict__ rows, int n_rows, float *__restrict__ ct,
                                     int64_t m, int64_t ldc) {
  for (int r = blockIdx.y; r < n_rows; r += gridDim.y) {
    float *p = ct + (int64_t)rows[r] * ldc;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
      p[i] = 0.f;
  }
}

template <typename T, bool kSplit>
cudaError_t prep_t(const float *a, int64_t m, int64_t k, int layout, T *at, int64_t ldat, cudaStream_t s) {
  if (layout == TW_ROW_MAJOR) {
    dim3 grid((unsigned)((m + 127) / 128), (unsigned)((k + 31) / 32));
    prep_transpose_kernel<T, kSplit><<<grid, 256, 0, s>>>(a, m, k, at, ldat);
  } else {
    int64_t blocks = (m * k / 8 + 255) / 256 + 1;
    if (blocks > 148 * 16) blocks = 148 * 16;
    prep_cast_kernel<T, kSplit><<<(unsigned)blocks, 256, 0, s>>>(a, m, k, at, ldat);
  }
  return cudaGetLastError();
}

template <typename AT, typename OutT, int T>
cudaError_t spmm_tiled(const void *at, int64_t m, int64_t k, int64_t lda, int64_t col_begin, int64_t n_cols,
                       const int32_t *cp, const int32_t *ri, const float *va, void *ct, int64_t ldc, int accumulate,
                       cudaStream_t s) {
  // A^T segment + room for the column group's CSC slice (up to the 227 KB limit)
  const int smem = 232448;
  auto kern = spmm_tiled_kernel<AT, OutT, T>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t segs = (m + T - 1) / T;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  // enough CTAs for ~2 waves, as few column groups (A^T re-reads) as that allows
  // one CTA per SM (the A^T segment fills shared memory): as many column
  // groups as make whole waves -- floor(2 * SMs / segments) -- so the last
  // wave is not a sliver (each group re-reads the segment from L2)
  const int64_t groups =
      std::max<int64_t>(1, std::min<int64_t>((n_cols + kSpmmWarps - 1) / kSpmmWarps, (2 * sms) / segs));
  const int cpc = (int)((n_cols + groups - 1) / groups);
  dim3 grid((unsigned)segs, (unsigned)((n_cols + cpc - 1) / cpc));
  kern<<<grid, kSpmmWarps * 32, smem, s>>>(reinterpret_cast<const AT *>(at), m, k, lda, col_begin, n_cols, cpc, cp, ri, va,
                               reinterpret_cast<OutT *>(ct), ldc, accumulate, (int64_t)smem);
  return cudaGetLastError();
}

template <typename AT, typename OutT>
cudaError_t spmm_t(const void *at, int64_t m, int64_t k, int64_t lda, int64_t col_begin, int64_t n_cols,
                   const int32_t *cp, const int32_t *ri, const float *va, void *ct, int64_t ldc, int accumulate,
                   cudaStream_t s) {
  // tiled (shared-memory) kernel when a T >= 32 token segment of all K rows fits
  constexpr int64_t kMaxSmem = 200 * 1024;
  const bool al = (reinterpret_cast<uintptr_t>(at) & 15) == 0 && (lda * (int64_t)sizeof(AT)) % 16 == 0;
  if (al && k > 0) {
    if (k * 128 * (int64_t)sizeof(AT) <= kMaxSmem)
      return spmm_tiled<AT, OutT, 128>(at, m, k, lda, col_begin, n_cols, cp, ri, va, ct, ldc, accumulate, s);
    if (k * 64 * (int64_t)sizeof(AT) <= kMaxSmem)
      return spmm_tiled<AT, OutT, 64>(at, m, k, lda, col_begin, n_cols, cp, ri, va, ct, ldc, accumulate, s);
    if (k * 32 * (int64_t)sizeof(AT) <= kMaxSmem)
      return spmm_tiled<AT, OutT, 32>(at, m, k, lda, col_begin, n_cols, cp, ri, va, ct, ldc, accumulate, s);
  }
  constexpr int seg = 32 * (16 / (int)sizeof(AT));
  // bit 0: 16-byte activation loads; bit 1: 16-byte output stores
  const int vec_ok = (((reinterpret_cast<uintptr_t>(at) & 15) == 0) && ((lda * (int64_t)sizeof(AT)) % 16 == 0) ? 1 : 0) |
                     (((reinterpret_cast<uintptr_t>(ct) & 15) == 0) && ((ldc * (int64_t)sizeof(OutT)) % 16 == 0) ? 2 : 0);
  dim3 grid((unsigned)((m + seg - 1) / seg), (unsigned)((n_cols + 7) / 8));
  spmm_csc_kernel<AT, OutT><<<grid, 256, 0, s>>>(reinterpret_cast<const AT *>(at), m, lda, col_begin, n_cols, cp, ri,
                                                  va, reinterpret_cast<OutT *>(ct), ldc, accumulate, vec_ok);
  return cudaGetLastError();
}

template <typename AT>
cudaError_t spmm_at(const void *at, int64_t m, int64_t k, int64_t lda, int64_t cb, int64_t nc, const int32_t *cp,
                    const int32_t *ri, const float *va, void *ct, int64_t ldc, int out_dtype, int acc,
                    cudaStream_t s) {
  switch (out_dtype) {
    case TW_F32: return spmm_t<AT, float>(at, m, k, lda, cb, nc, cp, ri, va, ct, ldc, acc, s);
    case TW_BF16: return spmm_t<AT, __nv_bfloat16>(at, m, k, lda, cb, nc, cp, ri, va, ct, ldc, acc, s);
    case TW_F16: return spmm_t<AT, __half>(at, m, k, lda, cb, nc, cp, ri, va, ct, ldc, acc, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

// ------------------------------------------------------- pruning scores
// prune_stage's unit scores (pruning.py:293 and :316-318), the step before
// the TW path.  numpy reduces axis 0 of the C-contiguous
// K x N float64 score map row after row, and the K x n_t fancy-indexed copy
// s[:, cols] along axis 1 column after column -- both plain sequential
// float64 sums (pinned by tests/golden/golden_prune.npz) -- then divides by
// the count.  One thread per output keeps exactly that order.
__global__ void prune_col_mean_kernel(const double *__restrict__ s, int64_t k, int64_t n, double *__restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double acc = 0.0;
  for (int64_t r = 0; r < k; ++r) acc += s[r * n + j];
  out[j] = acc / (double)k;
}

__global__ void prune_row_mean_kernel(const double *__restrict__ s, int64_t k, int64_t n,
                                      const int32_t *__restrict__ cols, const int64_t *__restrict__ off,
                                      int64_t n_tiles, double *__restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n_tiles * k) return;
  const int64_t t = idx / k, r = idx % k;
  const int64_t c0 = off[t], c1 = off[t + 1];
  double acc = 0.0;
  for (int64_t c = c0; c < c1; ++c) acc += s[r * n + cols[c]];
  out[idx] = acc / (double)(c1 - c0);
}

cudaError_t launch_prune_means(const double *s, int64_t k, int64_t n, const int32_t *cols, const int64_t *off,
                               int64_t n_tiles, double *out, cudaStream_t st) {
  if (cols == nullptr) {
    prune_col_mean_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(s, k, n, out);
  } else {
    prune_row_mean_kernel<<<(unsigned)((n_tiles * k + 255) / 256), 256, 0, st>>>(s, k, n, cols, off, n_tiles, out);
  }
  return cudaGetLastError();
}

cudaError_t launch_prep(const float *a, int64_t m, int64_t k, int layout, void *at, int64_t ldat, int out_dtype,
                        cudaStream_t s) {
  switch (out_dtype) {
    case TW_F32: return prep_t<float, false>(a, m, k, layout, reinterpret_cast<float *>(at), ldat, s);
    case TW_BF16: return prep_t<__nv_bfloat16, false>(a, m, k, layout, reinterpret_cast<__nv_bfloat16 *>(at), ldat, s);
    case TW_F16: return prep_t<__half, false>(a, m, k, layout, reinterpret_cast<__half *>(at), ldat, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_prep_split(const float *a, int64_t m, int64_t k, int layout, void *at, int64_t ldat, cudaStream_t s) {
  return prep_t<__nv_bfloat16, true>(a, m, k, layout, reinterpret_cast<__nv_bfloat16 *>(at), ldat, s);
}

cudaError_t launch_spmm(const void *at, int at_dtype, int64_t m, int64_t k, int64_t lda, int64_t col_begin, int64_t n_cols,
                        const int32_t *cp, const int32_t *ri, const float *va, void *ct, int64_t ldc, int out_dtype,
                        int accumulate, cudaStream_t s) {
  if (m == 0 || n_cols <= 0) return cudaSuccess;  // nothing to write (and no zero-width column groups)
  switch (at_dtype) {
    case TW_F32: return spmm_at<float>(at, m, k, lda, col_begin, n_cols, cp, ri, va, ct, ldc, out_dtype, accumulate, s);
    case TW_BF16:
      return spmm_at<__nv_bfloat16>(at, m, k, lda, col_begin, n_cols, cp, ri, va, ct, ldc, out_dtype, accumulate, s);
    case TW_F16: return spmm_at<__half>(at, m, k, lda, col_begin, n_cols, cp, ri, va, ct, ldc, out_dtype, accumulate, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_exact(const tw_plan *p, const float *at, int64_t m, int64_t lda, float *ct, int64_t ldc,
                         cudaStream_t s) {
  const HostPlan &hp = p->host;
  if (!hp.zero_rows.empty() && m > 0) {
    const size_t nz = hp.zero_rows.size();
    dim3 g((unsigned)((m + 255) / 256 > 64 ? 64 : (m + 255) / 256), (unsigned)(nz > 65535 ? 65535 : nz));
    zero_rows_f32_kernel<<<g, 256, 0, s>>>(p->d_zero, (int)hp.zero_rows.size(), ct, m, ldc);
  }
  if (!hp.tiles.empty() && m > 0) {
    dim3 g((unsigned)((m + 127) / 128), (unsigned)hp.tiles.size(), (unsigned)((hp.wrows + 15) / 16));
    exact_gemm_kernel<<<g, 128, 0, s>>>(p->d_tiles, p->d_kidx, p->d_colids, p->d_wimg, hp.wrows * 128, hp.in_dtype,
                                        p->d_w32, p->d_w32_off, at, m, lda, ct, ldc);
  }
  return cudaGetLastError();
}

}  // namespace tw
