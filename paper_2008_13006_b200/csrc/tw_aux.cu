// Auxiliary sm_100a kernels of libtw_b200.so:
//   prep   : A (fp32, ROW_/COL_MAJOR) -> A^T in bf16/fp16/fp32  (engine.py:129)
//   spmm   : K3, TEW residual CSC SpMM into C^T rows            (engine.py:167-181,
//            _kernels.py:30-41), fp32 mul-then-add in ascending p
//   exact  : bit-exact CUDA-core TW GEMM over a packed plan      (_kernels.py:13-27)
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
// ROW_MAJOR A (M x K) -> at (K x M): 64x64 tiles through shared memory,
// coalesced fp32 reads along K and coalesced 16-bit writes along M.
template <typename T>
__global__ void __launch_bounds__(256) prep_transpose_kernel(const float *__restrict__ a, int64_t m, int64_t k,
                                                             T *__restrict__ at, int64_t ldat) {
  __shared__ float tile[64][65];
  const int64_t m0 = (int64_t)blockIdx.y * 64, k0 = (int64_t)blockIdx.x * 64;
  const int tx = threadIdx.x & 63, ty = threadIdx.x >> 6;  // 64 x 4
  for (int r = ty; r < 64; r += 4) {
    const int64_t mm = m0 + r, kk = k0 + tx;
    tile[r][tx] = (mm < m && kk < k) ? __ldg(a + mm * k + kk) : 0.f;
  }
  __syncthreads();
  for (int r = ty; r < 64; r += 4) {
    const int64_t kk = k0 + r, mm = m0 + tx;
    if (kk < k && mm < m) at[kk * ldat + mm] = to_t<T>(tile[tx][r]);
  }
}
// COL_MAJOR A (its buffer is already A^T, K x M with row stride M): cast copy
template <typename T>
__global__ void __launch_bounds__(256) prep_cast_kernel(const float *__restrict__ a, int64_t m, int64_t k,
                                                        T *__restrict__ at, int64_t ldat) {
  const int64_t total = m * k;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t kk = i / m, mm = i - kk * m;
    at[kk * ldat + mm] = to_t<T>(__ldg(a + i));
  }
}

// ---------------------------------------------------------------- spmm (K3)
// One warp per output row j (CSC column j == CSR row of S^T), 4 consecutive
// tokens per lane (128 per warp).  Each stored entry p contributes
// v * at[row_idx[p], m] with a separately rounded multiply and add, in
// ascending p -- the exact operation sequence of spmm_accum.
template <typename AT, typename OutT>
__global__ void __launch_bounds__(256) spmm_csc_kernel(const AT *__restrict__ at, int64_t m, int64_t lda,
                                                       int64_t col_begin, int64_t n_cols,
                                                       const int32_t *__restrict__ col_ptr,
                                                       const int32_t *__restrict__ row_idx,
                                                       const float *__restrict__ values, OutT *__restrict__ ct,
                                                       int64_t ldc, int accumulate) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t jr = (int64_t)blockIdx.y * 8 + warp;  // output row (re-based)
  if (jr >= n_cols) return;
  const int64_t j = jr + col_begin;
  const int64_t mbase = (int64_t)blockIdx.x * 128 + lane * 4;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  const int p0 = __ldg(col_ptr + j), p1 = __ldg(col_ptr + j + 1);
  for (int p = p0; p < p1; ++p) {
    const int64_t kr = __ldg(row_idx + p);
    const float v = __ldg(values + p);
    const AT *arow = at + kr * lda;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t mm = mbase + e;
      if (mm < m) acc[e] = __fadd_rn(acc[e], __fmul_rn(v, to_f<AT>(arow[mm])));
    }
  }
  OutT *crow = ct + jr * ldc;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int64_t mm = mbase + e;
    if (mm < m) {
      float r = acc[e];
      if (accumulate) r = __fadd_rn(to_f<OutT>(crow[mm]), r);
      crow[mm] = to_t<OutT>(r);
    }
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
      if (n < t.n_i && kk < t.k_i) {
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

template <typename T>
cudaError_t prep_t(const float *a, int64_t m, int64_t k, int layout, T *at, int64_t ldat, cudaStream_t s) {
  if (layout == TW_ROW_MAJOR) {
    dim3 grid((unsigned)((k + 63) / 64), (unsigned)((m + 63) / 64));
    prep_transpose_kernel<T><<<grid, 256, 0, s>>>(a, m, k, at, ldat);
  } else {
    int64_t blocks = (m * k + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    prep_cast_kernel<T><<<(unsigned)blocks, 256, 0, s>>>(a, m, k, at, ldat);
  }
  return cudaGetLastError();
}

template <typename AT, typename OutT>
cudaError_t spmm_t(const void *at, int64_t m, int64_t lda, int64_t col_begin, int64_t n_cols, const int32_t *cp,
                   const int32_t *ri, const float *va, void *ct, int64_t ldc, int accumulate, cudaStream_t s) {
  dim3 grid((unsigned)((m + 127) / 128), (unsigned)((n_cols + 7) / 8));
  spmm_csc_kernel<AT, OutT><<<grid, 256, 0, s>>>(reinterpret_cast<const AT *>(at), m, lda, col_begin, n_cols, cp, ri,
                                                  va, reinterpret_cast<OutT *>(ct), ldc, accumulate);
  return cudaGetLastError();
}

template <typename AT>
cudaError_t spmm_at(const void *at, int64_t m, int64_t lda, int64_t cb, int64_t nc, const int32_t *cp,
                    const int32_t *ri, const float *va, void *ct, int64_t ldc, int out_dtype, int acc,
                    cudaStream_t s) {
  switch (out_dtype) {
    case TW_F32: return spmm_t<AT, float>(at, m, lda, cb, nc, cp, ri, va, ct, ldc, acc, s);
    case TW_BF16: return spmm_t<AT, __nv_bfloat16>(at, m, lda, cb, nc, cp, ri, va, ct, ldc, acc, s);
    case TW_F16: return spmm_t<AT, __half>(at, m, lda, cb, nc, cp, ri, va, ct, ldc, acc, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_prep(const float *a, int64_t m, int64_t k, int layout, void *at, int64_t ldat, int out_dtype,
                        cudaStream_t s) {
  switch (out_dtype) {
    case TW_F32: return prep_t<float>(a, m, k, layout, reinterpret_cast<float *>(at), ldat, s);
    case TW_BF16: return prep_t<__nv_bfloat16>(a, m, k, layout, reinterpret_cast<__nv_bfloat16 *>(at), ldat, s);
    case TW_F16: return prep_t<__half>(a, m, k, layout, reinterpret_cast<__half *>(at), ldat, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_spmm(const void *at, int at_dtype, int64_t m, int64_t lda, int64_t col_begin, int64_t n_cols,
                        const int32_t *cp, const int32_t *ri, const float *va, void *ct, int64_t ldc, int out_dtype,
                        int accumulate, cudaStream_t s) {
  switch (at_dtype) {
    case TW_F32: return spmm_at<float>(at, m, lda, col_begin, n_cols, cp, ri, va, ct, ldc, out_dtype, accumulate, s);
    case TW_BF16:
      return spmm_at<__nv_bfloat16>(at, m, lda, col_begin, n_cols, cp, ri, va, ct, ldc, out_dtype, accumulate, s);
    case TW_F16: return spmm_at<__half>(at, m, lda, col_begin, n_cols, cp, ri, va, ct, ldc, out_dtype, accumulate, s);
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
                                        at, m, lda, ct, ldc);
  }
  return cudaGetLastError();
}

}  // namespace tw
