// TMA 1-D bulk store throughput (B200): each CTA's elected thread streams
// cp.async.bulk.global.shared::cta copies of S bytes from a zeroed smem block
// to rows 16 KB apart (the C^T zero-row pattern), optionally while 4 warps
// run the TW producer's 16-byte cp.async gathers.  Reports chip GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench7 membench7.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__global__ void bulk_store(char *out, int64_t row_bytes, int rows_per_cta, int S, int inflight, int gather,
                           const __nv_bfloat16 *at, long long *cyc) {
  extern __shared__ __align__(1024) char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 16384 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  long long t0 = clock64();
  if (warp == 0) {
    if (lane == 0) {
      const uint32_t src = (uint32_t)__cvta_generic_to_shared(sm);
      int issued = 0;
      for (int r = 0; r < rows_per_cta; ++r) {
        char *row = out + ((int64_t)blockIdx.x * rows_per_cta + r) * row_bytes;
        for (int64_t off = 0; off < row_bytes; off += S) {
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(row + off), "r"(src), "r"(S)
                       : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          if (++issued > inflight) asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
        }
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      cyc[blockIdx.x] = clock64() - t0;
    }
  } else if (gather && warp <= 4) {
    char *dst = sm + 16384;
    for (int i = 0; i < 256; ++i) {
      for (int it = 0; it < 16; ++it) {
        const int r = (warp - 1) * 16 + it;
        const int krow = (r * 389 + i * 13 + blockIdx.x * 7) % 768;
        const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst + (i % 4) * 32768 + r * 512 + lane * 16);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d),
                     "l"(at + (int64_t)krow * 4096 + ((blockIdx.x * 256 + i * 256) % 4096) + lane * 8)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 3;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t row_bytes = 16384;
  const int rows_per_cta = 64;  // 1 MB per CTA
  char *out;
  __nv_bfloat16 *at;
  long long *cyc;
  cudaMalloc(&out, (size_t)sms * rows_per_cta * row_bytes * 2);
  cudaMalloc(&at, 768 * 4096 * 2);
  cudaMemset(at, 0, 768 * 4096 * 2);
  cudaMalloc(&cyc, 1024 * 8);
  const int smem = 16384 + 4 * 32768;
  cudaFuncSetAttribute(bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int gather = 0; gather < 2; ++gather)
    for (int S : {1024, 2048, 4096, 8192, 16384}) {
      for (int r = 0; r < 2; ++r) bulk_store<<<sms, 160, smem>>>(out, row_bytes, rows_per_cta, S, 16, gather, at, cyc);
      cudaEventRecord(a);
      bulk_store<<<sms, 160, smem>>>(out, row_bytes, rows_per_cta, S, 16, gather, at, cyc);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)sms * rows_per_cta * row_bytes;
      printf("bulk store S=%5d gather=%d: %7.1f GB/s chip (%.1f us)\n", S, gather, bytes / (ms * 1e-3) / 1e9,
             ms * 1e3);
    }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
