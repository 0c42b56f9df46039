// Write-path microbenchmark for the TW-GEMM epilogue design (B200).
// Measures achieved write GB/s for store shapes the epilogue can use:
//   stg32_w{4,16} : 4-byte STG, 128 B per warp instruction, contiguous
//   stg128_w4     : 16-byte STG, 512 B per warp instruction, contiguous
//   scat128_w4    : 128 B per warp instruction, consecutive instructions hit
//                   rows 16 KB apart (the C^T column-scatter pattern)
//   bulk{512,2048,8192}: TMA bulk smem->global stores of that many bytes,
//                   rows scattered 16 KB apart, issued by one thread
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                               \
    }                                                                         \
  } while (0)

constexpr int64_t kRowBytes = 16384;  // C^T row = 4096 tokens x fp32

__global__ void stg32(float *out, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) out[i] = 1.0f;
}
__global__ void stg128(float4 *out, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i < n; i += (int64_t)gridDim.x * blockDim.x) out[i] = make_float4(1, 1, 1, 1);
}
// warp w of CTA c owns a 32-token x (rows) patch: for each of its rows it
// writes 128 B (32 lanes x 4 B) at row*16KB + tokoff
__global__ void scat128(float *out, int rows, int tok_blocks) {
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nw = (gridDim.x * blockDim.x) >> 5;
  for (int tb = gw; tb < tok_blocks; tb += nw)
    for (int r = 0; r < rows; ++r) out[(int64_t)r * (kRowBytes / 4) + tb * 32 + lane] = 1.0f;
}
__global__ void bulk_store(char *out, int chunk, int64_t total) {
  extern __shared__ __align__(1024) char sm[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = 1;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const int64_t nchunks = total / chunk;
    const int64_t per_row = kRowBytes / chunk;
    int issued = 0;
    for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
      // scatter: consecutive chunks of a CTA land in different rows
      const int64_t row = c % (total / kRowBytes);
      const int64_t col = (c / (total / kRowBytes)) % per_row;
      char *dst = out + row * kRowBytes + col * chunk;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                   "r"((uint32_t)__cvta_generic_to_shared(sm + (issued & 7) * 2048 % 16384)), "r"(chunk)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      ++issued;
      asm volatile("cp.async.bulk.wait_group.read 16;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  const int64_t bytes = 48ll << 20;
  char *buf;
  CK(cudaMalloc(&buf, bytes * 4));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char *name, auto launch) {
    for (int i = 0; i < 3; ++i) launch(i);
    cudaEventRecord(a);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) launch(i);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-14s %8.1f GB/s  (%.2f us per 48 MB)\n", name, bytes * reps / (ms * 1e-3) / 1e9, ms * 1e3 / reps);
  };
  // rotate among 4 buffers (4 x 48 MB > L2) to force DRAM write-back
  auto off = [&](int i) { return buf + (i % 4) * bytes; };
  run("stg32_w4", [&](int i) { stg32<<<sms, 128>>>((float *)off(i), bytes / 4); });
  run("stg32_w16", [&](int i) { stg32<<<sms, 512>>>((float *)off(i), bytes / 4); });
  run("stg32_w64", [&](int i) { stg32<<<sms * 4, 512>>>((float *)off(i), bytes / 4); });
  run("stg128_w4", [&](int i) { stg128<<<sms, 128>>>((float4 *)off(i), bytes / 16); });
  run("stg128_w16", [&](int i) { stg128<<<sms, 512>>>((float4 *)off(i), bytes / 16); });
  run("scat128_w4", [&](int i) { scat128<<<sms, 128>>>((float *)off(i), (int)(bytes / kRowBytes), 4096 / 32); });
  run("scat128_w16", [&](int i) { scat128<<<sms, 512>>>((float *)off(i), (int)(bytes / kRowBytes), 4096 / 32); });
  CK(cudaFuncSetAttribute(bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  for (int chunk : {512, 1024, 2048, 4096, 8192, 16384}) {
    char name[32];
    snprintf(name, sizeof name, "bulk%d", chunk);
    run(name, [&](int i) { bulk_store<<<sms, 32, 16384>>>(off(i), chunk, bytes); });
  }
  CK(cudaDeviceSynchronize());
  CK(cudaGetLastError());
  return 0;
}
