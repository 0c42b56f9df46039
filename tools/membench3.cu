// L2 -> SM read microbenchmark for the TW-GEMM producer (B200).
// A^T: K=768 x M=4096 bf16 (6.3 MB, L2 resident).  Each CTA repeatedly
// gathers "stages" of 64 random kept rows x TB tokens into a shared-memory
// ring with 16-byte cp.async (the kernel's A path), optionally plus a 16 KB
// contiguous TMA bulk copy per stage (the W path).  Reports chip-wide GB/s.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench3 membench3.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int K = 768, M = 4096;

__device__ __forceinline__ void cp16(void *s, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}

// warps: producer warps per CTA; stages: ring depth (each 64 rows x TB tok)
template <int TB>
__global__ void gather(const __nv_bfloat16 *at, const int *kidx, int stages_total, int ring, float *sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  constexpr int kChunks = TB / 8, kRowsPerInst = 32 / kChunks;
  const int chunk = lane % kChunks, rsub = lane / kChunks;
  const int rows_per_warp = 64 / nw;
  const int mblocks = M / TB;
  for (int s = 0; s < stages_total; ++s) {
    const int g = blockIdx.x + s * gridDim.x;
    const int m0 = (g % mblocks) * TB;
    const int *ki = kidx + (g / mblocks % 6) * 64;
    uint8_t *dst = sm + (s % ring) * (64 * TB * 2);
    for (int it = 0; it < rows_per_warp / kRowsPerInst; ++it) {
      const int r = warp * rows_per_warp + it * kRowsPerInst + rsub;
      cp16(dst + r * TB * 2 + chunk * 16, at + (int64_t)ki[r] * M + m0 + chunk * 8);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 3;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (threadIdx.x == 0) sink[blockIdx.x] = (float)sm[5];
}

__global__ void plain_read(const uint4 *p, int64_t n16, int reps, float *sink) {
  uint32_t acc = 0;
  for (int r = 0; r < reps; ++r)
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
      uint4 v = __ldcg(p + i);
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  if (acc == 0x12345678) sink[0] = 1;
}

int main() {
  __nv_bfloat16 *at;
  int *kidx;
  float *sink;
  cudaMalloc(&at, (size_t)K * M * 2);
  cudaMemset(at, 0, (size_t)K * M * 2);
  std::vector<int> h(6 * 64);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (int)((i * 389 + 17) % K);
  cudaMalloc(&kidx, h.size() * 4);
  cudaMemcpy(kidx, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&sink, 4096 * 4);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char *name, double bytes, auto launch) {
    launch();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-26s %8.1f GB/s  (%.2f us/launch)\n", name, bytes * 10 / (ms * 1e-3) / 1e9, ms * 100);
  };
  const int stages = 64;
  for (int warps : {4, 8, 16}) {
    for (int ring : {4, 8}) {
      char nm[64];
      snprintf(nm, sizeof nm, "gather256_w%d_ring%d", warps, ring);
      int smem = ring * 64 * 256 * 2;
      cudaFuncSetAttribute(gather<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      run(nm, (double)sms * stages * 64 * 512, [&] { gather<256><<<sms, warps * 32, smem>>>(at, kidx, stages, ring, sink); });
      snprintf(nm, sizeof nm, "gather128_w%d_ring%d", warps, ring);
      smem = ring * 64 * 128 * 2;
      cudaFuncSetAttribute(gather<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      run(nm, (double)sms * stages * 64 * 256, [&] { gather<128><<<sms, warps * 32, smem>>>(at, kidx, stages, ring, sink); });
    }
  }
  run("plain_l2_read_w8", (double)K * M * 2 * 8,
      [&] { plain_read<<<sms, 256>>>((const uint4 *)at, (int64_t)K * M * 2 / 16, 8, sink); });
  run("plain_l2_read_w32", (double)K * M * 2 * 8,
      [&] { plain_read<<<sms * 4, 256>>>((const uint4 *)at, (int64_t)K * M * 2 / 16, 8, sink); });
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
