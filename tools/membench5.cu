// Write-pattern microbenchmark 5: "lane owns a row" epilogue (TMEM lane =
// output row) vs "warp owns a row" (smem-staged) for the TW C^T layout.
// Unit = 128 rows (scattered, ~2x spaced like a 50%-pruned tile) x TB tokens.
//   laneRow : thread t of warp w writes row (32*q + t)'s token slice with
//             consecutive 16 B stores (warp instruction = 32 rows x 16 B)
//   warpRow : warp writes one row's TB tokens per pass (512 B / instruction)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench5 membench5.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int M = 4096, N = 3072;

__device__ __forceinline__ int row_of(int t, int j) { return (t * 256 + 2 * j) % N; }  // ~50% of columns

template <int TB>
__global__ void lane_row(float *out, int units) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q = w & 3, h = w >> 2;  // 8 warps: quadrant, token half
  const int mblocks = M / TB;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int t = u / mblocks, m0 = (u % mblocks) * TB;
    const int r = row_of(t, q * 32 + lane);
    float4 *p = reinterpret_cast<float4 *>(out + (int64_t)r * M + m0 + h * (TB / 2));
#pragma unroll 8
    for (int i = 0; i < TB / 2 / 4; ++i) __stcs(p + i, make_float4(1, 1, 1, 1));
  }
}

template <int TB>
__global__ void warp_row(float *out, int units) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mblocks = M / TB;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int t = u / mblocks, m0 = (u % mblocks) * TB;
    for (int j = w; j < 128; j += 8) {
      float4 *p = reinterpret_cast<float4 *>(out + (int64_t)row_of(t, j) * M + m0);
      for (int i = lane; i < TB / 4; i += 32) __stcs(p + i, make_float4(1, 1, 1, 1));
    }
  }
}

int main() {
  const int64_t bytes = (int64_t)M * N * 4;
  char *buf;
  cudaMalloc(&buf, bytes * 4);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int units128 = (N / 256) * (M / 128), units256 = (N / 256) * (M / 256);  // tiles of 128 rows over 256 cols
  const double wbytes = (double)(N / 2) * M * 4;  // half the rows are written
  auto run = [&](const char *name, auto launch) {
    for (int i = 0; i < 3; ++i) launch(i);
    cudaEventRecord(a);
    for (int i = 0; i < 20; ++i) launch(i);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-16s %8.1f GB/s (%.2f us for %.0f MB)\n", name, wbytes * 20 / (ms * 1e-3) / 1e9, ms * 1e3 / 20, wbytes / 1e6);
  };
  auto off = [&](int i) { return (float *)(buf + (i % 4) * bytes); };
  run("laneRow TB256", [&](int i) { lane_row<256><<<sms, 256>>>(off(i), units256); });
  run("warpRow TB256", [&](int i) { warp_row<256><<<sms, 256>>>(off(i), units256); });
  run("laneRow TB128", [&](int i) { lane_row<128><<<sms, 256>>>(off(i), units128); });
  run("warpRow TB128", [&](int i) { warp_row<128><<<sms, 256>>>(off(i), units128); });
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
