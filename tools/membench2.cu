// Write-path microbenchmark 2: the TW epilogue's C^T access pattern.
// C^T is N x M fp32 (M = 4096 tokens -> 16 KB rows).  A "unit" is (tile t,
// m-block b): 128 rows (the tile's columns; contiguous row ids here) x TB
// tokens.  CTA c handles units c, c+G, ... (unit u -> t = u / (M/TB),
// b = u % (M/TB)), its 4 warps each writing rows j = w, w+4, ...:
//   mode 0: lane writes 4 B  -> 128 B per warp instruction (current epilogue)
//   mode 1: lane writes 16 B -> 512 B per warp instruction
// Also the "row-major" variant: the same bytes written with each unit owning
// TB/128 whole... see main.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench2 membench2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int M = 4096;
constexpr int N = 3072;

template <int MODE>
__global__ void unit_store(float *out, int tb, int rows_per_unit) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int mblocks = M / tb;
  const int units = (N / rows_per_unit) * mblocks;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int t = u / mblocks, b = u % mblocks;
    for (int j = w; j < rows_per_unit; j += nw) {
      float *row = out + (int64_t)(t * rows_per_unit + j) * M + b * tb;
      if (MODE == 0) {
        for (int x = lane; x < tb; x += 32) __stcs(row + x, 1.0f);
      } else {
        for (int x = lane * 4; x < tb; x += 128) __stcs(reinterpret_cast<float4 *>(row + x), make_float4(1, 1, 1, 1));
      }
    }
  }
}

// same units, but the 4 warps split the unit by token quarter and walk all
// 128 rows (each warp instruction = one row, 1/4 of the unit's token span)
__global__ void unit_store_colwalk(float *out, int tb) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int mblocks = M / tb;
  const int units = (N / 128) * mblocks;
  for (int u = blockIdx.x; u < units; u += gridDim.x) {
    const int t = u / mblocks, b = u % mblocks;
    for (int j = 0; j < 128; ++j) {
      float *row = out + (int64_t)(t * 128 + j) * M + b * tb + w * (tb / 4);
      for (int x = lane * 4; x < tb / 4; x += 128) __stcs(reinterpret_cast<float4 *>(row + x), make_float4(1, 1, 1, 1));
    }
  }
}

int main() {
  const int64_t bytes = (int64_t)M * N * 4;
  char *buf;
  if (cudaMalloc(&buf, bytes * 4) != cudaSuccess) return 1;
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
    printf("%-28s %8.1f GB/s  (%.2f us per %lld MB)\n", name, bytes * reps / (ms * 1e-3) / 1e9, ms * 1e3 / reps,
           (long long)(bytes >> 20));
  };
  auto off = [&](int i) { return (float *)(buf + (i % 4) * bytes); };
  char name[64];
  for (int tb : {128, 256, 512, 1024, 4096}) {
    for (int warps : {4, 8}) {
      snprintf(name, sizeof name, "tb%d_w%d_lane4B", tb, warps);
      run(name, [&](int i) { unit_store<0><<<sms, warps * 32>>>(off(i), tb, 128); });
      snprintf(name, sizeof name, "tb%d_w%d_lane16B", tb, warps);
      run(name, [&](int i) { unit_store<1><<<sms, warps * 32>>>(off(i), tb, 128); });
    }
    snprintf(name, sizeof name, "tb%d_colwalk", tb);
    run(name, [&](int i) { unit_store_colwalk<<<sms, 128>>>(off(i), tb); });
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
