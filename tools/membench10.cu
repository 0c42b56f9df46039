// Does the A^T geometry change the gather rate?  The kernel-like producer of
// membench9 (4 warps, SW128 destinations, mbarrier completion, 16 KB TMA
// weight load per stage, 4 stages of 64 kept rows x 256 tokens in flight) on
// the C2a and C5 layer shapes, with the row pitch padded or not, and units
// taken in the kernel's order (unit u = CTA + j * grid: tile u / blocks,
// token block u % blocks).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2008_13006_b200/csrc -o membench10 membench10.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "tw_ptx.cuh"

using namespace tw;

constexpr int kA = 32768, kB = 16384;

struct Geo {
  int K, M, pitch, keep, tiles, units_per_cta;
};

template <int kDepth>
__global__ void __launch_bounds__(128, 1) gather(const __nv_bfloat16 *at, const uint8_t *wimg, const int *kept, Geo g,
                                                 long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = sm, *sB = sm + kDepth * kA;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + kDepth * kB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDepth; ++s) ptx::mbar_init(&full[s], 129u);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const uint64_t keep = ptx::policy_evict_last();
  const int blk = lane >> 3, cc = lane & 7;
  const int blocks = g.M / 256, spu = g.keep / 64;
  long long t0 = clock64();
  int i = 0;
  for (int j = 0; j < g.units_per_cta; ++j) {
    const int u = (blockIdx.x + j * gridDim.x) % (g.tiles * blocks);
    const int tile = u / blocks, tb = u % blocks;
    for (int s0 = 0; s0 < spu; ++s0, ++i) {
      const int stage = i % kDepth;
      if (i >= kDepth) ptx::mbar_wait(&full[stage], (uint32_t)((i / kDepth - 1) & 1));
      if (threadIdx.x == 0) {
        ptx::mbar_arrive_expect_tx(&full[stage], kB);
        ptx::bulk_g2s(sB + stage * kB, wimg + ((int64_t)(tile * spu + s0) * kB) % (4 << 20), kB, &full[stage], keep);
      }
#pragma unroll
      for (int it = 0; it < 16; ++it) {
        const int r = warp * 16 + it;
        const int krow = kept[tile * g.keep + s0 * 64 + r];
        const void *src = at + (int64_t)krow * g.pitch + tb * 256 + lane * 8;
        ptx::cp_async_16_full(sA + stage * kA + blk * 8192 + r * 128 + ((cc ^ (r & 7)) * 16), src);
      }
      ptx::cp_async_mbar_arrive_noinc(&full[stage]);
    }
  }
  for (int j = i - kDepth; j < i; ++j)
    if (j >= 0) ptx::mbar_wait(&full[j % kDepth], (uint32_t)((j / kDepth) & 1));
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

template <int kDepth>
void run(const char *name, Geo g, long long *cyc, int sms) {
  __nv_bfloat16 *at;
  uint8_t *wimg;
  int *kept;
  cudaMalloc(&at, (size_t)g.K * g.pitch * 2);
  cudaMemset(at, 0, (size_t)g.K * g.pitch * 2);
  cudaMalloc(&wimg, 4 << 20);
  cudaMemset(wimg, 0, 4 << 20);
  std::vector<int> hk((size_t)g.tiles * g.keep);
  std::mt19937 rng(42);
  for (int t = 0; t < g.tiles; ++t) {
    std::vector<int> p(g.K);
    for (int i = 0; i < g.K; ++i) p[i] = i;
    std::shuffle(p.begin(), p.end(), rng);
    std::sort(p.begin(), p.begin() + g.keep);
    std::copy(p.begin(), p.begin() + g.keep, hk.begin() + (size_t)t * g.keep);
  }
  cudaMalloc(&kept, hk.size() * 4);
  cudaMemcpy(kept, hk.data(), hk.size() * 4, cudaMemcpyHostToDevice);
  const int smem = kDepth * (kA + kB) + 1024 + 256;
  cudaFuncSetAttribute(gather<kDepth>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0.f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    gather<kDepth><<<sms, 128, smem>>>(at, wimg, kept, g, cyc);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    cudaEventElapsedTime(&ms, e0, e1);
  }
  long long h[256];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0, mx = 0;
  for (int i = 0; i < sms; ++i) { avg += h[i]; mx = std::max(mx, (double)h[i]); }
  avg /= sms;
  const double bytes = (double)g.units_per_cta * (g.keep / 64) * (kA + kB);
  printf("depth %d %-40s A+W %6.1f B/clk/SM avg, slowest CTA %6.1f, launch %7.2f us (%s)\n", kDepth, name, bytes / avg,
         bytes / mx, ms * 1e3, cudaGetErrorString(cudaGetLastError()));
  cudaFree(at);
  cudaFree(wimg);
  cudaFree(kept);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long *cyc;
  cudaMalloc(&cyc, 256 * 8);
  run<3>("C2a 768x4096, 12 tiles, 2 units/CTA", Geo{768, 4096, 4096, 384, 12, 2}, cyc, sms);
  run<3>("C5 1024x16384, 16 tiles, 7 units/CTA", Geo{1024, 16384, 16384, 512, 16, 7}, cyc, sms);
  run<3>("C5 dense 1024x16384, 32 tiles, 14 units/CTA", Geo{1024, 16384, 16384, 1024, 32, 14}, cyc, sms);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
