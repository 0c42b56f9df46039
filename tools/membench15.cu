// Round 2 (late): per-SM cp.async gather throughput by row-piece width and pipeline depth.
// K2's producer (4 warps, SW128 MN-major destinations, 16 KB TMA weight block per stage, one
// consumer warp that releases a slot as soon as it is full -- no MMA) for 64-row stages of
// TOK tokens: TOK = 256 (512-byte row pieces, K2's wide stage) vs 128 (256-byte pieces, the
// half-width stage a CTA-pair "union" kernel would gather), at several depths.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_2008_13006_b200/csrc -o bin/membench15 membench15.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "tw_ptx.cuh"

using namespace tw;

constexpr int kB = 16384;

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <int TOK, int DEPTH>
__global__ void __launch_bounds__(448, 1)
    gather(const uint16_t *at, const uint8_t *wimg, const int *kept, int K, int M, int keep, int tiles, int upc,
           unsigned long long *ns) {
  constexpr int kA = 64 * TOK * 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = sm, *sB = sm + DEPTH * kA;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + DEPTH * kB);
  uint64_t *empty = full + DEPTH;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < DEPTH; ++s) {
      ptx::mbar_init(&full[s], 1u + 4 * 32u);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const unsigned long long t0 = gtime();
  const uint64_t pol = ptx::policy_evict_last();
  const int blocks = M / TOK, spu = keep / 64, total = upc * spu;
  constexpr int L = TOK / 8;        // 16-byte chunks (lanes) per row piece
  constexpr int R = 32 / L;         // rows per instruction
  if (warp < 4) {
    const int ch = lane % L, rs = lane / L, cq = ch & 7;
    for (int i = 0; i < total; ++i) {
      const int j = i / spu, s0 = i % spu;
      const int u = (blockIdx.x + j * gridDim.x) % (tiles * blocks);
      const int tile = u / blocks, tb = u % blocks;
      const int stage = i % DEPTH;
      if (i >= DEPTH) ptx::mbar_wait(&empty[stage], (uint32_t)((i / DEPTH - 1) & 1));
      const int *krows = kept + tile * keep + s0 * 64;
      if (threadIdx.x == 0) {
        ptx::mbar_arrive_expect_tx(&full[stage], kB);
        ptx::bulk_g2s(sB + stage * kB, wimg + ((int64_t)(tile * spu + s0) * kB) % (4 << 20), kB, &full[stage], pol);
      }
      uint8_t *aw = sA + stage * kA + (ch >> 3) * 8192 + warp * 16 * 128;
#pragma unroll
      for (int it = 0; it < 16 / R; ++it) {
        const int rl = it * R + rs;
        const int row = __ldg(krows + warp * 16 + rl);
        ptx::cp_async_16_full(aw + rl * 128 + ((cq ^ (rl & 7)) * 16), at + (int64_t)row * M + tb * TOK + ch * 8);
      }
      ptx::cp_async_mbar_arrive_noinc(&full[stage]);
    }
    ptx::cp_async_wait_group<0>();
  } else if (warp == 4) {
    for (int i = 0; i < total; ++i) {
      const int stage = i % DEPTH;
      ptx::mbar_wait(&full[stage], (uint32_t)((i / DEPTH) & 1));
      if (lane == 0) ptx::mbar_arrive(&empty[stage]);
      __syncwarp();
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ns[2 * blockIdx.x] = t0;
    ns[2 * blockIdx.x + 1] = gtime();
  }
}

template <int TOK, int DEPTH>
void run(const uint16_t *at, const uint8_t *wimg, const int *kept, int K, int M, int keep, int tiles,
         unsigned long long *ns, float *soakbuf) {
  constexpr int kA = 64 * TOK * 2;
  const int smem = DEPTH * (kA + kB) + 1024 + 256;
  auto k = gather<TOK, DEPTH>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int sms = 148;
  // same gathered bytes for every config: units of TOK tokens, upc units per CTA
  const int upc = 8 * 256 / TOK;
  for (int rep = 0; rep < 3; ++rep) k<<<sms, 448, smem>>>(at, wimg, kept, K, M, keep, tiles, upc, ns);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  const int reps = 20;
  for (int rep = 0; rep < reps; ++rep) k<<<sms, 448, smem>>>(at, wimg, kept, K, M, keep, tiles, upc, ns);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = (double)sms * upc * (keep / 64) * 64.0 * TOK * 2;
  const double s = ms * 1e-3 / reps;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("TOK %3d depth %d smem %6d: A gathered %.2f TB/s chip, %.1f B/clk/SM at the nominal clock, %.2f us/launch\n",
         TOK, DEPTH, smem, bytes / s / 1e12, bytes / s / sms / (clk * 1e3), s * 1e6);
}

int main() {
  const int K = 1024, M = 16384, keep = 512, tiles = 16;
  uint16_t *at;
  uint8_t *wimg;
  int *kept;
  unsigned long long *ns;
  float *soakbuf;
  cudaMalloc(&at, (size_t)K * M * 2);
  cudaMemset(at, 0, (size_t)K * M * 2);
  cudaMalloc(&wimg, 4 << 20);
  cudaMemset(wimg, 0, 4 << 20);
  cudaMalloc(&ns, 4096 * 16);
  cudaMalloc(&soakbuf, 4096);
  std::vector<int> hk((size_t)tiles * keep);
  std::mt19937 rng(42);
  for (int t = 0; t < tiles; ++t) {
    std::vector<int> p(K);
    for (int i = 0; i < K; ++i) p[i] = i;
    std::shuffle(p.begin(), p.end(), rng);
    std::sort(p.begin(), p.begin() + keep);
    std::copy(p.begin(), p.begin() + keep, hk.begin() + (size_t)t * keep);
  }
  cudaMalloc(&kept, hk.size() * 4);
  cudaMemcpy(kept, hk.data(), hk.size() * 4, cudaMemcpyHostToDevice);
  run<256, 2>(at, wimg, kept, K, M, keep, tiles, ns, soakbuf);
  run<256, 3>(at, wimg, kept, K, M, keep, tiles, ns, soakbuf);
  run<256, 4>(at, wimg, kept, K, M, keep, tiles, ns, soakbuf);
  run<128, 3>(at, wimg, kept, K, M, keep, tiles, ns, soakbuf);
  run<128, 4>(at, wimg, kept, K, M, keep, tiles, ns, soakbuf);
  run<128, 6>(at, wimg, kept, K, M, keep, tiles, ns, soakbuf);
  run<128, 7>(at, wimg, kept, K, M, keep, tiles, ns, soakbuf);
  run<256, 2>(at, wimg, kept, K, M, keep, tiles, ns, soakbuf);
  run<256, 3>(at, wimg, kept, K, M, keep, tiles, ns, soakbuf);
  run<128, 6>(at, wimg, kept, K, M, keep, tiles, ns, soakbuf);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
