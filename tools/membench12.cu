// Round 2: L2 vs HBM bandwidth on B200 in absolute units (TB/s), clocks
// soaked first, the SM clock measured inside the kernels (clock64 over
// globaltimer).  Decides whether K2's L2->SM operand traffic (gathers +
// weight blocks + output stores) or its HBM bytes bound the kernel.
//   read  : 148*k CTAs stream a buffer (L2-resident sizes and 1 GB) with
//           (a) 16 B ld.global.cg, (b) 16 B cp.async into an smem ring,
//           (c) 1-D TMA bulk copies of 16 KB into an smem ring
//   write : 16 B st.global.cs and 1-D TMA bulk stores from smem
//   gather: the K2 producer pattern (64 kept rows x 256 tokens per stage)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2008_13006_b200/csrc -o bin/membench12 membench12.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "tw_ptx.cuh"

using namespace tw;

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

struct Stamp {
  long long c0, c1;
  unsigned long long g0, g1;
};

__device__ __forceinline__ void stamp_begin(Stamp *s) {
  if (threadIdx.x == 0) {
    s[blockIdx.x].c0 = clock64();
    s[blockIdx.x].g0 = gtime();
  }
}
__device__ __forceinline__ void stamp_end(Stamp *s) {
  __syncthreads();
  if (threadIdx.x == 0) {
    s[blockIdx.x].c1 = clock64();
    s[blockIdx.x].g1 = gtime();
  }
}

__global__ void soak(float *x, int iters) {
  float v = threadIdx.x;
  for (int i = 0; i < iters; ++i) v = v * 1.0000001f + 0.5f;
  if (v == 12345.f) x[0] = v;
}

// (a) ld.global.cg 16 B, each CTA streams its slice `passes` times
__global__ void __launch_bounds__(512) rd_ldg(const uint4 *buf, int64_t n16, int passes, uint4 *sink, Stamp *st) {
  stamp_begin(st);
  const int64_t per = n16 / gridDim.x;
  const uint4 *p = buf + per * blockIdx.x;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (int ps = 0; ps < passes; ++ps)
    for (int64_t i = threadIdx.x; i < per; i += blockDim.x * 4) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = i + u * blockDim.x;
        v[u] = j < per ? __ldcg(p + j) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
    }
  if (acc.x == 0x12345678u) sink[0] = acc;
  stamp_end(st);
}

// (b) cp.async 16 B into an smem ring of 8 x 16 KB, 8-deep groups
__global__ void __launch_bounds__(256) rd_cpasync(const uint4 *buf, int64_t n16, int passes, uint4 *sink, Stamp *st) {
  extern __shared__ __align__(1024) uint8_t sm[];
  stamp_begin(st);
  const int64_t per = n16 / gridDim.x;
  const uint4 *p = buf + per * blockIdx.x;
  int slot = 0;
  for (int ps = 0; ps < passes; ++ps)
    for (int64_t i = 0; i < per; i += 1024) {  // 16 KB per group
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t j = i + u * 256 + threadIdx.x;
        if (j < per) ptx::cp_async_16_full(sm + slot * 16384 + (u * 256 + threadIdx.x) * 16, p + j);
      }
      ptx::cp_async_commit();
      ptx::cp_async_wait_group<7>();
      slot = (slot + 1) & 7;
    }
  ptx::cp_async_wait_group<0>();
  stamp_end(st);
}

// (c) TMA 1-D bulk copies, 16 KB each, 8 in flight, one issuing thread
__global__ void __launch_bounds__(128) rd_bulk(const uint8_t *buf, int64_t bytes, int passes, uint4 *sink, Stamp *st) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + 8 * 16384);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 8; ++s) ptx::mbar_init(&bar[s], 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  stamp_begin(st);
  const int64_t per = bytes / gridDim.x / 16384 * 16384;
  const uint8_t *p = buf + per * blockIdx.x;
  if (threadIdx.x == 0) {
    const uint64_t pol = ptx::policy_evict_last();
    int64_t i = 0;
    for (int ps = 0; ps < passes; ++ps)
      for (int64_t off = 0; off < per; off += 16384, ++i) {
        const int s = (int)(i & 7);
        if (i >= 8) ptx::mbar_wait(&bar[s], (uint32_t)(((i >> 3) - 1) & 1));
        ptx::mbar_arrive_expect_tx(&bar[s], 16384);
        ptx::bulk_g2s(sm + s * 16384, p + off, 16384, &bar[s], pol);
      }
    for (int64_t j = (i > 8 ? i - 8 : (int64_t)0); j < i; ++j) ptx::mbar_wait(&bar[j & 7], (uint32_t)((j >> 3) & 1));
  }
  stamp_end(st);
}

__global__ void __launch_bounds__(512) wr_stg(uint4 *buf, int64_t n16, int passes, Stamp *st) {
  stamp_begin(st);
  const int64_t per = n16 / gridDim.x;
  uint4 *p = buf + per * blockIdx.x;
  for (int ps = 0; ps < passes; ++ps)
    for (int64_t i = threadIdx.x; i < per; i += blockDim.x) __stcs(p + i, make_uint4(ps, 0, 0, 0));
  stamp_end(st);
}

__global__ void __launch_bounds__(128) wr_bulk(uint8_t *buf, int64_t bytes, int passes, Stamp *st) {
  extern __shared__ __align__(1024) uint8_t sm[];
  for (int i = threadIdx.x; i < 8192 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  __syncthreads();
  stamp_begin(st);
  const int64_t per = bytes / gridDim.x / 8192 * 8192;
  uint8_t *p = buf + per * blockIdx.x;
  if (threadIdx.x == 0) {
    for (int ps = 0; ps < passes; ++ps)
      for (int64_t off = 0; off < per; off += 8192) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off), "r"(ptx::smem_u32(sm)),
                     "r"(8192)
                     : "memory");
        ptx::bulk_commit();
        ptx::bulk_wait_read<6>();
      }
    ptx::bulk_wait<0>();
  }
  stamp_end(st);
}

// K2 producer pattern: 4 warps, 64 kept rows x 256 tokens per stage (32 KB),
// kDepth stages in flight (no weights / consumer: pure gather), units in
// kernel order over a C2a-like A^T (K x M bf16).
template <int kDepth>
__global__ void __launch_bounds__(128, 1) gather(const uint16_t *at, const int *kept, int K, int M, int keep, int tiles,
                                                 int units_per_cta, Stamp *st) {
  extern __shared__ __align__(1024) uint8_t sm[];
  stamp_begin(st);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int blocks = M / 256, spu = keep / 64;
  int i = 0;
  for (int j = 0; j < units_per_cta; ++j) {
    const int u = (blockIdx.x + j * gridDim.x) % (tiles * blocks);
    const int tile = u / blocks, tb = u % blocks;
    for (int s0 = 0; s0 < spu; ++s0, ++i) {
#pragma unroll
      for (int it = 0; it < 16; ++it) {
        const int r = warp * 16 + it;
        const void *src = at + (int64_t)kept[tile * keep + s0 * 64 + r] * M + tb * 256 + lane * 8;
        ptx::cp_async_16_full(sm + (i % kDepth) * 32768 + r * 512 + lane * 16, src);
      }
      ptx::cp_async_commit();
      ptx::cp_async_wait_group<kDepth - 1>();
    }
  }
  ptx::cp_async_wait_group<0>();
  stamp_end(st);
}

struct Res {
  double us, mhz, active_frac;
};

template <typename F>
Res timed(F launch, Stamp *d_st, int grid) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f, ms;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  std::vector<Stamp> h(grid);
  cudaMemcpy(h.data(), d_st, grid * sizeof(Stamp), cudaMemcpyDeviceToHost);
  double cyc = 0, ns = 0;
  unsigned long long gmin = ~0ull, gmax = 0;
  for (auto &s : h) {
    cyc += (double)(s.c1 - s.c0);
    ns += (double)(s.g1 - s.g0);
    gmin = std::min(gmin, s.g0);
    gmax = std::max(gmax, s.g1);
  }
  return Res{best * 1e3, ns > 0 ? cyc / ns * 1e3 : 0, (double)(gmax - gmin) / 1e3 / (best * 1e3)};
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  Stamp *st;
  cudaMalloc(&st, 4096 * sizeof(Stamp));
  uint4 *sink;
  cudaMalloc(&sink, 64);
  float *x;
  cudaMalloc(&x, 64);
  const size_t big = (size_t)1 << 30;
  uint8_t *buf;
  cudaMalloc(&buf, big);
  cudaMemset(buf, 1, big);
  // clock soak ~0.4 s
  for (int i = 0; i < 20; ++i) soak<<<sms * 4, 256>>>(x, 200000);
  cudaDeviceSynchronize();
  cudaFuncSetAttribute(rd_cpasync, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384);
  cudaFuncSetAttribute(rd_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 16384 + 1024);
  cudaFuncSetAttribute(wr_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
  const size_t sizes[] = {(size_t)8 << 20, (size_t)32 << 20, (size_t)64 << 20, big};
  for (size_t sz : sizes) {
    const int passes = sz >= big ? 1 : (int)std::max<size_t>(1, ((size_t)1 << 30) / sz);
    const double bytes = (double)sz * passes;
    const int64_t n16 = (int64_t)(sz / 16);
    for (int cpsm : {1, 2}) {
      const int grid = sms * cpsm;
      Res r = timed([&] { rd_ldg<<<grid, 512>>>((const uint4 *)buf, n16, passes, sink, st); }, st, grid);
      printf("read  ldg.cg    %5zu MB x%3d grid %3d: %7.2f TB/s  (%.0f us, SM %.0f MHz, span %.2f)\n", sz >> 20, passes, grid,
             bytes / r.us / 1e6, r.us, r.mhz, r.active_frac);
    }
    {
      const int grid = sms;
      Res r = timed([&] { rd_cpasync<<<grid, 256, 8 * 16384>>>((const uint4 *)buf, n16, passes, sink, st); }, st, grid);
      printf("read  cp.async  %5zu MB x%3d grid %3d: %7.2f TB/s  (%.0f us, SM %.0f MHz, span %.2f)\n", sz >> 20, passes, grid,
             bytes / r.us / 1e6, r.us, r.mhz, r.active_frac);
    }
    {
      const int grid = sms;
      Res r = timed([&] { rd_bulk<<<grid, 128, 8 * 16384 + 1024>>>(buf, (int64_t)sz, passes, sink, st); }, st, grid);
      printf("read  bulk16K   %5zu MB x%3d grid %3d: %7.2f TB/s  (%.0f us, SM %.0f MHz, span %.2f)\n", sz >> 20, passes, grid,
             bytes / r.us / 1e6, r.us, r.mhz, r.active_frac);
    }
    {
      const int grid = sms * 2;
      Res r = timed([&] { wr_stg<<<grid, 512>>>((uint4 *)buf, n16, passes, st); }, st, grid);
      printf("write stg.cs    %5zu MB x%3d grid %3d: %7.2f TB/s  (%.0f us, SM %.0f MHz, span %.2f)\n", sz >> 20, passes, grid,
             bytes / r.us / 1e6, r.us, r.mhz, r.active_frac);
    }
    {
      const int grid = sms;
      Res r = timed([&] { wr_bulk<<<grid, 128, 8192>>>(buf, (int64_t)sz, passes, st); }, st, grid);
      printf("write bulk8K    %5zu MB x%3d grid %3d: %7.2f TB/s  (%.0f us, SM %.0f MHz, span %.2f)\n", sz >> 20, passes, grid,
             bytes / r.us / 1e6, r.us, r.mhz, r.active_frac);
    }
  }
  // K2 gather pattern, C2a and C5 geometry, L2-warm A^T (re-launched), depth 4 and 6
  struct G { const char *name; int K, M, keep, tiles, upc; };
  for (G g : {G{"C2a", 768, 4096, 384, 12, 8}, G{"C5@75", 1024, 16384, 512, 16, 8}}) {
    std::vector<int> hk((size_t)g.tiles * g.keep);
    std::mt19937 rng(42);
    for (int t = 0; t < g.tiles; ++t) {
      std::vector<int> p(g.K);
      for (int i = 0; i < g.K; ++i) p[i] = i;
      std::shuffle(p.begin(), p.end(), rng);
      std::sort(p.begin(), p.begin() + g.keep);
      std::copy(p.begin(), p.begin() + g.keep, hk.begin() + (size_t)t * g.keep);
    }
    int *kept;
    cudaMalloc(&kept, hk.size() * 4);
    cudaMemcpy(kept, hk.data(), hk.size() * 4, cudaMemcpyHostToDevice);
    const double bytes = (double)sms * g.upc * g.keep * 256 * 2;
    cudaFuncSetAttribute(gather<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
    cudaFuncSetAttribute(gather<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768);
    Res r4 = timed([&] { gather<4><<<sms, 128, 4 * 32768>>>((const uint16_t *)buf, kept, g.K, g.M, g.keep, g.tiles, g.upc, st); }, st, sms);
    Res r6 = timed([&] { gather<6><<<sms, 128, 6 * 32768>>>((const uint16_t *)buf, kept, g.K, g.M, g.keep, g.tiles, g.upc, st); }, st, sms);
    printf("gather %-6s %d units/CTA: depth 4 %7.2f TB/s (%.1f us, SM %.0f MHz) | depth 6 %7.2f TB/s (%.1f us)\n", g.name, g.upc,
           bytes / r4.us / 1e6, r4.us, r4.mhz, bytes / r6.us / 1e6, r6.us);
    cudaFree(kept);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
