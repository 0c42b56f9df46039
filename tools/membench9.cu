// Which feature of the TW kernel's producer costs gather throughput?
// 148 CTAs x 4 producer warps gather kernel-like 64-row stages (sorted kept
// rows of a 768 x 4096 bf16 A^T, 512 B per row, 4 stages in flight), adding
// one kernel feature at a time:
//   W    a 16 KB TMA bulk weight load per stage (like the B operand)
//   SW   SW128 destination addressing (4 blocks of 128 B rows, XOR swizzle)
//   MB   completion through cp.async.mbarrier.arrive.noinc + mbarrier waits
//        instead of cp.async.wait_group
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2008_13006_b200/csrc -o membench9 membench9.cu
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

constexpr int kDepth = 4;
constexpr int kA = 32768, kB = 16384;

template <bool W, bool SW, bool MB, bool CONS = false, bool RING = false>
__global__ void __launch_bounds__(416, 1) gather(const __nv_bfloat16 *at, const uint8_t *wimg, const int *kept, int reps,
                                                 long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = sm, *sB = sm + kDepth * kA;
  uint64_t *full = reinterpret_cast<uint64_t *>(sB + kDepth * kB);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t *done = full + kDepth;
  uint64_t *empty = done + 1;
  int32_t *ring = reinterpret_cast<int32_t *>(full + 16);  // 4 warps x 8 slots x 16 ints
  if (threadIdx.x == 0) {
    ptx::mbar_init(done, 1);
    for (int s = 0; s < kDepth; ++s) ptx::mbar_init(&empty[s], 1);
    for (int s = 0; s < kDepth; ++s) ptx::mbar_init(&full[s], (MB ? 128u : 0u) + (W ? 1u : 0u) + (!MB && !W ? 1u : 0u));
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int tb = blockIdx.x % 16, tile = (blockIdx.x / 16) % 12;
  if (CONS && warp == 4) {  // consumer: full -> (fence, commit) -> empty, like the MMA warp
    for (int j = 0; j < reps * 6; ++j) {
      ptx::mbar_wait(&full[j % kDepth], (uint32_t)((j / kDepth) & 1));
      ptx::fence_proxy_async_smem();
      ptx::tc_fence_after();
      if (ptx::elect_one()) ptx::mma_commit(&empty[j % kDepth]);
      __syncwarp();
    }
    return;
  }
  if (warp >= 4) {  // the kernel's epilogue warps, parked on an mbarrier
    ptx::mbar_wait(done, 0);
    return;
  }
  int32_t *wring = ring + warp * 8 * 16;
  auto prefetch = [&](int j) {  // stage j's 16 row indices of this warp into its ring
    if (lane < 4) ptx::cp_async_16(wring + (j % 8) * 16 + lane * 4, kept + tile * 384 + (j % 6) * 64 + warp * 16 + lane * 4, 16);
  };
  if (RING) {
    for (int j = 0; j < 4; ++j) { prefetch(j); ptx::cp_async_commit(); }
  }
  const uint64_t keep = ptx::policy_evict_last();
  const int blk = lane >> 3, cc = lane & 7;
  long long t0 = clock64();
  int i = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int s0 = 0; s0 < 6; ++s0, ++i) {
      const int stage = i % kDepth;
      if (CONS) {
        if (i >= kDepth) ptx::mbar_wait(&empty[stage], (uint32_t)((i / kDepth - 1) & 1));
      } else if ((MB || W) && i >= kDepth) {
        ptx::mbar_wait(&full[stage], (uint32_t)((i / kDepth - 1) & 1));
      }
      int rows[16];
      if (RING) {
        ptx::cp_async_wait_group<3>();
        __syncwarp();
#pragma unroll
        for (int v4 = 0; v4 < 4; ++v4) {
          const int4 r4 = reinterpret_cast<const int4 *>(wring + (i % 8) * 16)[v4];
          rows[4 * v4] = r4.x; rows[4 * v4 + 1] = r4.y; rows[4 * v4 + 2] = r4.z; rows[4 * v4 + 3] = r4.w;
        }
      }
      if (W && threadIdx.x == 0) {
        ptx::mbar_arrive_expect_tx(&full[stage], kB);
        ptx::bulk_g2s(sB + stage * kB, wimg + ((int64_t)i * kB) % (2 << 20), kB, &full[stage], keep);
      }
      const int col = ((tb + rep) % 16) * 256;
#pragma unroll
      for (int it = 0; it < 16; ++it) {
        const int r = warp * 16 + it;
        const int krow = RING ? rows[it] : kept[tile * 384 + s0 * 64 + r];
        const void *src = at + (int64_t)krow * 4096 + col + lane * 8;
        uint8_t *dst = SW ? sA + stage * kA + blk * 8192 + r * 128 + ((cc ^ (r & 7)) * 16)
                          : sA + stage * kA + r * 512 + lane * 16;
        ptx::cp_async_16_full(dst, src);
      }
      if (RING) {
        prefetch(i + 4);
        ptx::cp_async_mbar_arrive_noinc(&full[stage]);
        ptx::cp_async_commit();
      } else if (MB) {
        ptx::cp_async_mbar_arrive_noinc(&full[stage]);
      } else {
        ptx::cp_async_commit();
        ptx::cp_async_wait_group<kDepth - 1>();
        if (!W && threadIdx.x == 0) ptx::mbar_arrive(&full[stage]);
      }
    }
  }
  if (CONS) {
    for (int j = i - kDepth; j < i; ++j)
      if (j >= 0) ptx::mbar_wait(&empty[j % kDepth], (uint32_t)((j / kDepth) & 1));
  } else if (MB || W) {
    for (int j = i - kDepth; j < i; ++j)
      if (j >= 0) ptx::mbar_wait(&full[j % kDepth], (uint32_t)((j / kDepth) & 1));
  }
  ptx::cp_async_wait_group<0>();
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = clock64() - t0;
    ptx::mbar_arrive(done);
  }
}

template <bool W, bool SW, bool MB, bool CONS = false, bool RING = false>
void run(const char *name, const __nv_bfloat16 *at, const uint8_t *wimg, const int *kept, long long *cyc, int sms,
         int threads = 128, int extra_smem = 0) {
  auto k = gather<W, SW, MB, CONS, RING>;
  const int smem = kDepth * (kA + kB) + 1024 + 4096 + extra_smem;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int reps = 8;
  for (int r = 0; r < 2; ++r) {
    k<<<sms, threads, smem>>>(at, wimg, kept, reps, cyc);
    cudaDeviceSynchronize();
  }
  long long h[256];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double a_bytes = 6.0 * reps * kA, w_bytes = W ? 6.0 * reps * kB : 0.0;
  printf("%-28s A %6.1f B/clk/SM   A+W %6.1f B/clk/SM  (%s)\n", name, a_bytes / avg, (a_bytes + w_bytes) / avg,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  __nv_bfloat16 *at;
  uint8_t *wimg;
  int *kept;
  long long *cyc;
  cudaMalloc(&at, 768 * 4096 * 2);
  cudaMemset(at, 0, 768 * 4096 * 2);
  cudaMalloc(&wimg, 2 << 20);
  cudaMemset(wimg, 0, 2 << 20);
  std::vector<int> hk(12 * 384);
  std::mt19937 rng(42);
  for (int t = 0; t < 12; ++t) {
    std::vector<int> p(768);
    for (int i = 0; i < 768; ++i) p[i] = i;
    std::shuffle(p.begin(), p.end(), rng);
    std::sort(p.begin(), p.begin() + 384);
    std::copy(p.begin(), p.begin() + 384, hk.begin() + t * 384);
  }
  cudaMalloc(&kept, hk.size() * 4);
  cudaMemcpy(kept, hk.data(), hk.size() * 4, cudaMemcpyHostToDevice);
  cudaMalloc(&cyc, 256 * 8);
  run<false, false, false>("plain (membench8 mode 1)", at, wimg, kept, cyc, sms);
  run<false, true, false>("+SW128 dst", at, wimg, kept, cyc, sms);
  run<false, false, true>("+mbarrier completion", at, wimg, kept, cyc, sms);
  run<true, false, false>("+W bulk", at, wimg, kept, cyc, sms);
  run<true, true, true>("all (kernel producer)", at, wimg, kept, cyc, sms);
  run<true, true, false>("W + SW (wait_group)", at, wimg, kept, cyc, sms);
  run<true, true, true>("all + 227 KB smem", at, wimg, kept, cyc, sms, 128, 232448 - (kDepth * (kA + kB) + 1024 + 4096));
  run<true, true, true>("all + 9 parked warps", at, wimg, kept, cyc, sms, 416, 0);
  run<true, true, true>("all + both", at, wimg, kept, cyc, sms, 416, 232448 - (kDepth * (kA + kB) + 1024 + 4096));
  run<true, true, true, true, false>("all + consumer warp", at, wimg, kept, cyc, sms, 416, 0);
  run<true, true, true, false, true>("all + index ring", at, wimg, kept, cyc, sms, 416, 0);
  run<true, true, true, true, true>("all + consumer + ring", at, wimg, kept, cyc, sms, 416, 0);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
