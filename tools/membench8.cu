// Does the TW kernel's gather ORDER matter?  148 CTAs gather 64-row stages
// of 512 B A^T row segments (cp.async 16 B, 4 warps, 4 stages in flight) from
// a 768 x 4096 bf16 A^T (L2-resident), in three orders:
//   0 random rows, every CTA its own token segment (membench6's pattern)
//   1 kernel-like: CTA b works on token block b % 16 and "tile" b / 16, whose
//     kept rows are a sorted random half of K; ~10 CTAs read the same token
//     block in ascending row order at the same time
//   2 as 1, but each tile starts at a different 64-row block (rotated order)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench8 membench8.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

__device__ __forceinline__ void cp16(void *s, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}

constexpr int kDepth = 4;

__global__ void gather(const __nv_bfloat16 *at, const int *kept /*12 x 384*/, int mode, int reps, long long *cyc) {
  extern __shared__ __align__(1024) char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= 4) return;
  const int tb = blockIdx.x % 16, tile = (blockIdx.x / 16) % 12;
  const int nst = 6;  // 384 kept rows = 6 stages
  long long t0 = clock64();
  int i = 0;
  for (int rep = 0; rep < reps; ++rep) {
    for (int s0 = 0; s0 < nst; ++s0, ++i) {
      const int s = mode == 2 ? (s0 + tile) % nst : s0;
      for (int it = 0; it < 16; ++it) {
        const int r = warp * 16 + it;
        int krow, col;
        if (mode == 0) {
          krow = (r * 389 + i * 13 + blockIdx.x * 7) % 768;
          col = (blockIdx.x * 256 + i * 256) % 4096;
        } else {
          krow = kept[tile * 384 + s * 64 + r];
          col = ((tb + rep) % 16) * 256;
        }
        cp16(sm + (i % kDepth) * 32768 + r * 512 + lane * 16, at + (int64_t)krow * 4096 + col + lane * 8);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(kDepth - 1) : "memory");
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  __nv_bfloat16 *at;
  int *kept;
  long long *cyc;
  cudaMalloc(&at, 768 * 4096 * 2);
  cudaMemset(at, 0, 768 * 4096 * 2);
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
  cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, kDepth * 32768);
  const char *names[3] = {"random rows, own token segment", "kernel-like (same token block, ascending)",
                          "kernel-like, rotated start block per tile"};
  for (int reps : {2, 8}) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int r = 0; r < 2; ++r) {
        gather<<<sms, 128, kDepth * 32768>>>(at, kept, mode, reps, cyc);
        cudaDeviceSynchronize();
      }
      long long h[256];
      cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
      double avg = 0, mx = 0;
      for (int i = 0; i < sms; ++i) { avg += h[i]; mx = std::max(mx, (double)h[i]); }
      avg /= sms;
      const double bytes = 6.0 * reps * 32768;
      printf("reps %d mode %d %-44s %6.1f B/clk/SM avg (slowest CTA %6.1f)\n", reps, mode, names[mode], bytes / avg,
             bytes / mx);
    }
  }
  // cold: A^T evicted from L2 before each launch (write 256 MB elsewhere)
  char *junk;
  cudaMalloc(&junk, 256 << 20);
  for (int mode = 0; mode < 3; ++mode) {
    cudaMemset(junk, mode, 256 << 20);
    gather<<<sms, 128, kDepth * 32768>>>(at, kept, mode, 2, cyc);
    cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    printf("cold mode %d: %6.1f B/clk/SM\n", mode, 6.0 * 2 * 32768 / avg);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
