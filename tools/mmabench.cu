// tcgen05.mma issue-rate microbenchmark (B200): cycles per 128xNx16 bf16 MMA
// with both operands in shared memory, A MN-major vs K-major (SW128), to
// calibrate the TW kernel's MMA pacing.  One CTA per SM, one elected thread
// issues `iters` MMAs into TMEM, then commits and waits.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mmabench mmabench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N, bool A_MN>
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, long long *cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tmem_holder;
  __shared__ __align__(8) uint64_t bar;
  uint8_t *base = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) base[i] = 0;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_holder;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(base), b = smem_u32(base + 32768);
    // idesc: f32 acc, bf16 A/B, A major per template, B K-major, M=128, N
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((A_MN ? 1u : 0u) << 15) | ((uint32_t)(N >> 3) << 17) |
                           ((128u >> 4) << 24);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int kk = i & 3;
      const uint64_t ad = A_MN ? desc(a + kk * 2048, 8192, 1024) : desc(a + kk * 32, 16, 1024);
      const uint64_t bd = desc(b + kk * 32, 16, 1024);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(i > 0 ? 1 : 0));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    uint32_t ok = 0;
    while (!ok) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.b32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(smem_u32(&bar)));
    }
    long long t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
  }
}

template <int N, bool A_MN>
void run(const char *name, long long *d, int sms) {
  const int iters = 4096;
  cudaFuncSetAttribute(mma_rate<N, A_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  mma_rate<N, A_MN><<<sms, 128, 70000>>>(iters, d);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < sms; ++i) s += h[i];
  s /= sms;
  const double flops = 2.0 * 128 * N * 16;
  printf("%-22s %7.1f cyc/MMA  (ideal %d)  %6.0f flop/clk/SM\n", name, s / iters, 128 * N / 256, flops * iters / s);
}

int main() {
  long long *d;
  cudaMalloc(&d, 256 * 8);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<128, true>("M128 N128 A=MN-major", d, sms);
  run<128, false>("M128 N128 A=K-major", d, sms);
  run<256, true>("M128 N256 A=MN-major", d, sms);
  run<256, false>("M128 N256 A=K-major", d, sms);
  run<64, true>("M128 N64 A=MN-major", d, sms);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
