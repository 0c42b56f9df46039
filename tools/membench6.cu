// cp.async gather throughput vs bytes in flight per SM (B200), with and
// without a concurrent DRAM-bound store stream on the same SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench6 membench6.cu
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void cp16(void *s, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(s)), "l"(g)
               : "memory");
}

// 4 gather warps: stage = 64 rows x 512 B (32 KB); keep `depth` stages in flight
template <int kDepth, bool kStores>
__global__ void gather(const __nv_bfloat16 *at, int stages, float4 *out, int64_t out_per_cta, long long *cyc) {
  extern __shared__ __align__(1024) char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 4) {
    long long t0 = clock64();
    for (int i = 0; i < stages; ++i) {
      for (int it = 0; it < 16; ++it) {
        const int r = warp * 16 + it;
        const int krow = (r * 389 + i * 13 + blockIdx.x * 7) % 768;
        cp16(sm + (i % kDepth) * 32768 + r * 512 + lane * 16,
             at + (int64_t)krow * 4096 + ((blockIdx.x * 256 + i * 256) % 4096) + lane * 8);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(kDepth - 1) : "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  } else if (kStores) {
    float4 *o = out + (int64_t)blockIdx.x * out_per_cta;
    for (int64_t i = (warp - 4) * 32 + lane; i < out_per_cta; i += 256) __stcs(o + i, make_float4(0, 0, 0, 0));
  }
}

template <int kDepth>
__global__ void split(const __nv_bfloat16 *at, int stages, float4 *out, int64_t out_per_cta, long long *cyc) {
  extern __shared__ __align__(1024) char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (blockIdx.x % 2 == 0) {
    if (warp >= 4) return;
    long long t0 = clock64();
    for (int i = 0; i < stages; ++i) {
      for (int it = 0; it < 16; ++it) {
        const int r = warp * 16 + it;
        const int krow = (r * 389 + i * 13 + blockIdx.x * 7) % 768;
        cp16(sm + (i % kDepth) * 32768 + r * 512 + lane * 16,
             at + (int64_t)krow * 4096 + ((blockIdx.x * 256 + i * 256) % 4096) + lane * 8);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(kDepth - 1) : "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  } else {
    float4 *o = out + (int64_t)(blockIdx.x / 2) * out_per_cta;
    for (int64_t i = threadIdx.x; i < out_per_cta; i += blockDim.x) __stcs(o + i, make_float4(0, 0, 0, 0));
  }
}

// gathers (cp.async, 4 warps) + TMA bulk zero stores (one thread) on the same SM
template <int kDepth>
__global__ void gather_tma_store(const __nv_bfloat16 *at, int stages, char *out, int64_t out_bytes_per_cta,
                                 long long *cyc) {
  extern __shared__ __align__(1024) char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char *zero = sm + kDepth * 32768;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) zero[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (warp < 4) {
    long long t0 = clock64();
    for (int i = 0; i < stages; ++i) {
      for (int it = 0; it < 16; ++it) {
        const int r = warp * 16 + it;
        const int krow = (r * 389 + i * 13 + blockIdx.x * 7) % 768;
        cp16(sm + (i % kDepth) * 32768 + r * 512 + lane * 16,
             at + (int64_t)krow * 4096 + ((blockIdx.x * 256 + i * 256) % 4096) + lane * 8);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(kDepth - 1) : "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
  } else if (threadIdx.x == 128) {
    char *o = out + (int64_t)blockIdx.x * out_bytes_per_cta;
    for (int64_t off = 0; off < out_bytes_per_cta; off += 16384) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(o + off),
                   "r"((uint32_t)__cvta_generic_to_shared(zero)));
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 8;");
    }
    asm volatile("cp.async.bulk.wait_group 0;");
  }
}

// gather (4 warps) with 9 more warps parked on an mbarrier try_wait loop
// (as the kernel's MMA / epilogue warps are) -- do they slow the gathers?
template <int kDepth>
__global__ void gather_spinners(const __nv_bfloat16 *at, int stages, long long *cyc) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
  }
  __syncthreads();
  if (warp < 4) {
    long long t0 = clock64();
    for (int i = 0; i < stages; ++i) {
      for (int it = 0; it < 16; ++it) {
        const int r = warp * 16 + it;
        const int krow = (r * 389 + i * 13 + blockIdx.x * 7) % 768;
        cp16(sm + (i % kDepth) * 32768 + r * 512 + lane * 16,
             at + (int64_t)krow * 4096 + ((blockIdx.x * 256 + i * 256) % 4096) + lane * 8);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(kDepth - 1) : "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (threadIdx.x == 0) {
      cyc[blockIdx.x] = clock64() - t0;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    }
  } else {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.b32 %0,1,0,p;\n\t}"
                   : "=r"(ok)
                   : "r"((uint32_t)__cvta_generic_to_shared(&bar)));
  }
}

template <int D, bool S>
void run(const __nv_bfloat16 *at, float4 *out, long long *cyc, int sms) {
  auto k = gather<D, S>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, D * 32768);
  const int stages = 64;
  const int64_t opc = 131072;  // 2 MB of stores per CTA (DRAM bound, longer than the gathers)
  k<<<sms, S ? 384 : 128, D * 32768>>>(at, stages, out, opc, cyc);
  cudaDeviceSynchronize();
  k<<<sms, S ? 384 : 128, D * 32768>>>(at, stages, out, opc, cyc);
  cudaDeviceSynchronize();
  long long h[256];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double bytes = 64.0 * 32768;
  printf("depth %d (%3d KB in flight) stores=%d: %6.1f B/clk/SM  (~%5.1f GB/s/SM at 1.9 GHz)\n", D, D * 32, (int)S,
         bytes / avg, bytes / avg * 1.9);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  __nv_bfloat16 *at;
  float4 *out;
  long long *cyc;
  cudaMalloc(&at, 768 * 4096 * 2);
  cudaMemset(at, 0, 768 * 4096 * 2);
  cudaMalloc(&out, (size_t)sms * 131072 * 16);
  cudaMalloc(&cyc, 256 * 8);
  run<1, false>(at, out, cyc, sms);
  run<2, false>(at, out, cyc, sms);
  run<3, false>(at, out, cyc, sms);
  run<4, false>(at, out, cyc, sms);
  run<6, false>(at, out, cyc, sms);
  run<2, true>(at, out, cyc, sms);
  run<4, true>(at, out, cyc, sms);
  run<6, true>(at, out, cyc, sms);
  {
    auto k = gather_tma_store<4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 16384);
    for (int r = 0; r < 2; ++r) {
      k<<<sms, 160, 4 * 32768 + 16384>>>(at, 64, (char *)out, 2 << 20, cyc);
      cudaDeviceSynchronize();
    }
    long long h[256];
    cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    printf("gathers + TMA bulk stores on the same SM: %6.1f B/clk/SM (~%5.1f GB/s/SM)\n", 64.0 * 32768 / avg,
           64.0 * 32768 / avg * 1.9);
  }
  {
    auto k = gather_spinners<3>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * 32768);
    for (int r = 0; r < 2; ++r) {
      k<<<sms, 416, 3 * 32768>>>(at, 64, cyc);
      cudaDeviceSynchronize();
    }
    long long h[256];
    cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < sms; ++i) avg += h[i];
    avg /= sms;
    printf("gather depth 3 + 9 spinning warps: %6.1f B/clk/SM (~%5.1f GB/s/SM)\n", 64.0 * 32768 / avg,
           64.0 * 32768 / avg * 1.9);
  }
  // split roles: even CTAs gather only, odd CTAs store only
  {
    auto k = split<4>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768);
    for (int r = 0; r < 2; ++r) {
      k<<<sms, 384, 4 * 32768>>>(at, 64, out, 131072 * 2, cyc);
      cudaDeviceSynchronize();
    }
    long long h[256];
    cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    int n = 0;
    for (int i = 0; i < sms; i += 2) { avg += h[i]; ++n; }
    avg /= n;
    printf("split roles (gather CTAs beside store-only CTAs): %6.1f B/clk/SM (~%5.1f GB/s/SM)\n", 64.0 * 32768 / avg,
           64.0 * 32768 / avg * 1.9);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
