// Per-SM memory-interface microbenchmark (B200): how many bytes per ns can one
// SM move, by path, with G active SMs?
//   bulk_in   : TMA 1-D bulk copies global(L2-resident) -> smem, 16 KB each
//   bulk_out  : TMA 1-D bulk copies smem -> global (streamed, DRAM-bound)
//   gather4   : TMA tensor gather4 (4 rows x 128 B) from an 8 KB-pitch matrix
//   cpasync   : 16 B cp.async row gathers (512 B per warp instruction), 4 warps
//   mixed     : cp.async gather (4 warps) + STG.128 stream (8 warps) together
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench4 membench4.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t n) {
  asm volatile("{\n\t.reg .b64 s;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 s, [%0], %1;\n\t}" ::"r"(su(b)), "r"(n));
}
__device__ __forceinline__ void wait_par(uint64_t *b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.b32 %0,1,0,p;\n\t}"
                 : "=r"(ok)
                 : "r"(su(b)), "r"(ph));
}

// bulk_in: each CTA streams `iters` x 16 KB from an L2-resident 8 MB buffer
__global__ void bulk_in(const char *src, int iters) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t bar[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int i = 0; i < iters; ++i) {
    const int s = i & 3;
    if (i >= 4) wait_par(&bar[s], ((i >> 2) - 1) & 1);
    expect_tx(&bar[s], 16384);
    const char *g = src + ((int64_t)(blockIdx.x * 131 + i * 7) % 512) * 16384;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 16384, [%2];" ::"r"(
                     su(sm + s * 16384)),
                 "l"(g), "r"(su(&bar[s])));
  }
  for (int s = 0; s < 4; ++s) wait_par(&bar[s], ((iters - 1 - ((iters - 1 - s) & 3)) >> 2) & 1);
}

// bulk_out: each CTA writes `iters` x 16 KB to its own region of dst
__global__ void bulk_out(char *dst, int iters) {
  extern __shared__ __align__(1024) char sm[];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sm[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  if (threadIdx.x != 0) return;
  char *base = dst + (int64_t)blockIdx.x * iters * 16384;
  for (int i = 0; i < iters; ++i) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(base + (int64_t)i * 16384),
                 "r"(su(sm)));
    asm volatile("cp.async.bulk.commit_group;");
    asm volatile("cp.async.bulk.wait_group.read 8;");
  }
  asm volatile("cp.async.bulk.wait_group 0;");
}

// gather4: 4 rows x 64 bf16 from A^T (K=768 x M=4096), warp 0 lanes 0..15 issue
__global__ void gather4(const __grid_constant__ CUtensorMap tm, int iters) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ __align__(8) uint64_t bar[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  for (int i = 0; i < iters; ++i) {  // one "stage" = 64 rows x 256 tokens = 32 KB = 64 gather4
    const int s = i & 3;
    if (lane == 0) {
      if (i >= 4) wait_par(&bar[s], ((i >> 2) - 1) & 1);
      expect_tx(&bar[s], 32768);
    }
    __syncwarp();
    for (int g = lane; g < 64; g += 32) {
      const int rb = (g & 15) * 4, tb = g >> 4;
      const int r0 = (rb * 389 + i * 13 + blockIdx.x) % 768;
      const int c0 = ((blockIdx.x * 4 + tb) * 64) % 4096;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su(sm + s * 32768 + g * 512)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c0), "r"(r0), "r"((r0 + 97) % 768), "r"((r0 + 211) % 768),
          "r"((r0 + 401) % 768), "r"(su(&bar[s])));
    }
  }
  if (lane == 0)
    for (int s = 0; s < 4; ++s) wait_par(&bar[s], ((iters - 1 - ((iters - 1 - s) & 3)) >> 2) & 1);
}

__device__ __forceinline__ void cp16(void *s, const void *g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su(s)), "l"(g) : "memory");
}
// cpasync gather (4 warps) and optionally 8 streaming-store warps
template <bool kStores>
__global__ void cpasync_mixed(const __nv_bfloat16 *at, float4 *out, int iters, int64_t out_per_cta) {
  extern __shared__ __align__(1024) char sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < 4) {
    for (int i = 0; i < iters; ++i) {
      for (int it = 0; it < 16; ++it) {
        const int r = warp * 16 + it;
        const int krow = (r * 389 + i * 13 + blockIdx.x) % 768;
        cp16(sm + (i & 3) * 32768 + r * 512 + lane * 16, at + (int64_t)krow * 4096 + ((blockIdx.x * 256) % 4096) + lane * 8);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 3;" ::: "memory");
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else if (kStores) {
    float4 *o = out + (int64_t)blockIdx.x * out_per_cta;
    for (int64_t i = (warp - 4) * 32 + lane; i < out_per_cta; i += 256) __stcs(o + i, make_float4(0, 0, 0, 0));
  }
}

typedef CUresult (*EncFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                          const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  char *src, *dst;
  __nv_bfloat16 *at;
  cudaMalloc(&src, 8 << 20);
  cudaMemset(src, 1, 8 << 20);
  cudaMalloc(&dst, (size_t)1 << 30);
  cudaMalloc(&at, 768 * 4096 * 2);
  cudaMemset(at, 0, 768 * 4096 * 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    launch();
    cudaEventRecord(a);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5;
  };
  cudaFuncSetAttribute(bulk_in, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(bulk_out, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaFuncSetAttribute(gather4, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(cpasync_mixed<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(cpasync_mixed<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {4096, 768}, strides[1] = {4096 * 2};
  cuuint32_t box[2] = {64, 1}, es[2] = {1, 1};
  ((EncFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, at, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  for (int G : {sms, sms / 2, sms / 8}) {
    const int it = 256;
    float ms = timeit([&] { bulk_in<<<G, 32, 65536>>>(src, it); });
    printf("G=%3d bulk_in   %7.1f GB/s/SM  (%7.0f GB/s total)\n", G, (double)it * 16384 / (ms * 1e6), (double)G * it * 16384 / (ms * 1e6));
    ms = timeit([&] { bulk_out<<<G, 32, 16384>>>(dst, it); });
    printf("G=%3d bulk_out  %7.1f GB/s/SM  (%7.0f GB/s total)\n", G, (double)it * 16384 / (ms * 1e6), (double)G * it * 16384 / (ms * 1e6));
    ms = timeit([&] { gather4<<<G, 32, 131072>>>(tm, 64); });
    printf("G=%3d gather4   %7.1f GB/s/SM  (%7.0f GB/s total)\n", G, 64.0 * 32768 / (ms * 1e6), (double)G * 64 * 32768 / (ms * 1e6));
    ms = timeit([&] { cpasync_mixed<false><<<G, 128, 131072>>>(at, nullptr, 64, 0); });
    printf("G=%3d cpasync   %7.1f GB/s/SM  (%7.0f GB/s total)\n", G, 64.0 * 32768 / (ms * 1e6), (double)G * 64 * 32768 / (ms * 1e6));
    const int64_t opc = 2ll << 20;  // 2M float4 = 32 MB? no: 2M*16B = 32 MB per CTA is too much; use 128K float4 = 2 MB
    ms = timeit([&] { cpasync_mixed<true><<<G, 384, 131072>>>(at, (float4 *)dst, 64, 131072); });
    printf("G=%3d mixed     %7.1f GB/s/SM in+out (%.1f us)\n", G, (64.0 * 32768 + 131072.0 * 16) / (ms * 1e6), ms * 1e3);
    (void)opc;
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
