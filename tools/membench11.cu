// Round 2: is TMA gather4 (+ TMA bulk stores) a faster A^T row gather than
// 16-byte cp.async on B200?  Kernel-like producer on the C2a / C5 layer
// geometry: stages of 64 kept rows x 256 tokens (32 KB, SW128 blocks) + a
// 16 KB weight block, 4 stages in flight, units in the kernel's order.
//   mode 0: cp.async, 4 producer warps (the round-1 kernel's producer)
//   mode 1: TMA gather4, one thread issues the whole stage (64 x gather4)
//   mode 2: TMA gather4, lane 0 of each of the 4 producer warps issues 16
//   mode 3: TMA gather4, every lane of one warp issues 2 (lane-parallel issue)
// +stores: a store warp emulates the epilogue: after each unit's last stage
// it writes 128 C^T row pieces (256 tokens x 2 B) and its share of zero rows
//   (st 1) with 1-D TMA bulk stores from a staging buffer, or
//   (st 2) with 16-byte STG from registers (8 warps).
// Also: launch overhead of an empty 416-thread / 227 KB kernel, back to back
// in a CUDA graph, with and without programmatic dependent launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I ../paper_2008_13006_b200/csrc -o bin/membench11 membench11.cu -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "tools_ptx.cuh"

using namespace tw;

constexpr int kA = 32768, kB = 16384, kDepth = 4, kStageOut = 32768;

struct Geo {
  int K, M, keep, tiles, units_per_cta;
  int zero_rows_per_unit;  // 8 KB-row zero rows written per unit (store emulation)
};

__device__ __forceinline__ void bulk_s2g(void *g, const void *s, uint32_t n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(ptx::smem_u32(s)), "r"(n)
               : "memory");
}

template <int kMode, int kSt>
__global__ void __launch_bounds__(416, 1)
    gather(const __grid_constant__ CUtensorMap tmap, const __nv_bfloat16 *at, const uint8_t *wimg, const int *kept, Geo g,
           char *out, long long *cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = sm, *sB = sm + kDepth * kA, *sOut = sB + kDepth * kB;
  uint64_t *full = reinterpret_cast<uint64_t *>(sOut + kStageOut);
  uint64_t *empty = full + kDepth;
  uint64_t *unit_done = empty + kDepth;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t full_count = kMode == 0 ? 129u : 1u;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDepth; ++s) {
      ptx::mbar_init(&full[s], full_count);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(unit_done, 1);
    ptx::fence_mbar_init();
  }
  for (int i = threadIdx.x; i < kStageOut / 16; i += blockDim.x) reinterpret_cast<uint4 *>(sOut)[i] = make_uint4(0, 0, 0, 0);
  ptx::fence_proxy_async_smem();
  __syncthreads();
  const uint64_t keep = ptx::policy_evict_last();
  const int blocks = g.M / 256, spu = g.keep / 64;
  const int total = g.units_per_cta * spu;
  long long t0 = clock64();
  if (warp < 4) {
    for (int i = 0; i < total; ++i) {
      const int j = i / spu, s0 = i % spu;
      const int u = (blockIdx.x + j * gridDim.x) % (g.tiles * blocks);
      const int tile = u / blocks, tb = u % blocks;
      const int stage = i % kDepth;
      if (i >= kDepth) ptx::mbar_wait(&empty[stage], (uint32_t)((i / kDepth - 1) & 1));
      const int *krows = kept + tile * g.keep + s0 * 64;
      if (threadIdx.x == 0) {
        ptx::mbar_arrive_expect_tx(&full[stage], kMode == 0 ? kB : kA + kB);
        ptx::bulk_g2s(sB + stage * kB, wimg + ((int64_t)(tile * spu + s0) * kB) % (4 << 20), kB, &full[stage], keep);
      }
      if constexpr (kMode == 0) {
        const int blk = lane >> 3, cc = lane & 7;
#pragma unroll
        for (int it = 0; it < 16; ++it) {
          const int r = warp * 16 + it;
          const void *src = at + (int64_t)krows[r] * g.M + tb * 256 + lane * 8;
          ptx::cp_async_16_full(sA + stage * kA + blk * 8192 + r * 128 + ((cc ^ (r & 7)) * 16), src);
        }
        ptx::cp_async_mbar_arrive_noinc(&full[stage]);
      } else if constexpr (kMode == 1) {
        if (threadIdx.x == 0) {
          for (int grp = 0; grp < 16; ++grp) {
            const int4 r4 = reinterpret_cast<const int4 *>(krows)[grp];
#pragma unroll
            for (int b = 0; b < 4; ++b)
              ptx::tma_gather4(sA + stage * kA + b * 8192 + grp * 512, &tmap, &full[stage], tb * 256 + b * 64, r4, keep);
          }
        }
      } else if constexpr (kMode == 2) {
        if (lane == 0) {
          for (int q = 0; q < 4; ++q) {
            const int grp = warp * 4 + q;
            const int4 r4 = reinterpret_cast<const int4 *>(krows)[grp];
#pragma unroll
            for (int b = 0; b < 4; ++b)
              ptx::tma_gather4(sA + stage * kA + b * 8192 + grp * 512, &tmap, &full[stage], tb * 256 + b * 64, r4, keep);
          }
        }
      } else {
        if (warp == 0) {
          // lane l: row group l / 2 (16 groups), 64-token blocks 2 (l & 1) .. +1
          const int grp = lane >> 1;
          const int4 r4 = reinterpret_cast<const int4 *>(krows)[grp];
#pragma unroll
          for (int bb = 0; bb < 2; ++bb) {
            const int b = (lane & 1) * 2 + bb;
            ptx::tma_gather4(sA + stage * kA + b * 8192 + grp * 512, &tmap, &full[stage], tb * 256 + b * 64, r4, keep);
          }
        }
      }
    }
    if constexpr (kMode == 0) ptx::cp_async_wait_group<0>();
  } else if (warp == 4) {
    // consumer: full -> empty (the MMA warp's protocol, no MMA), and unit_done per unit
    for (int i = 0; i < total; ++i) {
      const int stage = i % kDepth;
      ptx::mbar_wait(&full[stage], (uint32_t)((i / kDepth) & 1));
      if (lane == 0) {
        ptx::mbar_arrive(&empty[stage]);
        if (i % spu == spu - 1) ptx::mbar_arrive(unit_done);
      }
      __syncwarp();
    }
  } else if (kSt == 1 && warp == 5) {
    // TMA bulk stores of each finished unit: 128 rows x 512 B + zero rows (8 KB bulks)
    for (int j = 0; j < g.units_per_cta; ++j) {
      ptx::mbar_wait(unit_done, (uint32_t)(j & 1));
      const int u = (blockIdx.x + j * gridDim.x) % (g.tiles * blocks);
      const int tile = u / blocks, tb = u % blocks;
      if (lane == 0) {
        for (int r = 0; r < 128; ++r) {
          char *dst = out + ((int64_t)(tile * 128 + r) * g.M + tb * 256) * 2;
          bulk_s2g(dst, sOut + (r & 63) * 512, 512);
        }
        for (int z = 0; z < g.zero_rows_per_unit; ++z) {
          char *dst = out + ((int64_t)(g.tiles * 128 + (u * g.zero_rows_per_unit + z) % (g.tiles * 128)) * g.M) * 2;
          for (int o = 0; o < g.M * 2; o += 8192) bulk_s2g(dst + o, sOut, 8192);
        }
        ptx::bulk_commit();
      }
    }
    if (lane == 0) ptx::bulk_wait<0>();
  } else if (kSt == 2 && warp >= 5) {
    const int e = warp - 5;  // 8 warps
    for (int j = 0; j < g.units_per_cta; ++j) {
      ptx::mbar_wait(unit_done, (uint32_t)(j & 1));
      const int u = (blockIdx.x + j * gridDim.x) % (g.tiles * blocks);
      const int tile = u / blocks, tb = u % blocks;
      // two rows per instruction (16 lanes x 16 B = 256 tokens x 2 B per row... 512 B = 32 lanes)
      for (int r = e; r < 128; r += 8) {
        uint4 *dst = reinterpret_cast<uint4 *>(out + ((int64_t)(tile * 128 + r) * g.M + tb * 256) * 2);
        __stcs(dst + lane, make_uint4(0, 0, 0, 0));
      }
      for (int z = e; z < g.zero_rows_per_unit; z += 8) {
        uint4 *dst = reinterpret_cast<uint4 *>(out + ((int64_t)(g.tiles * 128 + (u * g.zero_rows_per_unit + z) % (g.tiles * 128)) * g.M) * 2);
        for (int o = lane; o < g.M * 2 / 16; o += 32) __stcs(dst + o, make_uint4(0, 0, 0, 0));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

__global__ void __launch_bounds__(416, 1) empty_kernel(int pdl) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 1000) smem_raw[0] = 1;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *, const cuuint64_t *,
                             const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn encode_fn() {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<EncodeFn>(p);
}

template <int kMode, int kSt>
void run(const char *name, Geo g, long long *cyc, int sms) {
  __nv_bfloat16 *at;
  uint8_t *wimg;
  int *kept;
  char *out;
  const size_t out_bytes = (size_t)g.tiles * 256 * g.M * 2;
  cudaMalloc(&at, (size_t)g.K * g.M * 2);
  cudaMemset(at, 0, (size_t)g.K * g.M * 2);
  cudaMalloc(&wimg, 4 << 20);
  cudaMemset(wimg, 0, 4 << 20);
  cudaMalloc(&out, out_bytes);
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
  CUtensorMap tmap;
  cuuint64_t dims[2] = {(cuuint64_t)g.M, (cuuint64_t)g.K};
  cuuint64_t strides[1] = {(cuuint64_t)g.M * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, at, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) printf("encode failed %d\n", (int)r);
  const int smem = kDepth * (kA + kB) + kStageOut + 1024 + 256;
  cudaFuncSetAttribute(gather<kMode, kSt>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0.f, best = 1e9f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(out, 1, out_bytes);  // evict / dirty
    cudaEventRecord(e0);
    gather<kMode, kSt><<<sms, 416, smem>>>(tmap, at, wimg, kept, g, out, cyc);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  long long h[256];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0, mx = 0;
  for (int i = 0; i < sms; ++i) {
    avg += h[i];
    mx = std::max(mx, (double)h[i]);
  }
  avg /= sms;
  const double bytes = (double)g.units_per_cta * (g.keep / 64) * (kA + kB);
  printf("mode %d st %d %-34s A+W %6.1f B/clk/SM avg, slowest %6.1f, launch %7.2f us (%s)\n", kMode, kSt, name,
         bytes / avg, bytes / mx, best * 1e3, cudaGetErrorString(cudaGetLastError()));
  cudaFree(at);
  cudaFree(wimg);
  cudaFree(kept);
  cudaFree(out);
}

template <int kSt>
void all_modes(const char *name, Geo g, long long *cyc, int sms) {
  run<0, kSt>(name, g, cyc, sms);
  run<1, kSt>(name, g, cyc, sms);
  run<2, kSt>(name, g, cyc, sms);
  run<3, kSt>(name, g, cyc, sms);
}

void launch_overhead(int sms) {
  const int smem = 227 * 1024;
  cudaFuncSetAttribute(empty_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int small = 0; small < 2; ++small) {
      cudaGraph_t graph;
      cudaGraphExec_t exec;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int i = 0; i < 100; ++i) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(sms);
        cfg.blockDim = dim3(416);
        cfg.dynamicSmemBytes = small ? 0 : smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl;
        cudaLaunchKernelEx(&cfg, empty_kernel, pdl);
      }
      cudaStreamEndCapture(s, &graph);
      cudaGraphInstantiate(&exec, graph, 0);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float best = 1e9f, ms;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0, s);
        cudaGraphLaunch(exec, s);
        cudaEventRecord(e1, s);
        cudaStreamSynchronize(s);
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
      }
      printf("empty kernel x100 in a graph, 416 thr, smem %s, pdl %d: %.2f us per launch (%s)\n", small ? "0" : "227K",
             pdl, best * 10.f, cudaGetErrorString(cudaGetLastError()));
    }
  }
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long *cyc;
  cudaMalloc(&cyc, 256 * 8);
  launch_overhead(sms);
  // C2a: 12 tiles x 16 token blocks = 192 units; 2 units per CTA; zero rows 1536 x 8 KB / 192 units = 8 per unit
  const Geo c2a{768, 4096, 384, 12, 2, 8};
  const Geo c5{1024, 16384, 512, 16, 7, 2};
  all_modes<0>("C2a gathers only", c2a, cyc, sms);
  all_modes<1>("C2a + TMA bulk stores", c2a, cyc, sms);
  all_modes<2>("C2a + STG stores", c2a, cyc, sms);
  all_modes<0>("C5@75 gathers only", c5, cyc, sms);
  all_modes<1>("C5@75 + TMA bulk stores", c5, cyc, sms);
  all_modes<2>("C5@75 + STG stores", c5, cyc, sms);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
