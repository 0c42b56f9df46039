// Round 2: TMA gather4 issued by many warps vs the 4-warp cp.async producer,
// at soaked clocks, in TB/s.  membench11 showed gather4 issue cost is per
// warp (one thread: 8 B/clk, 4 warps x 1 lane: 21 B/clk, 1 warp x 32 lanes:
// 10 B/clk), so this sweeps the number of issuing warps.  Stages are K2's:
// 64 kept rows x 256 tokens (32 KB SW128) + a 16 KB weight block (1-D TMA),
// 4 stages in flight, a consumer warp (full -> empty).
//   P = cp.async producer warps (0 = gather4 mode), I = gather4 issuing warps
//   E = epilogue emulation after each unit: 0 none, 1 STS+LDS+STG by 8 warps
//       (the round-1 epilogue), 2 STS by 8 warps + 1-D bulk stores (one per
//       512 B row piece) issued by lane 0 of each of the 8 warps
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I ../paper_2008_13006_b200/csrc -o bin/membench13 membench13.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "tools_ptx.cuh"

using namespace tw;

constexpr int kA = 32768, kB = 16384, kDepth = 4, kOut = 32768;

struct Geo {
  int K, M, keep, tiles, units_per_cta;
};

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void soak(float *x, int iters) {
  float v = threadIdx.x;
  for (int i = 0; i < iters; ++i) v = v * 1.0000001f + 0.5f;
  if (v == 12345.f) x[0] = v;
}

template <int P, int I, int E>
__global__ void __launch_bounds__(1024, 1)
    gather(const __grid_constant__ CUtensorMap tmap, const uint16_t *at, const uint8_t *wimg, const int *kept, Geo g,
           char *out, unsigned long long *ns) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t *sA = sm, *sB = sm + kDepth * kA, *sOut = sB + kDepth * kB;
  uint64_t *full = reinterpret_cast<uint64_t *>(sOut + kOut);
  uint64_t *empty = full + kDepth;
  uint64_t *unit_done = empty + kDepth;  // [2]
  uint64_t *epi_empty = unit_done + 2;   // [2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kProd = P > 0 ? P : I;  // producer warps: 0 .. kProd-1
  constexpr int kCons = kProd;          // consumer warp
  constexpr int kEpi0 = kProd + 1;      // 8 epilogue warps
  if (threadIdx.x == 0) {
    for (int s = 0; s < kDepth; ++s) {
      ptx::mbar_init(&full[s], P > 0 ? 1u + P * 32u : 1u);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&unit_done[s], 1);
      ptx::mbar_init(&epi_empty[s], 8);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const unsigned long long t0 = gtime();
  const uint64_t keep = ptx::policy_evict_last();
  const int blocks = g.M / 256, spu = g.keep / 64;
  const int total = g.units_per_cta * spu;
  if (warp < kProd) {
    for (int i = 0; i < total; ++i) {
      const int j = i / spu, s0 = i % spu;
      const int u = (blockIdx.x + j * gridDim.x) % (g.tiles * blocks);
      const int tile = u / blocks, tb = u % blocks;
      const int stage = i % kDepth;
      if (i >= kDepth) ptx::mbar_wait(&empty[stage], (uint32_t)((i / kDepth - 1) & 1));
      const int *krows = kept + tile * g.keep + s0 * 64;
      if (threadIdx.x == 0) {
        ptx::mbar_arrive_expect_tx(&full[stage], P > 0 ? kB : kA + kB);
        ptx::bulk_g2s(sB + stage * kB, wimg + ((int64_t)(tile * spu + s0) * kB) % (4 << 20), kB, &full[stage], keep);
      }
      if constexpr (P > 0) {
        constexpr int R = 64 / P;
        const int blk = lane >> 3, cc = lane & 7;
#pragma unroll
        for (int it = 0; it < R; ++it) {
          const int r = warp * R + it;
          const void *src = at + (int64_t)__ldg(krows + r) * g.M + tb * 256 + lane * 8;
          ptx::cp_async_16_full(sA + stage * kA + blk * 8192 + r * 128 + ((cc ^ (r & 7)) * 16), src);
        }
        ptx::cp_async_mbar_arrive_noinc(&full[stage]);
      } else {
        // 64 gather4 per stage (16 row groups x 4 token blocks) over I warps, lane 0 each
        if (lane == 0) {
#pragma unroll 1
          for (int q = warp; q < 64; q += I) {
            const int grp = q >> 2, b = q & 3;
            const int4 r4 = __ldg(reinterpret_cast<const int4 *>(krows) + grp);
            ptx::tma_gather4(sA + stage * kA + b * 8192 + grp * 512, &tmap, &full[stage], tb * 256 + b * 64, r4, keep);
          }
        }
      }
    }
    if constexpr (P > 0) ptx::cp_async_wait_group<0>();
  } else if (warp == kCons) {
    for (int i = 0; i < total; ++i) {
      const int stage = i % kDepth;
      ptx::mbar_wait(&full[stage], (uint32_t)((i / kDepth) & 1));
      if (lane == 0) {
        ptx::mbar_arrive(&empty[stage]);
        if (E && i % spu == spu - 1) {
          const int j = i / spu;
          if (j >= 2) ptx::mbar_wait(&epi_empty[j & 1], (uint32_t)(((j >> 1) - 1) & 1));
          ptx::mbar_arrive(&unit_done[j & 1]);
        }
      }
      __syncwarp();
    }
  } else if (E && warp >= kEpi0 && warp < kEpi0 + 8) {
    const int e = warp - kEpi0;
    for (int j = 0; j < g.units_per_cta; ++j) {
      ptx::mbar_wait(&unit_done[j & 1], (uint32_t)((j >> 1) & 1));
      const int u = (blockIdx.x + j * gridDim.x) % (g.tiles * blocks);
      const int tile = u / blocks, tb = u % blocks;
      // 128 rows x 512 B per unit in 2 passes of 64 rows (32 KB staging)
      for (int pass = 0; pass < 2; ++pass) {
        // STS: warp e writes rows e*8 .. +8 of the pass (lane = 16 B chunk)
        for (int r = 0; r < 8; ++r)
          reinterpret_cast<uint4 *>(sOut + (e * 8 + r) * 512)[lane] = make_uint4(j, r, pass, e);
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if constexpr (E == 1) {
          for (int r = 0; r < 8; ++r) {
            const uint4 v = reinterpret_cast<const uint4 *>(sOut + (e * 8 + r) * 512)[lane];
            uint4 *dst = reinterpret_cast<uint4 *>(out + ((int64_t)(tile * 128 + pass * 64 + e * 8 + r) * g.M + tb * 256) * 2);
            __stcs(dst + lane, v);
          }
        } else {
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            for (int r = 0; r < 8; ++r) {
              char *dst = out + ((int64_t)(tile * 128 + pass * 64 + e * 8 + r) * g.M + tb * 256) * 2;
              asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 512;" ::"l"(dst),
                           "r"(ptx::smem_u32(sOut + (e * 8 + r) * 512))
                           : "memory");
            }
            ptx::bulk_commit();
            ptx::bulk_wait_read<0>();
          }
          __syncwarp();
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
      if (lane == 0) ptx::mbar_arrive(&epi_empty[j & 1]);
    }
    if (E == 2 && lane == 0) ptx::bulk_wait<0>();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ns[2 * blockIdx.x] = t0;
    ns[2 * blockIdx.x + 1] = gtime();
  }
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

struct Bufs {
  uint16_t *at;
  uint8_t *wimg;
  int *kept;
  char *out;
  unsigned long long *ns;
  CUtensorMap tmap;
};

Bufs make(Geo g) {
  Bufs b;
  cudaMalloc(&b.at, (size_t)g.K * g.M * 2);
  cudaMemset(b.at, 0, (size_t)g.K * g.M * 2);
  cudaMalloc(&b.wimg, 4 << 20);
  cudaMemset(b.wimg, 0, 4 << 20);
  cudaMalloc(&b.out, (size_t)g.tiles * 128 * g.M * 2);
  cudaMalloc(&b.ns, 4096 * 16);
  std::vector<int> hk((size_t)g.tiles * g.keep);
  std::mt19937 rng(42);
  for (int t = 0; t < g.tiles; ++t) {
    std::vector<int> p(g.K);
    for (int i = 0; i < g.K; ++i) p[i] = i;
    std::shuffle(p.begin(), p.end(), rng);
    std::sort(p.begin(), p.begin() + g.keep);
    std::copy(p.begin(), p.begin() + g.keep, hk.begin() + (size_t)t * g.keep);
  }
  cudaMalloc(&b.kept, hk.size() * 4);
  cudaMemcpy(b.kept, hk.data(), hk.size() * 4, cudaMemcpyHostToDevice);
  cuuint64_t dims[2] = {(cuuint64_t)g.M, (cuuint64_t)g.K};
  cuuint64_t strides[1] = {(cuuint64_t)g.M * 2};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t estr[2] = {1, 1};
  encode_fn()(&b.tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, b.at, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return b;
}

template <int P, int I, int E>
void run(const char *name, Geo g, const Bufs &b, int sms) {
  const int smem = kDepth * (kA + kB) + kOut + 1024 + 256;
  constexpr int kProd = P > 0 ? P : I;
  const int threads = (kProd + 1 + (E ? 8 : 0)) * 32;
  cudaFuncSetAttribute(gather<P, I, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9f, ms;
  for (int r = 0; r < 7; ++r) {
    cudaEventRecord(e0);
    gather<P, I, E><<<sms, threads, smem>>>(b.tmap, b.at, b.wimg, b.kept, g, b.out, b.ns);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  std::vector<unsigned long long> h(2 * sms);
  cudaMemcpy(h.data(), b.ns, 16 * sms, cudaMemcpyDeviceToHost);
  double avg = 0, mx = 0;
  for (int i = 0; i < sms; ++i) {
    const double d = (double)(h[2 * i + 1] - h[2 * i]);
    avg += d / sms;
    mx = std::max(mx, d);
  }
  const double in_bytes = (double)sms * g.units_per_cta * (g.keep / 64) * (kA + kB);
  const double out_bytes = E ? (double)sms * g.units_per_cta * 128 * 512 : 0;
  printf("P%d I%-2d E%d %-22s in %6.2f TB/s (CTA avg), out %5.2f TB/s | launch %7.2f us, CTA avg %6.2f slowest %6.2f (%s)\n", P,
         I, E, name, in_bytes / avg / 1e3, out_bytes / avg / 1e3, best * 1e3, avg / 1e3, mx / 1e3,
         cudaGetErrorString(cudaGetLastError()));
}

template <int E>
void sweep(const char *name, Geo g, const Bufs &b, int sms) {
  run<4, 0, E>(name, g, b, sms);
  run<0, 4, E>(name, g, b, sms);
  run<0, 8, E>(name, g, b, sms);
  run<0, 12, E>(name, g, b, sms);
  run<0, 16, E>(name, g, b, sms);
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float *x;
  cudaMalloc(&x, 64);
  for (int i = 0; i < 20; ++i) soak<<<sms * 4, 256>>>(x, 200000);
  cudaDeviceSynchronize();
  const Geo steady{768, 4096, 384, 12, 8};
  const Geo c2a{768, 4096, 384, 12, 2};
  Bufs b = make(steady);
  sweep<0>("C2a 8 u/CTA", steady, b, sms);
  sweep<1>("C2a 8 u/CTA", steady, b, sms);
  sweep<2>("C2a 8 u/CTA", steady, b, sms);
  sweep<0>("C2a 2 u/CTA", c2a, b, sms);
  sweep<1>("C2a 2 u/CTA", c2a, b, sms);
  sweep<2>("C2a 2 u/CTA", c2a, b, sms);
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
