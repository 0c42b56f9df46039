// C ABI (include/tw_b200.h): plan upload, argument checking and the launch
// wrappers of libtw_b200.so.
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "tw_internal.h"

namespace tw {
int tokens_per_unit(int block_n);
cudaError_t launch_tw_gemm_sm100(const GemmArgs &args, int out_dtype, int grid, int tb, cudaStream_t stream);
cudaError_t launch_tw_pair_sm100(const GemmArgs &args, int out_dtype, int grid, cudaStream_t stream);
int pair_clusters_max(int out_dtype);
cudaError_t launch_prep(const float *a, int64_t m, int64_t k, int layout, void *at, int64_t ldat, int out_dtype,
                        cudaStream_t s);
cudaError_t launch_spmm(const void *at, int at_dtype, int64_t m, int64_t k, int64_t lda, int64_t col_begin, int64_t n_cols,
                        const int32_t *cp, const int32_t *ri, const float *va, void *ct, int64_t ldc, int out_dtype,
                        int accumulate, cudaStream_t s);
cudaError_t launch_prep_split(const float *a, int64_t m, int64_t k, int layout, void *at, int64_t ldat, cudaStream_t s);
cudaError_t launch_exact(const tw_plan *p, const float *at, int64_t m, int64_t lda, float *ct, int64_t ldc,
                         cudaStream_t s);
cudaError_t launch_prune_means(const double *s, int64_t k, int64_t n, const int32_t *cols, const int64_t *off,
                               int64_t n_tiles, double *out, cudaStream_t st);


namespace {

int cuda_fail(cudaError_t e, const char *what) {
  return fail(TW_ERR_CUDA, std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

int sm_count_of_current(int *sms, int *major) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  static int cache_sms[64] = {0}, cache_major[64] = {0};
  if (dev < 64 && cache_sms[dev]) {
    *sms = cache_sms[dev];
    *major = cache_major[dev];
    return TW_OK;
  }
  int s = 0, mj = 0;
  if ((e = cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess)
    return cuda_fail(e, "cudaDeviceGetAttribute");
  if ((e = cudaDeviceGetAttribute(&mj, cudaDevAttrComputeCapabilityMajor, dev)) != cudaSuccess)
    return cuda_fail(e, "cudaDeviceGetAttribute");
  if (dev < 64) { cache_sms[dev] = s; cache_major[dev] = mj; }
  *sms = s;
  *major = mj;
  return TW_OK;
}

int require_sm100(int *sms) {
  int major = 0;
  int rc = sm_count_of_current(sms, &major);
  if (rc) return rc;
  if (major != 10) return fail(TW_ERR_CUDA, "libtw_b200 requires an sm_100 (B200) device; found compute capability " +
                                                std::to_string(major) + ".x");
  // experiment knob: schedule for fewer SMs (profiling only)
  static const int cap = [] {
    const char *e = std::getenv("TW_B200_SMS");
    return e ? std::atoi(e) : 0;
  }();
  if (cap > 0 && cap < *sms) *sms = cap;
  return TW_OK;
}

template <typename T>
int upload(T **dst, const std::vector<T> &src) {
  *dst = nullptr;
  if (src.empty()) return TW_OK;
  cudaError_t e = cudaMalloc(reinterpret_cast<void **>(dst), src.size() * sizeof(T));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  e = cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy");
  return TW_OK;
}

int out_size(int dtype) { return dtype == TW_F32 ? 4 : 2; }

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda:
// the .so still loads on a CPU-only host)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// Makes the plan's GPU current for the lifetime of the guard (schedules are
// uploaded and kernels launched on the device that holds the plan, whatever
// device the caller has current), restoring the caller's device after.
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (dev < 0) return;
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && prev != dev) err = cudaSetDevice(dev);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void free_schedule(tw_dev_schedule &ds) {
  cudaFree(ds.units);
  cudaFree(ds.off);
  cudaFree(ds.zoff);
  cudaFree(ds.stream);
  cudaFree(ds.soff);
  ds = tw_dev_schedule{};
}

// CTA pairs of K4 that fit the device at once (persistent grid), per output
// dtype; 0 when the kernel cannot be launched as a cluster here.
int pair_cluster_count(int out_dtype) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, int> cache;  // (device, dtype)
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, out_dtype});
  if (it != cache.end()) return it->second;
  const int n = pair_clusters_max(out_dtype);
  cache[{dev, out_dtype}] = n;
  return n;
}

// K4 runs a pair_ok plan when the layer fills at least one wave of the
// device's CTA pairs (smaller layers: K2's 128-column units spread wider).
int pair_clusters_for(const tw_plan *p, int64_t m, int out_dtype, bool force = false) {
  if (!p->pair_ok) return 0;
  const int c = pair_cluster_count(out_dtype);
  if (c <= 0) return 0;
  if (force) return c;
  // Stage-makespan model of both kernels (B200 measurements):
  // a K4 stage (2 x 128 x 256 x 64 MACs per pair) ~0.44 us, every pair runs
  // ceil(units / pairs) units of ceil(K / 64) stages; a K2 stage (128 x 256
  // tokens x 64 kept rows) ~0.75 us, a 128-token tail stage ~0.62 us, the
  // CTAs run the unpadded plan's ceil(kbar / 64) stages per unit.  K4 also
  // needs half a wave of pairs (tiny layers: K2's units spread wider).
  const HostPlan &hp = p->host;
  const int64_t L = (int64_t)hp.tiles.size();
  const int64_t blocks = (m + 255) / 256;
  const int64_t u4 = blocks * ((L + 1) / 2);
  if (2 * u4 < c) return 0;
  const double t4 = 0.44 * (double)((u4 + c - 1) / c) * (double)((hp.k + 63) / 64);
  const int64_t kbar = L > 0 ? (hp.kept_rows_live + L - 1) / L : hp.k;
  const int64_t u2 = blocks * L, sms = 2 * (int64_t)c;
  const double waves2 = (double)(u2 / sms) * 0.75 + (u2 % sms == 0 ? 0.0 : (u2 % sms <= sms / 2 ? 0.62 : 0.75));
  const double t2 = waves2 * (double)((kbar + 63) / 64);
  return t4 < t2 ? c : 0;
}

// Static schedule for (M, output width, zero rows on/off), built once per
// launch shape and cached on the plan (uploaded to the plan's device).
int get_schedule(const tw_plan *p, int64_t m, int ob, bool zero_rows, int sms, const tw_dev_schedule **out,
                 int pair_clusters = 0) {
  std::lock_guard<std::mutex> lk(p->sched_mu);
  const auto key = std::make_tuple(m, ob + (pair_clusters > 0 ? 100 : 0), zero_rows ? 1 : 0);
  auto it = p->sched.find(key);
  if (it != p->sched.end()) {
    *out = &it->second;
    return TW_OK;
  }
  HostSchedule hs;
  int rc = pair_clusters > 0 ? build_pair_schedule(p->host, m, ob, zero_rows, pair_clusters, hs)
                             : build_schedule(p->host, m, ob, zero_rows, sms, tokens_per_unit(p->host.block_n), hs);
  if (rc) return rc;
  if (hs.units.empty()) hs.units.assign(4, 0);
  tw_dev_schedule ds;
  ds.grid = hs.grid;
  ds.has_contig = hs.has_contig;
  ds.has_tma_rows = hs.has_tma_rows;
  ds.pair = hs.pair;
  ds.zero_cpr = hs.zero_cpr;
  ds.zero_chunk = hs.zero_chunk;
  // the K2 instantiation: the narrowest unit width that holds every piece
  // (narrow kernels run deeper pipelines; TW_B200_NARROW=0 keeps the wide one)
  static const bool narrow = [] {
    const char *e = std::getenv("TW_B200_NARROW");
    return !(e && e[0] == '0');
  }();
  ds.tb = narrow ? std::max(64, 64 * hs.max_nq) : 256;
  ds.h_off = hs.off;
  ds.h_soff = hs.soff;
  ds.h_zoff = hs.zoff;
  std::vector<int4> units(hs.units.size() / 4);
  for (size_t i = 0; i < units.size(); ++i)
    units[i] = make_int4(hs.units[4 * i], hs.units[4 * i + 1], hs.units[4 * i + 2], hs.units[4 * i + 3]);
  if (hs.stream.empty()) hs.stream.assign(68, -1);
  if ((rc = upload(&ds.units, units)) || (rc = upload(&ds.off, hs.off)) || (rc = upload(&ds.zoff, hs.zoff)) ||
      (rc = upload(&ds.stream, hs.stream)) || (rc = upload(&ds.soff, hs.soff))) {
    free_schedule(ds);
    return rc;
  }
  auto ins = p->sched.emplace(key, ds);
  *out = &ins.first->second;
  return TW_OK;
}

}  // namespace
}  // namespace tw

using namespace tw;

extern "C" {

int tw_copy_2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width_bytes, int64_t height,
               int kind, void *stream) {
  clear_error();
  if (width_bytes < 0 || height < 0 || dpitch < width_bytes || spitch < width_bytes)
    return fail(TW_ERR_DIMENSION, "bad 2-D copy extents");
  if (width_bytes == 0 || height == 0) return TW_OK;
  const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
  cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width_bytes, (size_t)height, k,
                                    reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy2DAsync");
  return TW_OK;
}

int tw_device_sm_count(int *sms) {
  int major = 0;
  return sm_count_of_current(sms, &major);
}

int tw_plan_create_ex(int64_t k, int64_t n, int64_t g, int64_t n_tiles, const int64_t *col_off, const int32_t *col_ids,
                      const uint32_t *row_mask_words, const float *subs, const int64_t *sub_off, int in_dtype,
                      int64_t col_begin, int64_t col_end, int flags, tw_plan **out) {
  clear_error();
  if (!out) return fail(TW_ERR_ARG, "null out");
  *out = nullptr;
  tw_plan *p = new (std::nothrow) tw_plan();
  if (!p) return fail(TW_ERR_NOMEM, "out of host memory");
  int rc = build_host_plan(k, n, g, n_tiles, col_off, col_ids, row_mask_words, subs, sub_off, in_dtype, col_begin,
                           col_end, p->host, flags);
  if (rc) { delete p; return rc; }
  cudaGetDevice(&p->device);
  p->pair_ok = pair_eligible(p->host);
  if ((rc = upload(&p->d_tiles, p->host.tiles)) || (rc = upload(&p->d_kidx, p->host.kidx)) ||
      (rc = upload(&p->d_colids, p->host.colids)) || (rc = upload(&p->d_zero, p->host.zero_rows)) ||
      (rc = upload(&p->d_wimg, p->host.wimg)) || (rc = upload(&p->d_w32, p->host.w32)) ||
      (rc = upload(&p->d_w32_off, p->host.w32_off))) {
    tw_plan_destroy(p);
    return rc;
  }
  *out = p;
  return TW_OK;
}

int tw_plan_create(int64_t k, int64_t n, int64_t g, int64_t n_tiles, const int64_t *col_off, const int32_t *col_ids,
                   const uint32_t *row_mask_words, const float *subs, const int64_t *sub_off, int in_dtype,
                   int64_t col_begin, int64_t col_end, tw_plan **out) {
  return tw_plan_create_ex(k, n, g, n_tiles, col_off, col_ids, row_mask_words, subs, sub_off, in_dtype, col_begin,
                           col_end, 0, out);
}

int tw_plan_build_host(int64_t k, int64_t n, int64_t g, int64_t n_tiles, const int64_t *col_off,
                       const int32_t *col_ids, const uint32_t *row_mask_words, const float *subs,
                       const int64_t *sub_off, int in_dtype, int64_t col_begin, int64_t col_end, tw_plan **out) {
  clear_error();
  if (!out) return fail(TW_ERR_ARG, "null out");
  *out = nullptr;
  tw_plan *p = new (std::nothrow) tw_plan();
  if (!p) return fail(TW_ERR_NOMEM, "out of host memory");
  p->device = -1;
  int rc = build_host_plan(k, n, g, n_tiles, col_off, col_ids, row_mask_words, subs, sub_off, in_dtype, col_begin,
                           col_end, p->host);
  if (rc) { delete p; return rc; }
  *out = p;
  return TW_OK;
}

int tw_plan_destroy(tw_plan *p) {
  if (!p) return TW_OK;
  if (p->device < 0) { delete p; return TW_OK; }
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != p->device) cudaSetDevice(p->device);
  cudaFree(p->d_tiles);
  cudaFree(p->d_kidx);
  cudaFree(p->d_colids);
  cudaFree(p->d_zero);
  cudaFree(p->d_wimg);
  cudaFree(p->d_w32);
  cudaFree(p->d_w32_off);
  for (auto &kv : p->sched) free_schedule(kv.second);
  if (prev != p->device) cudaSetDevice(prev);
  delete p;
  return TW_OK;
}

static int gemm_impl(const tw_plan *p, const void *at, int64_t m, int64_t lda, void *ct, int64_t ldc,
                     int out_dtype, int accumulate, int64_t *trace, void *stream, const float *bias = nullptr,
                     int relu = 0, void *const *peers = nullptr, int n_peer = 0);

int tw_gemm(const tw_plan *p, const void *at, int64_t m, int64_t lda, void *ct, int64_t ldc, int out_dtype,
            int accumulate, void *stream) {
  return gemm_impl(p, at, m, lda, ct, ldc, out_dtype, accumulate, nullptr, stream);
}

int tw_gemm_bias(const tw_plan *p, const void *at, int64_t m, int64_t lda, void *ct, int64_t ldc, int out_dtype,
                 const float *bias, int relu, void *stream) {
  if (!bias) return fail(TW_ERR_ARG, "null bias");
  return tw_gemm_ex(p, at, m, lda, ct, ldc, out_dtype, 0, bias, relu, stream);
}

int tw_gemm_ex(const tw_plan *p, const void *at, int64_t m, int64_t lda, void *ct, int64_t ldc, int out_dtype,
               int flags, const float *bias, int relu, void *stream) {
  if (!p) return fail(TW_ERR_ARG, "null plan");
  if ((flags & TW_GEMM_ACCUMULATE) && bias) return fail(TW_ERR_ARG, "bias epilogue cannot accumulate");
  // bias is indexed by global output column; the kernel indexes by plan row
  return gemm_impl(p, at, m, lda, ct, ldc, out_dtype, flags, nullptr, stream, bias ? bias + p->host.col_begin : nullptr,
                   relu ? 1 : 0);
}

int tw_gemm_peers(const tw_plan *p, const void *at, int64_t m, int64_t lda, void *const *cts, int n_ct, int64_t ldc,
                  int out_dtype, void *stream) {
  clear_error();
  if (!p || !cts) return fail(TW_ERR_ARG, "null pointer");
  if (n_ct < 1 || n_ct > 1 + TW_MAX_PEERS) return fail(TW_ERR_ARG, "need 1 .. 1 + TW_MAX_PEERS output replicas");
  for (int d = 0; d < n_ct; ++d) {
    if (!cts[d]) return fail(TW_ERR_ARG, "null output replica");
    if ((reinterpret_cast<uintptr_t>(cts[d]) & 15) != (reinterpret_cast<uintptr_t>(cts[0]) & 15))
      return fail(TW_ERR_ARG, "output replicas must share their 16-byte alignment");
  }
  return gemm_impl(p, at, m, lda, cts[0], ldc, out_dtype, 0, nullptr, stream, nullptr, 0, cts + 1, n_ct - 1);
}

int tw_ipc_alloc(int64_t bytes, void **ptr, void *handle) {
  clear_error();
  if (!ptr || !handle || bytes < 1) return fail(TW_ERR_ARG, "bad ipc allocation request");
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e != cudaSuccess) return cuda_fail(e, "tw_ipc_alloc cudaMalloc");
  cudaIpcMemHandle_t h;
  e = cudaIpcGetMemHandle(&h, *ptr);
  if (e != cudaSuccess) {
    cudaFree(*ptr);
    *ptr = nullptr;
    return cuda_fail(e, "cudaIpcGetMemHandle");
  }
  std::memcpy(handle, &h, sizeof(h));
  return TW_OK;
}

int tw_ipc_free(void *ptr) {
  clear_error();
  if (!ptr) return TW_OK;
  cudaError_t e = cudaFree(ptr);
  return e == cudaSuccess ? TW_OK : cuda_fail(e, "tw_ipc_free");
}

int tw_ipc_open(const void *handle, void **ptr) {
  clear_error();
  if (!handle || !ptr) return fail(TW_ERR_ARG, "null pointer");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  return e == cudaSuccess ? TW_OK : cuda_fail(e, "cudaIpcOpenMemHandle");
}

int tw_ipc_close(void *ptr) {
  clear_error();
  if (!ptr) return TW_OK;
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  return e == cudaSuccess ? TW_OK : cuda_fail(e, "cudaIpcCloseMemHandle");
}

int tw_gemm_traced(const tw_plan *p, const void *at, int64_t m, int64_t lda, void *ct, int64_t ldc, int out_dtype,
                   int64_t *trace, void *stream) {
  if (!trace) return fail(TW_ERR_ARG, "null trace buffer");
  return gemm_impl(p, at, m, lda, ct, ldc, out_dtype, 0, trace, stream);
}

static int gemm_impl(const tw_plan *p, const void *at, int64_t m, int64_t lda, void *ct, int64_t ldc,
                     int out_dtype, int accumulate, int64_t *trace, void *stream, const float *bias, int relu,
                     void *const *peers, int n_peer) {
  clear_error();
  if (!p) return fail(TW_ERR_ARG, "null plan");
  if (p->device < 0) return fail(TW_ERR_ARG, "host-only plan (tw_plan_build_host) cannot run on the GPU");
  DeviceGuard guard(p->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice(plan device)");
  if (out_dtype != TW_F32 && out_dtype != TW_BF16 && out_dtype != TW_F16) return fail(TW_ERR_ARG, "bad out_dtype");
  if (m < 0) return fail(TW_ERR_DIMENSION, "M must be >= 0");
  if (m == 0) return TW_OK;
  const HostPlan &hp = p->host;
  const int64_t n_rows = hp.col_end - hp.col_begin;
  if (n_rows == 0) return TW_OK;
  if (m > (int64_t)1 << 30) return fail(TW_ERR_UNSUPPORTED, "M too large");
  if (ldc < m) return fail(TW_ERR_DIMENSION, "ldc < M");
  if (!ct) return fail(TW_ERR_ARG, "null output");
  int sms = 0;
  int rc = require_sm100(&sms);
  if (rc) return rc;
  const int64_t n_live = (int64_t)hp.tiles.size();
  if (n_live > 0) {
    if (!at) return fail(TW_ERR_ARG, "null activations");
    if (lda < m) return fail(TW_ERR_DIMENSION, "lda < M");
    if (lda % 8 != 0 || (reinterpret_cast<uintptr_t>(at) & 15) != 0)
      return fail(TW_ERR_ARG, "activations need lda % 8 == 0 and a 16-byte aligned base (16-byte row gathers)");
  }
  const tw_dev_schedule *sched = nullptr;
  const bool accum = (accumulate & TW_GEMM_ACCUMULATE) != 0;
  const bool keep_pruned = (accumulate & TW_GEMM_KEEP_PRUNED) != 0;
  const int ob = out_size(out_dtype);
  // K4 (CTA-pair kernel) for plans whose tiles keep every row in order, when
  // the output takes 16-byte bulk / TMA stores (TW_B200_PAIR=0 disables)
  static const bool pair_env = [] {
    const char *e = std::getenv("TW_B200_PAIR");
    return !(e && e[0] == '0');
  }();
  int pair_clusters = 0;
  if (pair_env && p->pair_ok && !accum && n_peer == 0 && trace == nullptr && hp.a_rows == hp.k &&
      (reinterpret_cast<uintptr_t>(ct) & 15) == 0 && (ldc * ob) % 16 == 0 && (m * ob) % 16 == 0)
    pair_clusters = pair_clusters_for(p, m, out_dtype, (accumulate & TW_GEMM_FORCE_PAIR) != 0);
  if ((rc = get_schedule(p, m, ob, !accum && !keep_pruned, sms, &sched, pair_clusters))) return rc;
  GemmArgs a{};
  a.tiles = p->d_tiles;
  a.kidx = p->d_kidx;
  a.colids = p->d_colids;
  a.zero_rows = p->d_zero;
  a.zero_cpr = sched->zero_cpr;
  a.zero_chunk = sched->zero_chunk;
  a.wimg = p->d_wimg;
  a.sched = sched->units;
  a.sched_off = sched->off;
  a.zero_off = sched->zoff;
  a.stream = sched->stream;
  a.stream_off = sched->soff;
  a.out = ct;
  a.ldc = ldc;
  a.at = at;
  a.lda = lda;
  a.M = (int32_t)m;
  a.accumulate = accum ? 1 : 0;
  a.keep_pruned = keep_pruned ? 1 : 0;
  a.no_pdl = (accumulate & TW_GEMM_NO_PDL) ? 1 : 0;
  a.wbytes = hp.wrows * 128;
  // kind::f16 instruction descriptor: D f32 [4,6)=1, A/B bf16 [7,10)/[10,13)=1
  // (fp16 = 0), A (weights) K-major [15]=0, B (gathered A^T) MN-major [16]=1,
  // M=128 tile columns -> [24,29)=8; N (tokens) is set per unit in the kernel.
  const uint32_t ab = hp.in_dtype == TW_BF16 ? 1u : 0u;
  a.idesc = (1u << 4) | (ab << 7) | (ab << 10) | (1u << 16) | ((128u >> 4) << 24);
  a.block_n = hp.block_n;
  if (sched->has_contig || sched->pair) {
    // A^T as a 2-D tensor (tokens innermost) for the TMA tile loads of
    // consecutive-row stages: box 64 tokens x 64 rows, 128B swizzle (the
    // layout the row gathers produce); out-of-range tokens read as zero
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return fail(TW_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)hp.a_rows};
    cuuint64_t strides[1] = {(cuuint64_t)lda * 2};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&a.tmap_at, hp.in_dtype == TW_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                     2, const_cast<void *>(at), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  }
  if (sched->pair) {
    // the weight image as a 2-D tensor of 128-byte rows (already swizzled:
    // copied verbatim), box = one 128-row weight block
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return fail(TW_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {64, (cuuint64_t)(hp.wimg.size() / 128)};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {64, (cuuint32_t)hp.wrows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&a.tmap_w, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, p->d_wimg, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_CUDA, "cuTensorMapEncodeTiled (weights) failed: " + std::to_string((int)r));
  }
  if (sched->has_tma_rows && !accum && n_peer == 0 && (reinterpret_cast<uintptr_t>(ct) & 15) == 0 &&
      (ldc * ob) % 16 == 0) {
    // C^T as a 2-D tensor (tokens innermost) for the epilogue's TMA tensor
    // stores: box 128 B of tokens x 128 rows, 128B swizzle (the staging
    // layout); tokens >= M are clipped by the TMA unit
    EncodeTiledFn enc = encode_tiled();
    if (!enc) return fail(TW_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)n_rows};
    cuuint64_t strides[1] = {(cuuint64_t)(ldc * ob)};
    cuuint32_t box[2] = {(cuuint32_t)(128 / ob), 128};
    cuuint32_t estr[2] = {1, 1};
    const CUtensorMapDataType dt = out_dtype == TW_F32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : out_dtype == TW_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                          : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
    CUresult r = enc(&a.tmap_out, dt, 2, ct, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(TW_ERR_CUDA, "cuTensorMapEncodeTiled (output) failed: " + std::to_string((int)r));
    a.tma_out = 1;
  }
  if (sched->grid <= kParamCtas) {
    a.cta_par = 1;
    for (size_t i = 0; i < sched->h_off.size() && i <= (size_t)kParamCtas; ++i) a.cta_off[0][i] = sched->h_off[i];
    for (size_t i = 0; i < sched->h_soff.size() && i <= (size_t)kParamCtas; ++i) a.cta_off[1][i] = sched->h_soff[i];
    for (size_t i = 0; i < sched->h_zoff.size() && i <= (size_t)kParamCtas; ++i) a.cta_off[2][i] = sched->h_zoff[i];
  }
  a.trace = trace;
  a.bias = bias;
  a.relu = relu;
  a.n_peer = n_peer;
  for (int d = 0; d < n_peer; ++d) a.peer[d] = peers[d];
  static const int zero_policy = [] {
    const char *e = std::getenv("TW_B200_ZERO");
    return e ? std::atoi(e) : 0;
  }();
  a.zero_policy = zero_policy;
  if (trace) {  // experiment knobs only honoured on the profiling entry point
    const char *dbg = std::getenv("TW_B200_DEBUG");
    a.debug = dbg ? std::atoi(dbg) : 0;
  }
  const int grid = sched->grid;
  cudaError_t e = sched->pair ? launch_tw_pair_sm100(a, out_dtype, grid, reinterpret_cast<cudaStream_t>(stream))
                              : launch_tw_gemm_sm100(a, out_dtype, grid, sched->tb, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tw_gemm launch");
  return TW_OK;
}

int tw_plan_kernel(const tw_plan *p, int64_t m, int out_dtype, int *kernel) {
  clear_error();
  if (!p || !kernel) return fail(TW_ERR_ARG, "null argument");
  if (p->device < 0) return fail(TW_ERR_ARG, "host-only plan");
  DeviceGuard guard(p->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice(plan device)");
  const int ob = out_size(out_dtype);
  static const bool pair_env = [] {
    const char *e = std::getenv("TW_B200_PAIR");
    return !(e && e[0] == '0');
  }();
  *kernel = (pair_env && (m * ob) % 16 == 0 && pair_clusters_for(p, m, out_dtype) > 0) ? 4 : 2;
  return TW_OK;
}

int tw_gemm_exact(const tw_plan *p, const float *at, int64_t m, int64_t lda, float *ct, int64_t ldc, void *stream) {
  clear_error();
  if (!p) return fail(TW_ERR_ARG, "null plan");
  if (p->device < 0) return fail(TW_ERR_ARG, "host-only plan cannot run on the GPU");
  DeviceGuard guard(p->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice(plan device)");
  if (m < 0 || lda < m || ldc < m) return fail(TW_ERR_DIMENSION, "bad M / lda / ldc");
  if (p->host.flags & TW_PLAN_SPLIT3)
    return fail(TW_ERR_ARG, "tw_gemm_exact needs a plain plan (TW_PLAN_SPLIT3 plans hold 3 k_i rows per tile)");
  int sms = 0;
  int rc = require_sm100(&sms);
  if (rc) return rc;
  cudaError_t e = launch_exact(p, at, m, lda, ct, ldc, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tw_gemm_exact launch");
  return TW_OK;
}

int tw_prune_col_means(const double *scores, int64_t k, int64_t n, double *out, void *stream) {
  clear_error();
  if (!scores || !out) return fail(TW_ERR_ARG, "null pointer");
  if (k < 1 || n < 1) return fail(TW_ERR_DIMENSION, "bad score-map dims");
  int sms = 0;
  int rc = require_sm100(&sms);
  if (rc) return rc;
  cudaError_t e = launch_prune_means(scores, k, n, nullptr, nullptr, 0, out, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TW_OK : cuda_fail(e, "tw_prune_col_means launch");
}

int tw_prune_row_means(const double *scores, int64_t k, int64_t n, const int32_t *cols, const int64_t *off,
                       int64_t n_tiles, double *out, void *stream) {
  clear_error();
  if (!scores || !cols || !off || !out) return fail(TW_ERR_ARG, "null pointer");
  if (k < 1 || n < 1 || n_tiles < 0) return fail(TW_ERR_DIMENSION, "bad score-map dims");
  if (n_tiles == 0) return TW_OK;
  int sms = 0;
  int rc = require_sm100(&sms);
  if (rc) return rc;
  cudaError_t e = launch_prune_means(scores, k, n, cols, off, n_tiles, out, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? TW_OK : cuda_fail(e, "tw_prune_row_means launch");
}

int tw_prep_activations(const float *a, int64_t m, int64_t k, int layout, void *at, int64_t ldat, int out_dtype,
                        void *stream) {
  clear_error();
  if (m < 0 || k < 0) return fail(TW_ERR_DIMENSION, "negative dims");
  if (layout != TW_ROW_MAJOR && layout != TW_COL_MAJOR) return fail(TW_ERR_ARG, "bad layout");
  if (ldat < m) return fail(TW_ERR_DIMENSION, "ldat < M");
  if (m == 0 || k == 0) return TW_OK;
  int sms = 0;
  int rc = require_sm100(&sms);
  if (rc) return rc;
  cudaError_t e = launch_prep(a, m, k, layout, at, ldat, out_dtype, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tw_prep_activations launch");
  return TW_OK;
}

int tw_prep_activations_split(const float *a, int64_t m, int64_t k, int layout, void *at2, int64_t ldat,
                              void *stream) {
  clear_error();
  if (m < 0 || k < 0) return fail(TW_ERR_DIMENSION, "negative dims");
  if (layout != TW_ROW_MAJOR && layout != TW_COL_MAJOR) return fail(TW_ERR_ARG, "bad layout");
  if (ldat < m) return fail(TW_ERR_DIMENSION, "ldat < M");
  if (m == 0 || k == 0) return TW_OK;
  int sms = 0;
  int rc = require_sm100(&sms);
  if (rc) return rc;
  cudaError_t e = launch_prep_split(a, m, k, layout, at2, ldat, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tw_prep_activations_split launch");
  return TW_OK;
}

int tw_spmm_csc(const void *at, int at_dtype, int64_t k, int64_t m, int64_t lda, int64_t n, const int32_t *col_ptr,
                const int32_t *row_idx, const float *values, void *ct, int64_t ldc, int out_dtype, int accumulate,
                void *stream) {
  clear_error();
  if (m < 0 || n < 0 || lda < m || ldc < m) return fail(TW_ERR_DIMENSION, "bad M / N / lda / ldc");
  if (m == 0 || n == 0) return TW_OK;
  int sms = 0;
  int rc = require_sm100(&sms);
  if (rc) return rc;
  cudaError_t e = launch_spmm(at, at_dtype, m, k, lda, 0, n, col_ptr, row_idx, values, ct, ldc, out_dtype, accumulate,
                              reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tw_spmm_csc launch");
  return TW_OK;
}

int tw_gemm_tew(const tw_plan *p, const void *at, int64_t m, int64_t lda, const int32_t *col_ptr,
                const int32_t *row_idx, const float *values, int64_t nnz, void *ct, int64_t ldc, int out_dtype,
                void *stream) {
  clear_error();
  if (!p) return fail(TW_ERR_ARG, "null plan");
  if (p->device < 0) return fail(TW_ERR_ARG, "host-only plan cannot run on the GPU");
  if (nnz == 0) return tw_gemm(p, at, m, lda, ct, ldc, out_dtype, 0, stream);  // engine.py:194-195
  if (m == 0) return TW_OK;
  const HostPlan &hp = p->host;
  if (hp.col_end == hp.col_begin) return TW_OK;  // empty column range: nothing to write
  DeviceGuard guard(p->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "cudaSetDevice(plan device)");
  if (lda < m || ldc < m) return fail(TW_ERR_DIMENSION, "bad lda / ldc");
  int sms = 0;
  int rc = require_sm100(&sms);
  if (rc) return rc;
  // The TW kernel writes every row of the plan's column range (kept rows and
  // the zero rows of pruned columns); the SpMM then adds the overlay into
  // every row it touches (it covers pruned columns too, pruning.py:548-549):
  // C = TW + S, one fp32 addition of the two separately computed products as
  // in engine.py:197.  This order is the cheaper one: the accumulating pass
  // is the SpMM's (C4: 20 + 50 us) rather than the TW kernel's (42 + 34 us).
  if ((rc = tw_gemm(p, at, m, lda, ct, ldc, out_dtype, 0, stream))) return rc;
  cudaError_t e = launch_spmm(at, hp.in_dtype, m, hp.k, lda, hp.col_begin, hp.col_end - hp.col_begin, col_ptr, row_idx,
                              values, ct, ldc, out_dtype, 1, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "tw_gemm_tew spmm launch");
  return TW_OK;
}

}  // extern "C"
