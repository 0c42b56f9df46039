// Internal declarations shared by the host packer, the C-ABI layer and the
// CUDA launchers of libtw_b200.so.
#pragma once

#include <cstdint>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "tw_b200.h"

#include <cuda.h>          // CUtensorMap
#include <vector_types.h>  // int4

namespace tw {

// thread-local error message behind tw_last_error()
int fail(int code, const std::string &msg);
void clear_error();

// One live tile of a plan, in launch (LPT) order.  Mirrors a TileTask
// (engine.py:24-37): the kept-K index list is `kidx[kidx_off .. +nkb*64)`
// (padded with K), the output rows are `colids[col_off .. +n_i)` (re-based to
// the plan's column range), the weight image is `wimg + w_off` (nkb blocks of
// wrows x 128 B, pre-swizzled for the SW128 K-major UMMA operand).
struct TileMeta {
  int32_t kidx_off;
  int32_t col_off;
  int32_t n_i;
  int32_t k16;      // ceil(k_i / 16): MMA k-steps
  int64_t w_off;    // byte offset into the weight image
  int32_t nkb;      // ceil(k_i / 64): pipeline stages
  int32_t k_i;
};
static_assert(sizeof(TileMeta) == 32, "TileMeta layout");

struct HostPlan {
  int64_t k = 0, n = 0, g = 0;
  int64_t col_begin = 0, col_end = 0;
  int64_t n_tiles = 0;
  int in_dtype = TW_BF16;
  int flags = 0;       // TW_PLAN_* (tw_b200.h)
  int64_t a_rows = 0;  // rows of the A^T operand the kept lists index: K, or 2K for TW_PLAN_SPLIT3
  int block_n = 128;   // MMA N tile (<= 256)
  int wrows = 128;     // weight-image rows per k-block (multiple of 16, <= block_n)
  std::vector<TileMeta> tiles;        // live tiles, LPT order
  std::vector<int32_t> src_tile;      // reference tile index of each live tile
  std::vector<int32_t> kidx;          // padded kept-K lists
  std::vector<int32_t> colids;        // block_n entries per live tile (-1 padded)
  std::vector<int32_t> zero_rows;     // output rows written as zeros
  std::vector<uint8_t> wimg;          // swizzled 16-bit weight image
  std::vector<float> w32;             // TW_PLAN_F32_WEIGHTS: fp32 weights, per live tile nkb*64 x 128 (k-major)
  std::vector<int64_t> w32_off;       // per live tile offset into w32 (elements)
  int64_t kept_elems = 0, union_k = 0, sum_k = 0, sum_n = 0;
  int64_t kept_rows_live = 0;  // sum of the live tiles' own kept rows (before TW_PLAN_DENSE_PAD)
};

// Static work schedule of one launch shape (plan, M, output width): CTA c
// runs units[off[c] .. off[c+1]) in order -- each {live tile, first token,
// number of 64-token quarters, 0} -- and writes zero rows
// zero_rows[zoff[c] .. zoff[c+1]) in the gaps.  Built on the host by LPT
// over a byte-cost model (tw_schedule.cpp).
struct HostSchedule {
  int grid = 0;
  std::vector<int32_t> units;  // 4 ints per unit
  std::vector<int32_t> off;    // grid + 1
  std::vector<int32_t> zoff;   // grid + 1
  // Per-CTA stage streams: stage s of CTA c (s in [soff[c], soff[c+1])) is
  // one 64-k block of one unit: stream[68 s .. 68 s + 64) are its kept A^T
  // row indices (-1 = padding -> zero fill), stream[68 s + 64 .. + 68) the
  // record {weight-image byte offset, first token, quarters | k-steps << 4 |
  // MMA N << 8, unit-in-CTA | first-block << 16 | last-block << 17}.  The
  // kernel streams it into shared memory with TMA, so the producer's index
  // loads never wait behind its own gathers.
  std::vector<int32_t> stream;
  std::vector<int32_t> soff;   // grid + 1
  bool has_contig = false;     // some stage's 64 kept rows are consecutive (TMA tile loads, record bit 12)
  bool has_tma_rows = false;   // some unit's tile has 128 consecutive output rows (unit flag bit 1)
  bool pair = false;           // K4 (CTA-pair) schedule: off is per cluster, no stage stream
  int max_nq = 0;              // widest half (64-token quarters) of any unit
  // zero rows are scheduled as PIECES of zero_chunk tokens (zero_cpr pieces
  // per row; piece p = row zero_rows[p / zero_cpr], tokens from
  // (p % zero_cpr) * zero_chunk): a pruned column of a long layer (VGG conv1:
  // 6.4 MB per row) spreads over many CTAs instead of landing on one; zoff
  // counts pieces
  int32_t zero_cpr = 1;
  int32_t zero_chunk = 0;
  double makespan_ns = 0, mean_ns = 0;
};
int build_schedule(const HostPlan &hp, int64_t m, int out_bytes, bool zero_rows, int sms, int tb,
                   HostSchedule &s);
// K4 (CTA-pair kernel): every live tile keeps all K rows in order (a dense
// pattern or TW_PLAN_DENSE_PAD) with weight blocks of at most 128 rows.
bool pair_eligible(const HostPlan &hp);
// K4 schedule: units {tile of CTA rank 0, tile of rank 1 (-1: none), first
// token, consecutive-rows flags (bit r: rank r's tile owns 128 consecutive
// C^T rows)} of 256 tokens, dealt round-robin to `clusters` CTA pairs
// (off: clusters + 1); zero rows split evenly over the 2 * clusters CTAs.
int build_pair_schedule(const HostPlan &hp, int64_t m, int ob, bool zero_rows, int clusters, HostSchedule &s);

constexpr int kParamCtas = 160;

// Kernel arguments of the persistent TW-GEMM (tw_gemm_sm100.cu).
struct GemmArgs {
  const TileMeta *tiles;
  const int32_t *kidx;
  const int32_t *colids;
  const int32_t *zero_rows;
  int32_t zero_cpr;    // zero-row pieces per row (HostSchedule::zero_cpr)
  int32_t zero_chunk;  // tokens per zero-row piece
  const uint8_t *wimg;
  const int4 *sched;         // per-CTA unit lists (HostSchedule::units)
  const int32_t *sched_off;  // grid + 1
  const int32_t *zero_off;   // grid + 1
  const int32_t *stream;     // HostSchedule::stream
  const int32_t *stream_off; // grid + 1
  void *out;
  int64_t ldc;
  const void *at;     // A^T (K x M, 16-bit), row stride lda
  int64_t lda;
  int32_t M;
  int32_t accumulate;
  int32_t wbytes;     // weight-image bytes per k-block (wrows * 128)
  uint32_t idesc;     // instruction descriptor without the N field
  int32_t block_n;
  int64_t *trace;     // optional per-CTA event timeline (tw_gemm_traced), else null
  const float *bias;  // optional per-output-row bias (fp32, row-rebased), fused epilogue
  int32_t relu;       // 1: max(x, 0) after the bias (trainer.py:246-248)
  int32_t keep_pruned;  // 1: pruned-column rows are left untouched (resident output)
  int32_t zero_policy; // when the epilogue writes zero rows (kernel comment); env TW_B200_ZERO
  int32_t n_peer;      // replicas of the output on other GPUs (tw_gemm_peers): every store goes to all
  void *peer[7];       //   of them too (NVLink peer / IPC-mapped pointers, same layout and ldc)
  int32_t no_pdl;     // 1: launch without programmatic stream serialization (TW_GEMM_NO_PDL)
  CUtensorMap tmap_at; // A^T (a_rows x M, 16-bit) for the stages whose 64 kept rows are consecutive
                       // (schedule has_contig): box 64 tokens x 64 rows, 128B swizzle
  CUtensorMap tmap_out; // C^T (M x output rows) for the epilogue's 2-D TMA tensor stores of tiles
                        // whose 128 output rows are consecutive (unit flag bit 1): box 128 B x 128 rows,
                        // 128B swizzle; valid when tma_out != 0
  int32_t tma_out;
  CUtensorMap tmap_w;  // K4: the weight image as 2-D (128-byte rows), box 128 B x 128 rows, no swizzle
  // per-CTA schedule offsets as kernel parameters (cta_par = 1, grids of up
  // to kParamCtas CTAs): {sched_off, stream_off, zero_off}[i] without a
  // dependent global load at CTA start (one DRAM round trip less before the
  // first gather / weight load)
  int32_t cta_par;
  int32_t cta_off[3][kParamCtas + 1];
  int32_t debug;      // experiment knobs (TW_B200_DEBUG): bit0 skip zero rows, bit1 skip kept-row stores
};

int build_host_plan(int64_t k, int64_t n, int64_t g, int64_t n_tiles, const int64_t *col_off,
                    const int32_t *col_ids, const uint32_t *row_mask_words, const float *subs,
                    const int64_t *sub_off, int in_dtype, int64_t col_begin, int64_t col_end,
                    HostPlan &hp, int flags = 0);

uint16_t f32_to_bf16_rne(float f);
uint16_t f32_to_f16_rne(float f);

}  // namespace tw

// Device copy of a schedule, cached per launch shape inside the plan.
struct tw_dev_schedule {
  int grid = 0;
  bool has_contig = false;
  bool has_tma_rows = false;
  bool pair = false;  // K4 schedule (grid = 2 x clusters)
  int32_t zero_cpr = 1, zero_chunk = 0;  // zero-row pieces (HostSchedule)
  int tb = 256;       // K2 unit width the launch instantiates (64 / 128 / 256 tokens)
  std::vector<int32_t> h_off, h_soff, h_zoff;  // host copies (kernel-parameter offsets)
  int4 *units = nullptr;
  int32_t *off = nullptr;
  int32_t *zoff = nullptr;
  int32_t *stream = nullptr;
  int32_t *soff = nullptr;
};

// Device side of a plan (defined in tw_capi.cu).
struct tw_plan {
  tw::HostPlan host;
  int device = 0;
  tw::TileMeta *d_tiles = nullptr;
  int32_t *d_kidx = nullptr;
  int32_t *d_colids = nullptr;
  int32_t *d_zero = nullptr;
  uint8_t *d_wimg = nullptr;
  float *d_w32 = nullptr;        // TW_PLAN_F32_WEIGHTS
  int64_t *d_w32_off = nullptr;
  bool pair_ok = false;          // K4-eligible (pair_eligible)
  mutable std::mutex sched_mu;
  mutable std::map<std::tuple<int64_t, int, int>, tw_dev_schedule> sched;  // (M, out bytes, zero rows on)
};
