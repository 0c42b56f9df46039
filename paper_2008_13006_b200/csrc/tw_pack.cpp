// Host-side metadata packer (north_star item 1): TW masks -> kept-K index
// lists, pruned-column lists, compacted weight tiles, and the packed plan
// image the persistent sm_100a kernel consumes.  Pure CPU code.
//
// Reference semantics restated here (reference = tilewise package):
//   pack/unpack/mask_words_to_indices   pattern.py:169-189
//   compact                             pattern.py:223-241
//   _pruned_columns_of                  pruning.py:257-258
//   _plan_tasks / group_by_shape order  engine.py:72-81, :126-149 (LPT by work)
#include <algorithm>
#include <cstring>
#include <numeric>

#include "tw_internal.h"

namespace tw {

namespace {
thread_local std::string g_err;
}

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}
void clear_error() { g_err.clear(); }

uint16_t f32_to_bf16_rne(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((u >> 16) | 0x40);  // quiet NaN
  uint32_t lsb = (u >> 16) & 1u;
  u += 0x7fffu + lsb;
  return (uint16_t)(u >> 16);
}

uint16_t f32_to_f16_rne(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t ax = x & 0x7fffffffu;
  if (ax > 0x7f800000u) return (uint16_t)(sign | 0x7e00u);
  if (ax >= 0x477ff000u) return (uint16_t)(sign | 0x7c00u);  // >= 65520 rounds to inf
  if (ax < 0x38800000u) {                                    // subnormal / zero in fp16
    if (ax < 0x33000000u) return (uint16_t)sign;             // < 2^-25 -> 0
    uint32_t e = ax >> 23;
    uint32_t mant = (ax & 0x7fffffu) | 0x800000u;
    uint32_t shift = 126 - e;  // 14..24
    uint32_t q = mant >> shift;
    uint32_t rem = mant & ((1u << shift) - 1);
    uint32_t half = 1u << (shift - 1);
    if (rem > half || (rem == half && (q & 1))) ++q;
    return (uint16_t)(sign | q);
  }
  uint32_t r = ax + 0xfffu + ((ax >> 13) & 1u);
  return (uint16_t)(sign | ((r - 0x38000000u) >> 13));
}

static inline bool bit_of(const uint32_t *words, int64_t i) { return (words[i >> 5] >> (i & 31)) & 1u; }

int build_host_plan(int64_t k, int64_t n, int64_t g, int64_t n_tiles, const int64_t *col_off,
                    const int32_t *col_ids, const uint32_t *row_mask_words, const float *subs,
                    const int64_t *sub_off, int in_dtype, int64_t col_begin, int64_t col_end,
                    HostPlan &hp, int flags) {
  if (k < 1 || n < 1 || g < 1) return fail(TW_ERR_DIMENSION, "bad pattern dims");
  if (flags & ~(TW_PLAN_SPLIT3 | TW_PLAN_F32_WEIGHTS | TW_PLAN_DENSE_PAD)) return fail(TW_ERR_ARG, "unknown plan flags");
  const bool split = (flags & TW_PLAN_SPLIT3) != 0;
  const bool pad = (flags & TW_PLAN_DENSE_PAD) != 0;
  if (pad && (flags & (TW_PLAN_SPLIT3 | TW_PLAN_F32_WEIGHTS)))
    return fail(TW_ERR_ARG, "TW_PLAN_DENSE_PAD does not combine with TW_PLAN_SPLIT3 / TW_PLAN_F32_WEIGHTS");
  if (split && in_dtype != TW_BF16) return fail(TW_ERR_ARG, "TW_PLAN_SPLIT3 needs TW_BF16 operands");
  if (g > 256) return fail(TW_ERR_UNSUPPORTED, "tile width G > 256 is not supported by the sm_100a kernel");
  if (in_dtype != TW_BF16 && in_dtype != TW_F16) return fail(TW_ERR_ARG, "in_dtype must be TW_BF16 or TW_F16");
  if (col_begin < 0 || col_end > n || col_begin > col_end) return fail(TW_ERR_DIMENSION, "bad column range");
  if (k > (int64_t)1 << 30 || n > (int64_t)1 << 30) return fail(TW_ERR_UNSUPPORTED, "K/N too large");
  const int64_t nwords = (k + 31) / 32;
  hp = HostPlan{};
  hp.k = k; hp.n = n; hp.g = g; hp.n_tiles = n_tiles; hp.in_dtype = in_dtype;
  hp.col_begin = col_begin; hp.col_end = col_end;
  hp.flags = flags;
  hp.a_rows = split ? 2 * k : k;
  hp.block_n = g <= 128 ? 128 : 256;

  struct Live { int32_t src; int64_t j0, j1; int64_t k_i; std::vector<int32_t> rows; };
  std::vector<Live> live;
  std::vector<uint8_t> covered((size_t)(col_end - col_begin), 0);
  std::vector<uint8_t> union_rows((size_t)k, 0);
  int max_n = 0;
  for (int64_t t = 0; t < n_tiles; ++t) {
    const int64_t c0 = col_off[t], c1 = col_off[t + 1];
    if (c1 < c0) return fail(TW_ERR_DIMENSION, "col_off must be nondecreasing");
    if (c1 - c0 > g) return fail(TW_ERR_DIMENSION, "tile wider than G");
    const uint32_t *w = row_mask_words + t * nwords;
    int64_t k_i = 0;
    for (int64_t i = 0; i < k; ++i) k_i += bit_of(w, i);
    if (sub_off[t + 1] - sub_off[t] != k_i * (c1 - c0))
      return fail(TW_ERR_DIMENSION, "sub-matrix size does not match k_i x n_i");
    // select this tile's columns inside [col_begin, col_end) (ascending ids)
    int64_t j0 = c1, j1 = c0;
    for (int64_t j = c0; j < c1; ++j) {
      int32_t c = col_ids[j];
      if (c < 0 || c >= n) return fail(TW_ERR_DIMENSION, "column id out of range");
      if (j > c0 && col_ids[j] <= col_ids[j - 1]) return fail(TW_ERR_DIMENSION, "col_ids must be strictly ascending");
      if (c >= col_begin && c < col_end) { j0 = std::min(j0, j); j1 = std::max(j1, j + 1); }
    }
    if (j1 <= j0) continue;
    if (k_i == 0) continue;  // engine.py:134-135: output columns stay zero
    Live L{(int32_t)t, j0 - c0, j1 - c0, k_i, {}};
    L.rows.reserve((size_t)k_i);
    for (int64_t i = 0; i < k; ++i)
      if (bit_of(w, i)) { L.rows.push_back((int32_t)i); union_rows[(size_t)i] = 1; }
    for (int64_t j = j0; j < j1; ++j) covered[(size_t)(col_ids[j] - col_begin)] = 1;
    max_n = std::max<int>(max_n, (int)(j1 - j0));
    live.push_back(std::move(L));
  }
  // kept elements over the whole range counts every tile (k_i = 0 adds 0)
  hp.wrows = std::max(16, (max_n + 15) / 16 * 16);
  if (hp.wrows > hp.block_n) return fail(TW_ERR_UNSUPPORTED, "tile wider than block_n");
  // LPT order: largest work first, ties by reference tile index (engine.py:80, :109-114)
  std::stable_sort(live.begin(), live.end(), [](const Live &a, const Live &b) {
    int64_t wa = a.k_i * (a.j1 - a.j0), wb = b.k_i * (b.j1 - b.j0);
    return wa != wb ? wa > wb : a.src < b.src;
  });
  for (int64_t i = 0; i < k; ++i) hp.union_k += union_rows[(size_t)i];
  if (split) hp.union_k *= 2;  // the high and the low rows of every kept k
  for (int64_t c = 0; c < col_end - col_begin; ++c)
    if (!covered[(size_t)c]) hp.zero_rows.push_back((int32_t)c);

  const int bytes_per_kb = hp.wrows * 128;
  // TW_PLAN_SPLIT3 (fp32-faithful tensor-core mode): with A = Ah + Al and
  // W = Wh + Wl split into bf16 high / low parts (x = rn(x), rn(x - rn(x))),
  // A.W ~= Ah.Wh + Al.Wh + Ah.Wl (the dropped Al.Wl is ~2^-18 relative).  The
  // three products are one TW GEMM over 3 k_i kept rows per tile: kept rows r
  // of A^T (= Ah) with Wh, rows r + K (= Al, the second half of the 2K-row
  // split operand tw_prep_activations_split writes) with Wh, rows r with Wl.
  const int reps = split ? 3 : 1;
  std::vector<int32_t> kpos;  // TW_PLAN_DENSE_PAD: row -> position in the tile's kept list, or -1
  for (const Live &L : live) {
    TileMeta m{};
    const int64_t n_i = L.j1 - L.j0;
    const int64_t kx = pad ? k : L.k_i * reps;  // kept rows as the kernel sees them
    if (pad) {
      kpos.assign((size_t)k, -1);
      for (size_t r = 0; r < L.rows.size(); ++r) kpos[(size_t)L.rows[r]] = (int32_t)r;
    }
    m.n_i = (int32_t)n_i;
    m.k_i = (int32_t)kx;
    m.k16 = (int32_t)((kx + 15) / 16);
    m.nkb = (int32_t)((kx + 63) / 64);
    m.kidx_off = (int32_t)hp.kidx.size();
    m.col_off = (int32_t)hp.colids.size();
    m.w_off = (int64_t)hp.wimg.size();
    for (int64_t r = 0; r < (int64_t)m.nkb * 64; ++r) {
      int32_t idx = (int32_t)hp.a_rows;  // pad: out-of-range row -> zeros
      if (r < kx) idx = pad ? (int32_t)r : L.rows[(size_t)(r % L.k_i)] + (r / L.k_i == 1 ? (int32_t)k : 0);
      hp.kidx.push_back(idx);
    }
    const int64_t c0 = col_off[L.src];
    for (int64_t j = 0; j < hp.block_n; ++j)
      hp.colids.push_back(j < n_i ? (int32_t)(col_ids[c0 + L.j0 + j] - col_begin) : -1);
    // weight image: for each 64-wide k block, wrows rows (one per output
    // column j) of 64 16-bit values, 16-byte chunk c of row j stored at
    // chunk (c ^ (j & 7)) -- the 128B-swizzle the UMMA K-major SW128
    // descriptor expects (CUTLASS Swizzle<3,4,3>).
    const float *sub = subs + sub_off[L.src];  // COL_MAJOR k_i x n_tile (pattern.py:233)
    const int64_t ktile = L.k_i;
    size_t base = hp.wimg.size();
    hp.wimg.resize(base + (size_t)m.nkb * bytes_per_kb, 0);
    uint8_t *img = hp.wimg.data() + base;
    for (int kb = 0; kb < m.nkb; ++kb) {
      uint8_t *blk = img + (size_t)kb * bytes_per_kb;
      for (int64_t j = 0; j < n_i; ++j) {
        const float *colv = sub + (L.j0 + j) * ktile;
        for (int c = 0; c < 8; ++c) {
          uint16_t *dst = (uint16_t *)(blk + j * 128 + ((c ^ (j & 7)) * 16));
          for (int e = 0; e < 8; ++e) {
            const int64_t kk = (int64_t)kb * 64 + c * 8 + e;
            if (kk >= kx || (pad && kpos[(size_t)kk] < 0)) { dst[e] = 0; continue; }
            const float v = colv[pad ? kpos[(size_t)kk] : kk % ktile];
            if (!split) {
              dst[e] = in_dtype == TW_BF16 ? f32_to_bf16_rne(v) : f32_to_f16_rne(v);
            } else {
              const uint16_t hi = f32_to_bf16_rne(v);
              if (kk < 2 * ktile) {
                dst[e] = hi;
              } else {  // low part: v - hi exactly representable in fp32
                const uint32_t hb = (uint32_t)hi << 16;
                float hv;
                std::memcpy(&hv, &hb, 4);
                dst[e] = f32_to_bf16_rne(v - hv);
              }
            }
          }
        }
      }
    }
    if (flags & TW_PLAN_F32_WEIGHTS) {  // the reference's own fp32 weights, for tw_gemm_exact
      hp.w32_off.push_back((int64_t)hp.w32.size());
      const int64_t rows32 = (ktile + 63) / 64 * 64;
      hp.w32.resize(hp.w32.size() + (size_t)(rows32 * 128), 0.0f);
      float *w = hp.w32.data() + hp.w32_off.back();
      for (int64_t kk = 0; kk < ktile; ++kk)
        for (int64_t j = 0; j < n_i; ++j) w[kk * 128 + j] = sub[(L.j0 + j) * ktile + kk];
    }
    hp.kept_rows_live += L.k_i;
    hp.kept_elems += L.k_i * n_i;  // the reference's kept elements (FLOP count), not the split's 3x
    hp.sum_k += kx;
    hp.sum_n += n_i;
    hp.tiles.push_back(m);
    hp.src_tile.push_back(L.src);
  }
  return TW_OK;
}

}  // namespace tw

using namespace tw;

extern "C" {

const char *tw_last_error(void) { return g_err.c_str(); }
int tw_version(void) { return 100; }

int tw_pack_mask_words(const uint8_t *keep, int64_t length, uint32_t *words) {
  if (length < 0 || (length > 0 && (!keep || !words))) return fail(TW_ERR_ARG, "null pointer");
  const int64_t nwords = (length + 31) / 32;
  std::memset(words, 0, sizeof(uint32_t) * (size_t)nwords);
  for (int64_t i = 0; i < length; ++i)
    if (keep[i]) words[i >> 5] |= 1u << (i & 31);
  return TW_OK;
}

int tw_unpack_mask_words(const uint32_t *words, int64_t nwords, int64_t length, uint8_t *keep) {
  if (nwords * 32 < length)
    return fail(TW_ERR_DIMENSION, "mask words cover " + std::to_string(nwords * 32) + " bits, need " +
                                      std::to_string(length));
  for (int64_t i = 0; i < length; ++i) keep[i] = bit_of(words, i) ? 1 : 0;
  return TW_OK;
}

int tw_mask_words_to_indices(const uint32_t *words, int64_t nwords, int64_t length, int64_t *idx,
                             int64_t *count) {
  if (nwords * 32 < length)
    return fail(TW_ERR_DIMENSION, "mask words cover " + std::to_string(nwords * 32) + " bits, need " +
                                      std::to_string(length));
  int64_t c = 0;
  for (int64_t i = 0; i < length; ++i)
    if (bit_of(words, i)) idx[c++] = i;
  *count = c;
  return TW_OK;
}

int tw_compact(const float *b, int64_t k, int64_t n, int layout, int64_t n_tiles, const int64_t *col_off,
               const int32_t *col_ids, const uint32_t *row_mask_words, float *subs, int64_t *sub_off) {
  if (k < 1 || n < 1) return fail(TW_ERR_DIMENSION, "bad matrix dims");
  if (layout != TW_ROW_MAJOR && layout != TW_COL_MAJOR) return fail(TW_ERR_ARG, "bad layout");
  const int64_t nwords = (k + 31) / 32;
  std::vector<int64_t> rows;
  sub_off[0] = 0;
  for (int64_t t = 0; t < n_tiles; ++t) {
    const uint32_t *w = row_mask_words + t * nwords;
    rows.clear();
    for (int64_t i = 0; i < k; ++i)
      if (bit_of(w, i)) rows.push_back(i);
    const int64_t k_i = (int64_t)rows.size();
    const int64_t c0 = col_off[t], c1 = col_off[t + 1];
    float *dst = subs + sub_off[t];
    for (int64_t j = c0; j < c1; ++j) {
      const int64_t c = col_ids[j];
      if (c < 0 || c >= n) return fail(TW_ERR_DIMENSION, "column id out of range");
      for (int64_t r = 0; r < k_i; ++r) {
        const int64_t i = rows[(size_t)r];
        dst[(j - c0) * k_i + r] = layout == TW_ROW_MAJOR ? b[i * n + c] : b[c * k + i];
      }
    }
    sub_off[t + 1] = sub_off[t] + k_i * (c1 - c0);
  }
  return TW_OK;
}

int tw_pruned_columns(int64_t n, int64_t n_tiles, const int64_t *col_off, const int32_t *col_ids,
                      int64_t *out, int64_t *count) {
  std::vector<uint8_t> seen((size_t)n, 0);
  for (int64_t j = 0; j < (n_tiles > 0 ? col_off[n_tiles] : 0); ++j) {
    if (col_ids[j] < 0 || col_ids[j] >= n) return fail(TW_ERR_DIMENSION, "column id out of range");
    seen[(size_t)col_ids[j]] = 1;
  }
  int64_t c = 0;
  for (int64_t i = 0; i < n; ++i)
    if (!seen[(size_t)i]) out[c++] = i;
  *count = c;
  return TW_OK;
}

int tw_plan_export(const tw_plan *plan, int which, void *dst, int64_t *bytes) {
  if (!plan || !bytes) return fail(TW_ERR_ARG, "null pointer");
  const HostPlan &hp = plan->host;
  std::vector<int64_t> table;
  const void *src = nullptr;
  int64_t size = 0;
  switch (which) {
    case 0: src = hp.kidx.data(); size = (int64_t)hp.kidx.size() * 4; break;
    case 1: src = hp.colids.data(); size = (int64_t)hp.colids.size() * 4; break;
    case 2: src = hp.zero_rows.data(); size = (int64_t)hp.zero_rows.size() * 4; break;
    case 3: src = hp.wimg.data(); size = (int64_t)hp.wimg.size(); break;
    case 4:
      for (size_t i = 0; i < hp.tiles.size(); ++i) {
        const TileMeta &m = hp.tiles[i];
        int64_t row[8] = {hp.src_tile[i], m.kidx_off, m.col_off, m.n_i, m.k_i, m.k16, m.nkb, m.w_off};
        table.insert(table.end(), row, row + 8);
      }
      src = table.data(); size = (int64_t)table.size() * 8;
      break;
    default: return fail(TW_ERR_ARG, "bad export selector");
  }
  if (!dst) { *bytes = size; return TW_OK; }
  if (*bytes < size) return fail(TW_ERR_ARG, "export buffer too small");
  if (size) std::memcpy(dst, src, (size_t)size);
  *bytes = size;
  return TW_OK;
}

int tw_schedule_export(const tw_plan *plan, int64_t m, int out_dtype, int accumulate, int sms, int which, void *dst,
                       int64_t *bytes) {
  if (!plan || !bytes) return fail(TW_ERR_ARG, "null pointer");
  if (m < 1 || sms < 1) return fail(TW_ERR_DIMENSION, "need M >= 1 and sms >= 1");
  const int tb = plan->host.block_n <= 128 ? 256 : 128;
  HostSchedule hs;
  int rc = build_schedule(plan->host, m, out_dtype == TW_F32 ? 4 : 2, !accumulate, sms, tb, hs);
  if (rc) return rc;
  const std::vector<int32_t> &v = which == 0 ? hs.units : (which == 1 ? hs.off : hs.zoff);
  if (which < 0 || which > 2) return fail(TW_ERR_ARG, "bad export selector");
  const int64_t size = (int64_t)v.size() * 4;
  if (!dst) { *bytes = size; return TW_OK; }
  if (*bytes < size) return fail(TW_ERR_ARG, "export buffer too small");
  if (size) std::memcpy(dst, v.data(), (size_t)size);
  *bytes = size;
  return TW_OK;
}

int tw_plan_get_info(const tw_plan *plan, tw_plan_info *info) {
  if (!plan || !info) return fail(TW_ERR_ARG, "null pointer");
  const HostPlan &hp = plan->host;
  info->k = hp.k; info->n = hp.n; info->g = hp.g;
  info->col_begin = hp.col_begin; info->col_end = hp.col_end;
  info->n_tiles = hp.n_tiles;
  info->n_live = (int64_t)hp.tiles.size();
  info->n_zero_rows = (int64_t)hp.zero_rows.size();
  info->kept_elems = hp.kept_elems;
  info->union_k = hp.union_k;
  info->sum_k = hp.sum_k;
  info->sum_n = hp.sum_n;
  info->block_n = hp.block_n;
  info->wimg_bytes = (int64_t)hp.wimg.size();
  info->in_dtype = hp.in_dtype;
  info->flags = hp.flags;
  info->a_rows = hp.a_rows;
  return TW_OK;
}

}  // extern "C"
