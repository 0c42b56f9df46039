// Host-side static scheduler for the persistent TW-GEMM launch.
//
// Replaces the reference's shape-grouping + LPT worker assignment
// (engine.py:72-81 group_by_shape, :109-114 longest-processing-time bins)
// at a finer grain: the work items are (live tile, token block) units, the
// "workers" are the persistent CTAs, and the zero columns of C (pruned
// output columns, written as zero rows of C^T) are a divisible filler used to
// level the per-CTA output bytes -- on B200 the dense output write is the
// roofline of this kernel at high sparsity, so every CTA should
// write the same number of bytes.
//
// Piece cost model (ns per CTA-SM, calibrated on B200 with tools/membench*.cu):
// output bytes at ~30 B/ns per SM (4.5 TB/s DRAM write over 148 SMs), gathered
// input bytes at ~90 B/ns (L2 -> SM), MMA at 8192 flop/clk, plus a fixed
// pipeline fill and a per-stage producer overhead.  Every tile's token range
// is cut into equal pieces of at most P quarters for P = 1 .. 2 TB/64; the P
// whose LPT makespan is shortest wins (wave quantization vs weight re-reads).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <numeric>
#include <climits>
#include <queue>

#include "tw_internal.h"

namespace tw {

namespace {

// A piece = (live tile, first token, nq 64-token quarters).  Pieces of up to
// TB tokens are one accumulator "half"; longer pieces (up to 2 TB) are two
// halves sharing every weight block: the stage stream interleaves them per
// 64-k block (h0, h1, h0, h1, ...), the h1 stage reads the weight block the
// h0 stage loaded, so the tile's weights cross L2 -> SM once per 2 TB tokens.
struct Unit {
  int32_t tile, m0, nq;
  double cost;
};

constexpr double kWriteBps = 30.0;   // bytes / ns / SM
constexpr double kReadBps = 90.0;    // bytes / ns / SM
constexpr double kMmaFlops = 15000;  // flop / ns / SM (8192 flop/clk at ~1.85 GHz)
constexpr double kFixedNs = 300.0;
constexpr double kStageNs = 150.0;   // per-stage producer overhead (index loads, barriers)

double unit_cost(const TileMeta &t, int nq, int ob, int tb) {
  const double toks = 64.0 * nq;
  const double out_b = toks * t.n_i * ob;
  const double in_b = (double)t.k_i * (toks * 2.0 + t.n_i * 2.0);  // weights once per piece
  const double mma = 2.0 * toks * ((t.n_i + 15) / 16 * 16) * (t.k16 * 16.0) / kMmaFlops;
  const int halves = nq * 64 > tb ? 2 : 1;
  return std::max(std::max(out_b / kWriteBps, in_b / kReadBps), mma) + kFixedNs + kStageNs * t.nkb * halves;
}

// LPT: units (already sorted by cost, descending) to G workers; returns loads.
std::vector<double> lpt(const std::vector<Unit> &units, int G, std::vector<int> *owner) {
  std::vector<double> load((size_t)G, 0.0);
  using E = std::pair<double, int>;
  std::priority_queue<E, std::vector<E>, std::greater<E>> heap;
  for (int c = 0; c < G; ++c) heap.push({0.0, c});
  if (owner) owner->assign(units.size(), 0);
  for (size_t i = 0; i < units.size(); ++i) {
    E top = heap.top();
    heap.pop();
    top.first += units[i].cost;
    load[(size_t)top.second] = top.first;
    if (owner) (*owner)[i] = top.second;
    heap.push(top);
  }
  return load;
}

// Water-fill `rows` zero rows of cost zc each over the loads; returns per-CTA
// row counts and the resulting makespan.
std::vector<int64_t> water_fill(const std::vector<double> &load, int64_t rows, double zc, double *makespan) {
  const int G = (int)load.size();
  std::vector<int64_t> z((size_t)G, 0);
  double mk = *std::max_element(load.begin(), load.end());
  if (rows > 0 && zc > 0) {
    std::vector<double> s(load);
    std::sort(s.begin(), s.end());
    // find level L with sum_c max(0, L - load_c) / zc = rows
    double level = s.back();
    double pref = 0;
    for (int i = 0; i < G; ++i) {
      pref += s[(size_t)i];
      const double cand = (rows * zc + pref) / (i + 1);
      if (i + 1 == G || cand <= s[(size_t)i + 1]) {
        level = cand;
        break;
      }
    }
    int64_t used = 0;
    std::vector<std::pair<double, int>> frac;
    for (int c = 0; c < G; ++c) {
      const double want = std::max(0.0, (level - load[(size_t)c]) / zc);
      z[(size_t)c] = (int64_t)std::floor(want);
      used += z[(size_t)c];
      frac.push_back({want - std::floor(want), c});
    }
    std::sort(frac.begin(), frac.end(), [](auto &a, auto &b) { return a.first > b.first; });
    for (size_t i = 0; used < rows; i = (i + 1) % frac.size()) {
      ++z[(size_t)frac[i].second];
      ++used;
    }
    mk = 0;
    for (int c = 0; c < G; ++c) mk = std::max(mk, load[(size_t)c] + z[(size_t)c] * zc);
  }
  *makespan = mk;
  return z;
}

// Zero-row pieces: rows of more than kZeroPieceBytes are cut into pieces of
// equal token ranges (multiples of 64 tokens) so the water-fill can spread
// one long row over many CTAs.  Sets s.zero_cpr / s.zero_chunk; returns the
// number of pieces.
constexpr int64_t kZeroPieceBytes = 256 << 10;

int64_t zero_pieces(int64_t rows, int64_t m, int ob, HostSchedule &s) {
  int64_t cpr = std::max<int64_t>(1, (m * ob + kZeroPieceBytes - 1) / kZeroPieceBytes);
  int64_t chunk = (m + cpr - 1) / cpr;
  chunk = (chunk + 63) / 64 * 64;
  cpr = std::max<int64_t>(1, (m + chunk - 1) / chunk);
  while (cpr > 1 && rows * cpr > INT32_MAX / 2) {  // (huge layers) coarser pieces
    chunk *= 2;
    cpr = (m + chunk - 1) / chunk;
  }
  s.zero_cpr = (int32_t)cpr;
  s.zero_chunk = (int32_t)std::min<int64_t>(chunk, INT32_MAX);
  return rows * cpr;
}

}  // namespace

int build_schedule(const HostPlan &hp, int64_t m, int ob, bool zero_rows, int sms, int tb, HostSchedule &s) {
  s = HostSchedule{};
  const int64_t Z = zero_pieces(zero_rows ? (int64_t)hp.zero_rows.size() : 0, m, ob, s);
  const double zc = (double)std::min<int64_t>(m, s.zero_chunk) * ob / kWriteBps;
  const int qmax = 2 * tb / 64;  // quarters per piece (two halves of tb tokens)
  const int64_t q_tile = (m + 63) / 64;
  auto by_cost = [](const Unit &a, const Unit &b) {
    return a.cost != b.cost ? a.cost > b.cost : (a.tile != b.tile ? a.tile < b.tile : a.m0 < b.m0);
  };
  // pieces of at most P quarters: every tile's quarter range cut into
  // ceil(q / P) nearly equal contiguous pieces
  auto pieces = [&](int P) {
    std::vector<Unit> u;
    for (int32_t t = 0; t < (int32_t)hp.tiles.size(); ++t) {
      const int64_t np = (q_tile + P - 1) / P;
      int64_t q0 = 0;
      for (int64_t i = 0; i < np; ++i) {
        const int64_t q1 = (q_tile * (i + 1)) / np;
        const int nq = (int)(q1 - q0);
        if (nq > 0) u.push_back({t, (int32_t)(q0 * 64), nq, unit_cost(hp.tiles[(size_t)t], nq, ob, tb)});
        q0 = q1;
      }
    }
    std::stable_sort(u.begin(), u.end(), by_cost);
    return u;
  };
  const int64_t zero_ctas = Z > 0 ? (Z * std::min<int64_t>(m, s.zero_chunk) * ob + (256 << 10) - 1) / (256 << 10) : 0;
  // CTAs: enough for every piece of one quarter, so small layers (fewer
  // pieces than SMs) can spread over more SMs
  const int64_t quarters = q_tile * (int64_t)hp.tiles.size();
  int G = (int)std::min<int64_t>(sms, std::max<int64_t>({quarters, zero_ctas, (int64_t)1}));
  // Candidates: whole units of tb tokens; the tail past the last full wave,
  // or everything, split into pieces of P < tb/64 quarters; and (opt-in,
  // TW_B200_PAIRS=1) two-half pieces sharing weight blocks.  Measured on
  // B200: two-half pieces lose (C2a 12.5 -> 15.7 us) -- both TMEM regions
  // stay live to the end of a piece, so its epilogue no longer overlaps the
  // next piece's mainloop -- so they are off by default.
  static const bool pairs = [] {
    const char *e = std::getenv("TW_B200_PAIRS");
    return e && e[0] == '1';
  }();
  // (experiment) TW_B200_MAXQ = widest piece in 64-token quarters
  static const int maxq = [] {
    const char *e = std::getenv("TW_B200_MAXQ");
    return e ? std::atoi(e) : 0;
  }();
  const int qh = maxq > 0 ? std::min(tb / 64, maxq) : tb / 64;
  std::vector<std::vector<Unit>> cands{pieces(qh)};
  const std::vector<Unit> base = cands[0];  // a copy: cands grows below
  auto split_tail = [&](size_t from, int P) {
    std::vector<Unit> u(base.begin(), base.begin() + (std::ptrdiff_t)from);
    for (size_t i = from; i < base.size(); ++i) {
      const Unit &b = base[i];
      for (int q = 0; q < b.nq; q += P) {
        const int nq = std::min(P, b.nq - q);
        u.push_back({b.tile, b.m0 + 64 * q, nq, unit_cost(hp.tiles[(size_t)b.tile], nq, ob, tb)});
      }
    }
    std::stable_sort(u.begin(), u.end(), by_cost);
    return u;
  };
  const size_t full = base.size() / (size_t)G * (size_t)G;
  for (int P = 1; P < qh; ++P) {
    if (full < base.size() && full > 0) cands.push_back(split_tail(full, P));
    cands.push_back(pieces(P));
  }
  if (pairs)
    for (int P = qh + 1; P <= qmax; ++P) cands.push_back(pieces(P));
  // Pick the candidate with the shortest piece-only makespan (a CTA's pieces
  // run back to back and their outputs cannot be written before their MMA
  // completes); the zero rows are then water-filled around it.
  double best = 1e300, best_total = 0;
  size_t best_i = 0;
  std::vector<int> best_owner;
  std::vector<int64_t> best_z;
  for (size_t ci = 0; ci < cands.size(); ++ci) {
    if (cands[ci].empty() && ci > 0) continue;
    std::vector<int> owner;
    std::vector<double> load = lpt(cands[ci], G, &owner);
    const double unit_mk = *std::max_element(load.begin(), load.end());
    double mk = 0;
    std::vector<int64_t> z = water_fill(load, Z, zc, &mk);
    if (unit_mk < best * 0.99 || (unit_mk < best * 1.01 && mk < best_total)) {
      best = unit_mk;
      best_total = mk;
      best_i = ci;
      best_owner = owner;
      best_z = z;
    }
  }
  const std::vector<Unit> &units = cands[best_i];
  // per-CTA piece lists (pieces keep their global cost order within a CTA:
  // the smallest last, for the shortest epilogue tail)
  std::vector<std::vector<int>> per((size_t)G);
  for (size_t i = 0; i < units.size(); ++i) per[(size_t)best_owner[i]].push_back((int)i);
  s.grid = G;
  s.off.assign((size_t)G + 1, 0);
  s.zoff.assign((size_t)G + 1, 0);
  s.soff.assign((size_t)G + 1, 0);
  const int64_t wbytes = (int64_t)hp.wrows * 128;
  double total = 0;
  int64_t n_stages = 0;
  for (int c = 0; c < G; ++c) {
    int half_no = 0;  // accumulator region of a half = its ordinal in the CTA, mod 2
    for (int i : per[(size_t)c]) {
      const Unit &u = units[(size_t)i];
      total += u.cost;
      const TileMeta &t = hp.tiles[(size_t)u.tile];
      const bool pair = u.nq > qh;
      const int nh = pair ? 2 : 1;
      int hq[2] = {pair ? qh : u.nq, pair ? u.nq - qh : 0};
      int hm0[2] = {u.m0, u.m0 + qh * 64};
      int reg[2] = {half_no & 1, (half_no + 1) & 1};
      // epilogue units: one per half, in completion order; flag bit 1: the
      // tile's 128 output rows are consecutive C^T rows, so the epilogue
      // stores the unit with 2-D TMA tensor stores (4 boxes per 256 tokens)
      // instead of one bulk copy per row piece
      bool rows_consecutive = t.n_i == 128 && hp.block_n == 128;
      for (int r = 1; r < t.n_i && rows_consecutive; ++r)
        rows_consecutive = hp.colids[(size_t)t.col_off + r] == hp.colids[(size_t)t.col_off] + r;
      for (int h = 0; h < nh; ++h) {
        s.units.insert(s.units.end(), {u.tile, hm0[h], hq[h], reg[h] | (rows_consecutive ? 2 : 0)});
        s.max_nq = std::max(s.max_nq, hq[h]);
      }
      s.has_tma_rows = s.has_tma_rows || rows_consecutive;
      for (int kb = 0; kb < t.nkb; ++kb) {
        const int64_t woff = t.w_off + kb * wbytes;
        if (woff > INT32_MAX) return fail(TW_ERR_UNSUPPORTED, "weight image larger than 2 GiB");
        const int32_t nk = std::min(4, t.k16 - kb * 4);
        // a stage whose 64 kept rows are consecutive A^T rows (dense tiles:
        // gemm_dense, 0 % sparsity) is loaded by TMA 2-D tile copies
        // instead of row gathers: record bit 12
        const int32_t *kx = &hp.kidx[(size_t)t.kidx_off + (size_t)kb * 64];
        bool contig = kb * 64 + 63 < t.k_i && kx[0] >= 0 && kx[0] + 63 < hp.a_rows;
        for (int r = 1; r < 64 && contig; ++r) contig = kx[r] == kx[0] + r;
        s.has_contig = s.has_contig || contig;
        for (int h = 0; h < nh; ++h) {
          for (int r = 0; r < 64; ++r) {
            const int32_t idx = kx[r];
            s.stream.push_back(kb * 64 + r < t.k_i && idx < hp.a_rows ? idx : -1);
          }
          // record: {weight block offset (-1: reuse the previous stage's),
          //          first token, quarters | k-steps << 4 | region << 8 |
          //          W from the previous stage << 9 | defer the slot release << 10 |
          //          consecutive rows (TMA tile loads) << 12,
          //          half ordinal (tracing, 16 bits) | first << 16 | last << 17}
          const int32_t flags = hq[h] | (nk << 4) | (reg[h] << 8) | (h == 1 ? 1 << 9 : 0) |
                                (pair && h == 0 ? 1 << 10 : 0) | (contig ? 1 << 12 : 0);
          s.stream.insert(s.stream.end(),
                          {h == 0 ? (int32_t)woff : -1, hm0[h], flags,
                           ((half_no + h) & 0xffff) | (kb == 0 ? 1 << 16 : 0) | (kb == t.nkb - 1 ? 1 << 17 : 0)});
          ++n_stages;
        }
      }
      half_no += nh;
    }
    s.off[(size_t)c + 1] = (int32_t)(s.units.size() / 4);
    s.zoff[(size_t)c + 1] = (int32_t)(s.zoff[(size_t)c] + (best_z.empty() ? 0 : best_z[(size_t)c]));
    if (n_stages > INT32_MAX / 68) return fail(TW_ERR_UNSUPPORTED, "schedule too long");
    s.soff[(size_t)c + 1] = (int32_t)n_stages;
  }
  if (s.zoff[(size_t)G] != Z) return fail(TW_ERR_ARG, "internal: zero-row schedule does not cover the zero list");
  s.makespan_ns = best_total;
  s.mean_ns = (total + Z * zc) / G;
  return TW_OK;
}

bool pair_eligible(const HostPlan &hp) {
  // (weight blocks of wrows <= 128 rows: a shard's or a narrow layer's tiles;
  // the A operand rows past wrows are never stored)
  if (hp.tiles.empty() || (hp.flags & TW_PLAN_SPLIT3) || hp.block_n != 128 || hp.wrows > 128) return false;
  for (const TileMeta &t : hp.tiles) {
    if (t.k_i != hp.k) return false;
    const int32_t *kx = &hp.kidx[(size_t)t.kidx_off];
    for (int64_t r = 0; r < hp.k; ++r)
      if (kx[r] != (int32_t)r) return false;
  }
  return true;
}

int build_pair_schedule(const HostPlan &hp, int64_t m, int ob, bool zero_rows, int clusters, HostSchedule &s) {
  s = HostSchedule{};
  const int L = (int)hp.tiles.size();
  const int P = (L + 1) / 2;
  const int64_t nb = (m + 255) / 256;
  auto consecutive = [&](int t) {
    if (t < 0) return false;
    const TileMeta &tm = hp.tiles[(size_t)t];
    if (tm.n_i != 128) return false;
    for (int r = 1; r < 128; ++r)
      if (hp.colids[(size_t)tm.col_off + r] != hp.colids[(size_t)tm.col_off] + r) return false;
    return true;
  };
  std::vector<int32_t> flags((size_t)P);
  for (int p = 0; p < P; ++p) {
    const int t1 = 2 * p + 1 < L ? 2 * p + 1 : -1;
    flags[(size_t)p] = (consecutive(2 * p) ? 1 : 0) | (consecutive(t1) ? 2 : 0);
    s.has_tma_rows = s.has_tma_rows || flags[(size_t)p] != 0;
  }
  const int64_t n_units = nb * P;
  if (n_units > INT32_MAX / 4) return fail(TW_ERR_UNSUPPORTED, "schedule too long");
  const int C = (int)std::max<int64_t>(1, std::min<int64_t>(clusters, n_units));
  // token-block-major order dealt round-robin: pairs running at the same
  // time share their A^T token block in L2
  std::vector<std::vector<int32_t>> per((size_t)C);
  for (int64_t i = 0; i < n_units; ++i) {
    const int64_t b = i / P, p = i % P;
    const int t1 = 2 * (int)p + 1 < L ? 2 * (int)p + 1 : -1;
    auto &v = per[(size_t)(i % C)];
    v.insert(v.end(), {2 * (int32_t)p, t1, (int32_t)(b * 256), flags[(size_t)p]});
  }
  s.grid = 2 * C;
  s.pair = true;
  s.off.assign((size_t)C + 1, 0);
  for (int c = 0; c < C; ++c) {
    s.units.insert(s.units.end(), per[(size_t)c].begin(), per[(size_t)c].end());
    s.off[(size_t)c + 1] = (int32_t)(s.units.size() / 4);
  }
  const int64_t Z = zero_pieces(zero_rows ? (int64_t)hp.zero_rows.size() : 0, m, ob, s);
  s.zoff.assign((size_t)s.grid + 1, 0);
  for (int c = 0; c < s.grid; ++c) s.zoff[(size_t)c + 1] = (int32_t)(Z * (c + 1) / s.grid);
  s.soff.assign((size_t)s.grid + 1, 0);
  return TW_OK;
}

}  // namespace tw
