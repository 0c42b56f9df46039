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
// Unit cost model (ns per CTA-SM, calibrated on B200 with tools/membench*.cu):
// output bytes at ~30 B/ns per SM (4.5 TB/s DRAM write over 148 SMs), gathered
// input bytes at ~90 B/ns (L2 -> SM), MMA at 8192 flop/clk, plus a fixed
// pipeline fill.  Tail units of 256 tokens may be split into two 128-token
// units when that shortens the makespan (wave quantization).
#include <algorithm>
#include <cmath>
#include <functional>
#include <numeric>
#include <climits>
#include <queue>

#include "tw_internal.h"

namespace tw {

namespace {

// nq = the unit's tokens in 64-token quarters (1..4; 1..2 for G = 256)
struct Unit {
  int32_t tile, m0, nq;
  double cost;
};

constexpr double kWriteBps = 30.0;   // bytes / ns / SM
constexpr double kReadBps = 90.0;    // bytes / ns / SM
constexpr double kMmaFlops = 15000;  // flop / ns / SM (8192 flop/clk at ~1.85 GHz)
constexpr double kFixedNs = 300.0;

double unit_cost(const TileMeta &t, int nq, int ob) {
  const double toks = 64.0 * nq;
  const double out_b = toks * t.n_i * ob;
  const double in_b = (double)t.k_i * (toks * 2.0 + t.n_i * 2.0);
  const double mma = 2.0 * toks * ((t.n_i + 15) / 16 * 16) * (t.k16 * 16.0) / kMmaFlops;
  return std::max(std::max(out_b / kWriteBps, in_b / kReadBps), mma) + kFixedNs;
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

}  // namespace

int build_schedule(const HostPlan &hp, int64_t m, int ob, bool zero_rows, int sms, int tb, HostSchedule &s) {
  s = HostSchedule{};
  const int64_t Z = zero_rows ? (int64_t)hp.zero_rows.size() : 0;
  const double zc = (double)m * ob / kWriteBps;
  std::vector<Unit> base;
  for (int32_t t = 0; t < (int32_t)hp.tiles.size(); ++t) {
    for (int64_t m0 = 0; m0 < m; m0 += tb) {
      const int nq = (int)std::min<int64_t>(tb / 64, (m - m0 + 63) / 64);
      base.push_back({t, (int32_t)m0, nq, unit_cost(hp.tiles[(size_t)t], nq, ob)});
    }
  }
  const int64_t zero_ctas = Z > 0 ? (Z * m * ob + (256 << 10) - 1) / (256 << 10) : 0;
  // CTAs: enough for every unit -- or every 64-token quarter, so small
  // layers (fewer 256-token units than SMs) can spread over more SMs
  int64_t quarters = 0;
  for (const Unit &u : base) quarters += u.nq;
  int G = (int)std::min<int64_t>(sms, std::max<int64_t>({quarters, zero_ctas, (int64_t)1}));
  auto by_cost = [](const Unit &a, const Unit &b) {
    return a.cost != b.cost ? a.cost > b.cost : (a.tile != b.tile ? a.tile < b.tile : a.m0 < b.m0);
  };
  std::stable_sort(base.begin(), base.end(), by_cost);

  // Candidate unit sets: as is; the tail (units past the last whole wave)
  // or everything split into pieces of at most 2 quarters, or of 1 quarter.
  // A piece re-reads the tile's whole weight block, so smaller pieces only
  // win where they shorten the makespan -- the cost model decides.
  std::vector<std::vector<Unit>> cands{base};
  auto split = [&](const std::vector<Unit> &from_set, size_t from, int max_nq) {
    std::vector<Unit> u(from_set.begin(), from_set.begin() + (std::ptrdiff_t)from);
    for (size_t i = from; i < from_set.size(); ++i) {
      const Unit &b = from_set[i];
      const TileMeta &t = hp.tiles[(size_t)b.tile];
      for (int q = 0; q < b.nq; q += max_nq) {
        const int nq = std::min(max_nq, b.nq - q);
        u.push_back({b.tile, b.m0 + 64 * q, nq, unit_cost(t, nq, ob)});
      }
    }
    std::stable_sort(u.begin(), u.end(), by_cost);
    return u;
  };
  const size_t full = base.size() / (size_t)G * (size_t)G;
  for (int max_nq : {2, 1}) {
    if (max_nq >= tb / 64) continue;
    if (full < base.size() && full > 0) cands.push_back(split(base, full, max_nq));
    cands.push_back(split(base, 0, max_nq));
  }
  // Pick the candidate with the shortest unit-only makespan (a CTA's units
  // run back to back and their outputs cannot be written before their MMA
  // completes); the zero rows are then water-filled around it.
  double best = 1e300, best_total = 0;
  size_t best_i = 0;
  std::vector<int> best_owner;
  std::vector<int64_t> best_z;
  for (size_t ci = 0; ci < cands.size(); ++ci) {
    std::vector<int> owner;
    std::vector<double> load = lpt(cands[ci], G, &owner);
    const double unit_mk = *std::max_element(load.begin(), load.end());
    double mk = 0;
    std::vector<int64_t> z = water_fill(load, Z, zc, &mk);
    if (unit_mk < best * 0.98 || (unit_mk < best * 1.02 && mk < best_total)) {
      best = unit_mk;
      best_total = mk;
      best_i = ci;
      best_owner = owner;
      best_z = z;
    }
  }
  const std::vector<Unit> &units = cands[best_i];
  // emit per-CTA lists (units keep their global cost order within a CTA)
  std::vector<std::vector<int>> per((size_t)G);
  for (size_t i = 0; i < units.size(); ++i) per[(size_t)best_owner[i]].push_back((int)i);
  s.grid = G;
  s.off.assign((size_t)G + 1, 0);
  s.zoff.assign((size_t)G + 1, 0);
  double total = 0;
  for (int c = 0; c < G; ++c) {
    for (int i : per[(size_t)c]) {
      const Unit &u = units[(size_t)i];
      s.units.insert(s.units.end(), {u.tile, u.m0, u.nq, 0});
      total += u.cost;
    }
    s.off[(size_t)c + 1] = (int32_t)(s.units.size() / 4);
    s.zoff[(size_t)c + 1] = (int32_t)(s.zoff[(size_t)c] + (best_z.empty() ? 0 : best_z[(size_t)c]));
  }
  if (s.zoff[(size_t)G] != Z) return fail(TW_ERR_ARG, "internal: zero-row schedule does not cover the zero list");
  // per-CTA stage streams (see HostSchedule)
  const int64_t wbytes = (int64_t)hp.wrows * 128;
  s.soff.assign((size_t)G + 1, 0);
  int64_t n_stages = 0;
  for (int c = 0; c < G; ++c) {
    for (int32_t u = s.off[(size_t)c]; u < s.off[(size_t)c + 1]; ++u) {
      const int32_t *un = &s.units[(size_t)u * 4];
      const TileMeta &t = hp.tiles[(size_t)un[0]];
      const int32_t n_mma = (t.n_i + 15) & ~15;
      for (int kb = 0; kb < t.nkb; ++kb) {
        for (int r = 0; r < 64; ++r) {
          const int32_t idx = hp.kidx[(size_t)t.kidx_off + (size_t)kb * 64 + (size_t)r];
          s.stream.push_back(kb * 64 + r < t.k_i && idx < hp.a_rows ? idx : -1);
        }
        const int64_t woff = t.w_off + kb * wbytes;
        if (woff > INT32_MAX) return fail(TW_ERR_UNSUPPORTED, "weight image larger than 2 GiB");
        const int32_t nk = std::min(4, t.k16 - kb * 4);
        s.stream.insert(s.stream.end(),
                        {(int32_t)woff, un[1], un[2] | (nk << 4) | (n_mma << 8),
                         // unit ordinal (tracing only) masked to 16 bits: bits 16/17 are
                         // the first/last-block flags the MMA warp acts on
                         ((u - s.off[(size_t)c]) & 0xffff) | (kb == 0 ? 1 << 16 : 0) |
                             (kb == t.nkb - 1 ? 1 << 17 : 0)});
        ++n_stages;
      }
    }
    if (n_stages > INT32_MAX / 68) return fail(TW_ERR_UNSUPPORTED, "schedule too long");
    s.soff[(size_t)c + 1] = (int32_t)n_stages;
  }
  s.makespan_ns = best_total;
  s.mean_ns = (total + Z * zc) / G;
  return TW_OK;
}

}  // namespace tw
