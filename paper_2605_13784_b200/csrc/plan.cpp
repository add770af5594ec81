// plan.cpp — split-KV work planner (host, integer only).
//
// Turns the segments of one call into CTA work units: for every segment,
// every q tile of `q_tile_tokens` tokens and every KV head, the key tiles
// (cached pool tiles, then the segment's own tiles up to the q tile's last
// token — causal, reading R-2) are split into contiguous ranges so that the
// launch fills the GPU (148 SMs on B200).  Units of one (segment, q tile, kv
// head) form a Group merged by the combine kernel (log-sum-exp, reading R-11).
#include <algorithm>
#include <functional>
#include <queue>
#include <tuple>
#include <cstdint>
#include <vector>

#include "plan.h"

namespace ssa {

static int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

void plan_units(const std::vector<SegDesc>& segs, const PlanConfig& c, Plan* out) {
  out->units.clear();
  out->groups.clear();
  struct Item { int seg, kvh, tok0, ntok; int64_t tiles, pool_tiles; };
  std::vector<Item> items;
  int64_t total_tiles = 0;
  for (int s = 0; s < (int)segs.size(); ++s) {
    const SegDesc& sg = segs[s];
    const int64_t pool_tiles = ceil_div(sg.n_slots, c.key_tile);
    for (int tok0 = 0; tok0 < sg.m; tok0 += c.q_tile_tokens) {
      const int ntok = std::min(c.q_tile_tokens, sg.m - tok0);
      const int64_t tail_tiles = ceil_div(std::min(tok0 + ntok, sg.tail_m), c.key_tile);
      for (int h = 0; h < c.Hkv; ++h) {
        items.push_back({s, h, tok0, ntok, pool_tiles + tail_tiles, pool_tiles});
        total_tiles += pool_tiles + tail_tiles;
      }
    }
  }
  if (items.empty()) return;
  // Choose the tiles-per-unit cap by an LPT makespan estimate over the CTAs
  // the units will form.  A CTA runs two units (two softmax slots) and costs
  // about the sum of their tiles plus a fixed overhead per unit (launch, Q
  // load, TMEM setup) and per split unit (partial write + merge).  With a
  // moderate job count the greedy LPT assignment onto the SMs is simulated;
  // with many jobs the bound sum/m + max is used (quantization is then small).
  const int64_t m_slots = std::max<int64_t>(1, (int64_t)c.num_sms * std::max(1, c.ctas_per_sm / 2));
  int64_t max_tiles = 0;
  for (auto& it : items) max_tiles = std::max(max_tiles, it.tiles);
  const int max_splits = c.max_splits > 0 ? c.max_splits : 1 << 20;
  std::vector<int64_t> cands;
  for (int64_t div = 1; div <= 64; div = div < 8 ? div + 1 : div * 3 / 2) {
    const int64_t t = std::max<int64_t>(std::max<int64_t>(1, c.min_tiles_per_unit), (max_tiles + div - 1) / div);
    if (cands.empty() || cands.back() != t) cands.push_back(t);
  }
  int64_t best_tpu = 0;
  double best_cost = 1e300;
  std::vector<double> unit_cost, jobs;
  for (int64_t tpu : cands) {
    unit_cost.clear();
    bool ok = true;
    for (auto& it : items) {
      const int64_t n = ceil_div(it.tiles, tpu);
      if (n > max_splits) { ok = false; break; }
      for (int64_t s = 0; s < n; ++s) {
        const int64_t t = it.tiles * (s + 1) / n - it.tiles * s / n;
        unit_cost.push_back((double)t + c.unit_overhead_tiles + (n > 1 ? c.split_overhead_tiles : 0.0));
      }
    }
    if (!ok) continue;
    std::sort(unit_cost.begin(), unit_cost.end(), std::greater<double>());
    jobs.clear();
    for (size_t i = 0; i < unit_cost.size(); i += 2)
      jobs.push_back(unit_cost[i] + (i + 1 < unit_cost.size() ? unit_cost[i + 1] : 0.0));
    const int64_t n_jobs = (int64_t)jobs.size() * c.n_layers;
    double makespan;
    if (n_jobs <= 24 * m_slots) {
      std::priority_queue<double, std::vector<double>, std::greater<double>> load;
      for (int64_t i = 0; i < m_slots; ++i) load.push(0.0);
      for (double jc : jobs)
        for (int l = 0; l < c.n_layers; ++l) {
          const double x = load.top();
          load.pop();
          load.push(x + jc);
        }
      makespan = 0.0;
      while (!load.empty()) { makespan = std::max(makespan, load.top()); load.pop(); }
    } else {
      double sum = 0.0;
      for (double jc : jobs) sum += jc;
      makespan = sum * c.n_layers / (double)m_slots + jobs.front();
    }
    const double cost = makespan * (1.0 + 1e-6 * (double)unit_cost.size());
    if (cost < best_cost) { best_cost = cost; best_tpu = tpu; }
  }
  // Order groups by per-unit work, largest first (LPT over the CTA rasterizer).
  std::vector<int> order(items.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  // A unit that cannot share a CTA with another q tile over the same keys (a
  // one-tile segment whose cached pool no other segment of the call reads, e.g.
  // a 32-token query of one session in a multi-tenant batch) would run alone in
  // a two-slot tcgen05 CTA with one softmax warpgroup idle.  Split it (into an
  // two key ranges) so the halves pair up as one SPLIT CTA instead.
  std::vector<int> seg_qtiles(segs.size(), 0), pool_users(segs.size(), 0);
  for (size_t s = 0; s < segs.size(); ++s) {
    seg_qtiles[s] = (int)ceil_div(segs[s].m, c.q_tile_tokens);
    for (size_t t = 0; t < segs.size(); ++t)
      if (segs[t].n_slots > 0 && segs[t].pages == segs[s].pages && segs[t].n_slots == segs[s].n_slots) ++pool_users[s];
  }
  auto n_splits_of = [&](const Item& it) -> int64_t {
    int64_t n = best_tpu > 0 ? ceil_div(it.tiles, best_tpu) : std::min<int64_t>(max_splits, it.tiles);
    n = std::max<int64_t>(1, std::min<int64_t>(n, std::max<int64_t>(1, it.tiles)));
    const bool alone = seg_qtiles[it.seg] == 1 && pool_users[it.seg] <= 1;
    if (c.pair_slots && alone && it.tiles >= 2 && n == 1 && max_splits >= 2) n = 2;
    return std::min<int64_t>(n, it.tiles);
  };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    const double wa = (double)items[a].tiles / (double)n_splits_of(items[a]);
    const double wb = (double)items[b].tiles / (double)n_splits_of(items[b]);
    return wa > wb;
  });
  for (int idx : order) {
    const Item& it = items[idx];
    const int64_t n = n_splits_of(it);
    const int unit0 = (int)out->units.size();
    const int group = (n > 1 || c.force_groups) ? (int)out->groups.size() : -1;
    for (int64_t s = 0; s < n; ++s) {
      WorkUnit u;
      u.seg = it.seg;
      u.kv_head = it.kvh;
      u.q_tok0 = it.tok0;
      u.q_ntok = it.ntok;
      u.tile_lo = (int)(it.tiles * s / n);
      u.tile_hi = (int)(it.tiles * (s + 1) / n);
      u.group = group;
      u.split = (int)s;
      if (c.fault == 1 && s == n - 1) u.tile_hi = std::max(u.tile_lo, u.tile_hi - 1);
      out->units.push_back(u);
    }
    if (group >= 0) out->groups.push_back({it.seg, it.kvh, it.tok0, it.ntok, unit0, (int)n});
  }
}

// Leading key tiles two units can share: same KV head and start tile, and the
// same keys behind those tile indices (same segment, or the same cached pool for
// the pool part of the tile list).
static int shared_tiles(const std::vector<SegDesc>& segs, const WorkUnit& a, const WorkUnit& b, int key_tile) {
  if (a.kv_head != b.kv_head || a.tile_lo != b.tile_lo) return -1;
  const int na = a.tile_hi - a.tile_lo, nb = b.tile_hi - b.tile_lo;
  if (a.seg == b.seg) return std::min(na, nb);
  const SegDesc& x = segs[a.seg];
  const SegDesc& y = segs[b.seg];
  if (x.pages != y.pages || x.n_slots != y.n_slots || x.hole_lo != y.hole_lo || x.hole_hi != y.hole_hi) return -1;
  const int pool_tiles = (x.n_slots + key_tile - 1) / key_tile;
  return std::max(0, std::min(std::min(na, nb), pool_tiles - a.tile_lo));
}

void pair_units_cta2(const std::vector<SegDesc>& segs, const Plan& plan, int key_tile, std::vector<TcPair>* out,
                     std::vector<char>* used) {
  out->clear();
  const int n = (int)plan.units.size();
  used->assign(n, 0);
  // Two units can share every tcgen05.mma of a CTA pair when all their key
  // tiles are the same keys: same KV head and tile range, and the same segment
  // (q tiles of one append / prompt) or the same cached pool with no private
  // own-token tiles in the range.
  auto pool_tiles = [&](const WorkUnit& u) { return (segs[u.seg].n_slots + key_tile - 1) / key_tile; };
  auto same_keys = [&](const WorkUnit& a, const WorkUnit& b) {
    if (a.kv_head != b.kv_head || a.tile_lo != b.tile_lo || a.tile_hi != b.tile_hi) return false;
    if (a.seg == b.seg) return a.q_tok0 != b.q_tok0;
    const SegDesc& x = segs[a.seg];
    const SegDesc& y = segs[b.seg];
    return x.pages == y.pages && x.n_slots == y.n_slots && x.hole_lo == y.hole_lo && x.hole_hi == y.hole_hi &&
           a.tile_hi <= pool_tiles(a);
  };
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  auto key_of = [&](int i) {
    const WorkUnit& u = plan.units[i];
    const SegDesc& s = segs[u.seg];
    return std::make_tuple(u.kv_head, u.tile_lo, u.tile_hi, (uintptr_t)s.pages, s.n_slots, u.seg, u.q_tok0);
  };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return key_of(a) < key_of(b); });
  for (int ii = 0; ii + 1 < n; ++ii) {
    const int a = order[ii], b = order[ii + 1];
    if ((*used)[a] || (*used)[b]) continue;
    if (plan.units[a].tile_hi == plan.units[a].tile_lo) continue;
    if (same_keys(plan.units[a], plan.units[b])) {
      (*used)[a] = (*used)[b] = 1;
      out->push_back({a, b, plan.units[a].tile_hi - plan.units[a].tile_lo, 0});
    }
  }
  std::stable_sort(out->begin(), out->end(), [](const TcPair& x, const TcPair& y) { return x.n_shared > y.n_shared; });
}

void pair_units(const std::vector<SegDesc>& segs, const Plan& plan, int key_tile, std::vector<TcPair>* out,
                const std::vector<char>* skip) {
  out->clear();
  const int n = (int)plan.units.size();
  std::vector<char> used(n, 0);
  if (skip)
    for (int i = 0; i < n; ++i) used[i] = (*skip)[i];
  // 1. shared-key pairs: bucket by (kv_head, tile_lo, pool), pair neighbours
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  auto key_of = [&](int i) {
    const WorkUnit& u = plan.units[i];
    const SegDesc& s = segs[u.seg];
    return std::make_tuple(u.kv_head, u.tile_lo, (uintptr_t)s.pages, s.n_slots, u.seg, -(u.tile_hi - u.tile_lo));
  };
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return key_of(a) < key_of(b); });
  for (int ii = 0; ii < n; ++ii) {
    const int a = order[ii];
    if (used[a]) continue;
    for (int jj = ii + 1; jj < n && jj < ii + 8; ++jj) {
      const int b = order[jj];
      if (used[b]) continue;
      const WorkUnit& ua = plan.units[a];
      const WorkUnit& ub = plan.units[b];
      if (ua.seg == ub.seg && ua.q_tok0 == ub.q_tok0) continue;   // same q tile: split pair below
      const int sh = shared_tiles(segs, ua, ub, key_tile);
      if (sh > 0) {
        used[a] = used[b] = 1;
        out->push_back({a, b, sh, 0});
        break;
      }
    }
  }
  // 2. split pairs: two key ranges of one q tile (same group)
  for (int i = 0; i < n; ++i) {
    if (used[i]) continue;
    const WorkUnit& u = plan.units[i];
    int partner = -1;
    if (u.group >= 0)
      for (int j = i + 1; j < n; ++j)
        if (!used[j] && plan.units[j].group == u.group) { partner = j; break; }
    used[i] = 1;
    if (partner >= 0) {
      used[partner] = 1;
      out->push_back({i, partner, 0, 1});
    } else {
      out->push_back({i, -1, 0, 1});
    }
  }
  // Largest CTA first (tiles loaded + tiles computed).
  auto work = [&](const TcPair& p) {
    const int wa = plan.units[p.ua].tile_hi - plan.units[p.ua].tile_lo;
    const int wb = p.ub >= 0 ? plan.units[p.ub].tile_hi - plan.units[p.ub].tile_lo : 0;
    return 2 * (wa + wb) + (wa + wb - p.n_shared);
  };
  std::stable_sort(out->begin(), out->end(), [&](const TcPair& a, const TcPair& b) { return work(a) > work(b); });
}

}  // namespace ssa
