// plan.cpp — split-KV work planner (host, integer only).
//
// Turns the segments of one call into CTA work units: for every segment,
// every q tile of `q_tile_tokens` tokens and every KV head, the key tiles
// (cached pool tiles, then the segment's own tiles up to the q tile's last
// token — causal, reading R-2) are split into contiguous ranges so that the
// launch fills the GPU (148 SMs on B200).  Units of one (segment, q tile, kv
// head) form a Group merged by the combine kernel (log-sum-exp, reading R-11).
#include <algorithm>
#include <cmath>
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

namespace ssa {

double plan_cm(const std::vector<SegDesc>& segs, const PlanConfig& c, int C, int max_clusters, Plan* plan,
               std::vector<TcPair>* pairs, bool gbar) {
  plan->units.clear();
  plan->groups.clear();
  pairs->clear();
  if (C < 1 || max_clusters < 1) return -1.0;
  struct Item { int seg, kvh, tok0, ntok; int tiles; };
  std::vector<Item> items;
  for (int s = 0; s < (int)segs.size(); ++s) {
    const SegDesc& sg = segs[s];
    const int pool_tiles = (int)ceil_div(sg.n_slots, c.key_tile);
    for (int tok0 = 0; tok0 < sg.m; tok0 += c.q_tile_tokens) {
      const int ntok = std::min(c.q_tile_tokens, sg.m - tok0);
      const int tail_tiles = (int)ceil_div(std::min(tok0 + ntok, sg.tail_m), c.key_tile);
      for (int h = 0; h < c.Hkv; ++h) items.push_back({s, h, tok0, ntok, pool_tiles + tail_tiles});
    }
  }
  if (items.empty()) return -1.0;
  // pair-items: SHARED (two q tiles over common leading key tiles) or SPLIT (one q tile)
  struct PItem { int a, b; int sh; double work; int cap; };
  std::vector<int> order(items.size());
  for (size_t i = 0; i < order.size(); ++i) order[i] = (int)i;
  auto key_of = [&](int i) {
    const Item& it = items[i];
    const SegDesc& sg = segs[it.seg];
    return std::make_tuple(it.kvh, (uintptr_t)sg.pages, sg.n_slots, sg.hole_lo, sg.hole_hi, it.seg, it.tok0);
  };
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return key_of(x) < key_of(y); });
  auto common = [&](const Item& x, const Item& y) -> int {
    if (x.kvh != y.kvh) return 0;
    if (x.seg == y.seg) return std::min(x.tiles, y.tiles);
    const SegDesc& a = segs[x.seg];
    const SegDesc& b = segs[y.seg];
    if (a.n_slots == 0 || a.pages != b.pages || a.n_slots != b.n_slots || a.hole_lo != b.hole_lo || a.hole_hi != b.hole_hi)
      return 0;
    return (int)ceil_div(a.n_slots, c.key_tile);
  };
  std::vector<PItem> pis;
  for (size_t i = 0; i < order.size(); ++i) {
    const Item& x = items[order[i]];
    if (i + 1 < order.size()) {
      const Item& y = items[order[i + 1]];
      const int sh = common(x, y);
      if (sh > 0) {
        pis.push_back({order[i], order[i + 1], sh, (double)(x.tiles + y.tiles - sh), std::max(1, sh)});
        ++i;
        continue;
      }
    }
    // SPLIT: a CTA's two slots take two key ranges of the q tile
    pis.push_back({order[i], -1, 0, 0.5 * x.tiles + 0.5, std::max(1, x.tiles / 2)});
  }
  // clusters per pair-item: K_p = 1 each, then one more to the most loaded while they fit
  const int np = (int)pis.size();
  std::vector<int> K(np, 1);
  int used = np;
  // gbar: whole key tiles per slot (a split item's 2 C K ranges, a shared pair's C K
  // ranges), so clusters that leave the largest range unchanged are given back
  auto per_cta = [&](int i) {
    if (!gbar) return pis[i].work / (double)(C * K[i]);
    const PItem& pi = pis[i];
    if (pi.b < 0) return (double)ceil_div(items[pi.a].tiles, 2 * C * K[i]);
    return std::ceil(pi.work / (double)(C * K[i]) - 1e-9);
  };
  if (np <= max_clusters) {
    std::priority_queue<std::pair<double, int>> q;
    for (int i = 0; i < np; ++i) q.push({per_cta(i), i});
    while (used < max_clusters && !q.empty()) {
      const int i = q.top().second;
      q.pop();
      if (C * (K[i] + 1) > pis[i].cap) continue;   // no empty ranges beyond this
      ++K[i];
      ++used;
      q.push({per_cta(i), i});
    }
    // give back clusters that do not lower the makespan (ties: one spare cluster for
    // one of several equally loaded items only adds a merge)
    double mx = 0.0;
    for (int i = 0; i < np; ++i) mx = std::max(mx, per_cta(i));
    for (int i = 0; i < np; ++i)
      while (K[i] > 1) {
        --K[i];
        if (per_cta(i) > mx) { ++K[i]; break; }
        --used;
      }
  }
  // cost: largest per-CTA range, with waves if the clusters do not fit at once
  double cost = 0.0;
  const double waves = std::ceil((double)used / (double)max_clusters);
  if (gbar) {
    // group-barrier merge: one wave of single CTAs, a group's partial lse fit a warp
    if (C != 1 || used > max_clusters) return -1.0;
    for (int i = 0; i < np; ++i)
      if (K[i] > 32) return -1.0;
  }
  for (int i = 0; i < np; ++i) {
    const double merge = gbar ? (K[i] > 1 ? 1.0 : 0.0)
                              : (C > 1 ? 0.25 : 0.0) + (K[i] > 1 ? 1.0 + 0.5 * (K[i] - 1) / (double)C : 0.0);
    cost = std::max(cost, per_cta(i) + merge);
  }
  cost *= waves;
  // units, groups and CTAs, cluster by cluster
  for (int i = 0; i < np; ++i) {
    const PItem& pi = pis[i];
    const int S = C * K[i];
    auto new_group = [&](const Item& it) {
      plan->groups.push_back({it.seg, it.kvh, it.tok0, it.ntok, (int)plan->units.size(), K[i]});
      return (int)plan->groups.size() - 1;
    };
    if (pi.b < 0) {
      const Item& it = items[pi.a];
      const int g = new_group(it);
      for (int u = 0; u < 2 * S; ++u) {
        WorkUnit w;
        w.seg = it.seg;
        w.kv_head = it.kvh;
        w.q_tok0 = it.tok0;
        w.q_ntok = it.ntok;
        w.tile_lo = (int)((int64_t)it.tiles * u / (2 * S));
        w.tile_hi = (int)((int64_t)it.tiles * (u + 1) / (2 * S));
        w.group = g;
        w.split = (u / 2) / C;
        if (c.fault == 1 && u == 2 * S - 1) w.tile_hi = std::max(w.tile_lo, w.tile_hi - 1);
        plan->units.push_back(w);
      }
      const int u0 = plan->groups[g].unit0;
      for (int j = 0; j < S; ++j) pairs->push_back({u0 + 2 * j, u0 + 2 * j + 1, 0, 1});
    } else {
      const Item& ia = items[pi.a];
      const Item& ib = items[pi.b];
      const int ga = new_group(ia);
      for (int j = 0; j < S; ++j) {
        WorkUnit w;
        w.seg = ia.seg;
        w.kv_head = ia.kvh;
        w.q_tok0 = ia.tok0;
        w.q_ntok = ia.ntok;
        w.tile_lo = (int)((int64_t)pi.sh * j / S);
        w.tile_hi = j == S - 1 ? ia.tiles : (int)((int64_t)pi.sh * (j + 1) / S);
        w.group = ga;
        w.split = j / C;
        plan->units.push_back(w);
      }
      const int gb = new_group(ib);
      for (int j = 0; j < S; ++j) {
        WorkUnit w;
        w.seg = ib.seg;
        w.kv_head = ib.kvh;
        w.q_tok0 = ib.tok0;
        w.q_ntok = ib.ntok;
        w.tile_lo = (int)((int64_t)pi.sh * j / S);
        w.tile_hi = j == S - 1 ? ib.tiles : (int)((int64_t)pi.sh * (j + 1) / S);
        w.group = gb;
        w.split = j / C;
        if (c.fault == 1 && j == S - 1) w.tile_hi = std::max(w.tile_lo, w.tile_hi - 1);
        plan->units.push_back(w);
      }
      const int ua0 = plan->groups[ga].unit0, ub0 = plan->groups[gb].unit0;
      for (int j = 0; j < S; ++j) {
        const WorkUnit& a = plan->units[ua0 + j];
        const WorkUnit& b = plan->units[ub0 + j];
        const int n_sh = std::max(0, std::min(std::min(a.tile_hi, b.tile_hi), pi.sh) - a.tile_lo);
        pairs->push_back({ua0 + j, ub0 + j, n_sh, 0});
      }
    }
  }
  return cost;
}

void cm_regroup(Plan* plan, const std::vector<TcPair>& pairs) {
  // singleton groups for unsplit units
  for (int u = 0; u < (int)plan->units.size(); ++u) {
    WorkUnit& w = plan->units[u];
    if (w.group >= 0) continue;
    plan->groups.push_back({w.seg, w.kv_head, w.q_tok0, w.q_ntok, u, 1});
    w.group = (int)plan->groups.size() - 1;
    w.split = 0;
  }
  // CTA index of every unit within its group
  std::vector<int> n_ctas(plan->groups.size(), 0);
  for (const TcPair& pr : pairs) {
    WorkUnit& a = plan->units[pr.ua];
    const int ia = n_ctas[a.group]++;
    a.split = ia;
    if (pr.ub >= 0) {
      WorkUnit& b = plan->units[pr.ub];
      if (pr.same_q && b.group == a.group) {
        b.split = ia;   // merged with `a` in the CTA
      } else {
        b.split = n_ctas[b.group]++;
      }
    }
  }
  for (size_t g = 0; g < plan->groups.size(); ++g) plan->groups[g].n_splits = n_ctas[g];
}

}  // namespace ssa
