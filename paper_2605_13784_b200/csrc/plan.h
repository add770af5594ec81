// plan.h — split-KV work planner (host).
#pragma once
#include <vector>

#include "ssa_internal.h"

namespace ssa {

struct PlanConfig {
  int Hkv = 1;
  int q_tile_tokens = 1;     // tokens per q tile (rows_tile / G)
  int key_tile = 64;         // keys per tile
  int n_layers = 1;          // grid.y of the launch
  int num_sms = 148;
  int ctas_per_sm = 1;
  int max_splits = 0;        // 0 = unlimited
  int min_tiles_per_unit = 1;
  double unit_overhead_tiles = 1.0;
  double split_overhead_tiles = 1.0;   // extra cost of a split unit (partial write + merge), in tiles
  int fault = 0;
  bool force_groups = false;  // every item writes partials (sharded query)
  bool pair_slots = false;    // units run in two-slot (tcgen05) CTAs: avoid lone units
};

struct Plan {
  std::vector<WorkUnit> units;
  std::vector<Group> groups;
};

void plan_units(const std::vector<SegDesc>& segs, const PlanConfig& c, Plan* out);

// Pair units into two-slot tcgen05 CTAs (SHARED first, then SPLIT, then SINGLE),
// largest work first.
void pair_units(const std::vector<SegDesc>& segs, const Plan& plan, int key_tile, std::vector<TcPair>* out,
                const std::vector<char>* skip = nullptr);

// Cluster-merge plans (kernels_tc.cu "CM"; AttnParams::cm_C).
//
// plan_cm: a single launch layer.  Every (segment, q tile, kv head) item is a
// group; consecutive q tiles of one segment over the same keys (or single-q-tile
// segments over one cached pool, e.g. Flash Queries) pair up as SHARED CTAs, a
// lone q tile runs as SPLIT CTAs (two key ranges per CTA).  Pair-item p gets K_p
// clusters of C CTAs (consecutive CTAs, C key ranges each), K_p chosen so that
// the clusters fit `max_clusters` and the largest per-CTA key range is smallest.
// Returns the estimated makespan in key tiles (+ merge overheads), or -1 if the
// plan does not apply.
// gbar: the group-barrier merge (AttnParams::cm_gbar): C = 1, every CTA in one wave
// (used <= max_clusters), at most 32 CTAs per group, a flat merge cost.
double plan_cm(const std::vector<SegDesc>& segs, const PlanConfig& c, int C, int max_clusters, Plan* plan,
               std::vector<TcPair>* pairs, bool gbar = false);

// cm_regroup: turn an LPT plan (plan_units + pair_units) into a C = 1 CM plan:
// every unit gets a group (singletons for unsplit units), Group::n_splits becomes
// the number of CTAs holding the group and WorkUnit::split the unit's CTA index
// within it (both units of a SPLIT pair share one, merged in the CTA).
void cm_regroup(Plan* plan, const std::vector<TcPair>& pairs);

}  // namespace ssa
