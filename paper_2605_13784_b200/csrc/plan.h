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

// Pair units whose key tiles are the same keys into cta_group::2 CTA pairs
// (kernels_tc2.cu): ua runs on CTA rank 0, ub on rank 1; n_shared = tiles.
// `used` marks the paired units (the rest go to pair_units).
void pair_units_cta2(const std::vector<SegDesc>& segs, const Plan& plan, int key_tile, std::vector<TcPair>* out,
                     std::vector<char>* used);

}  // namespace ssa
