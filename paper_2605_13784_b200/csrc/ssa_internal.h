// ssa_internal.h — internal descriptors shared by the host core (store.cpp,
// plan.cpp) and the sm_100a kernels (*.cu).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <deque>
#include <string>
#include <vector>

#include "ssa.h"

namespace ssa {

// A segment is a run of m new tokens of one session (or a stateless prompt)
// whose rows attend to the session's cached keys followed by the segment's own
// keys, causally (Eq. query-attention; reading R-2).
struct SegDesc {
  int64_t row0;          // first token row of the segment in the packed inputs
  int32_t m;             // tokens (query rows) in the segment
  int32_t tail_m;        // own keys visible to the rows (m, or 0 on a non-tail rank of a sharded query)
  int32_t n_slots;       // slot extent of the visible cached keys (0: none)
  int32_t hole_lo;       // slots [hole_lo, hole_hi) hold no token (R0 page pad, R-9)
  int32_t hole_hi;
  int32_t append_slot0;  // slot of the first new token when the segment is appended, else -1
  int32_t n_pages;       // entries of `pages` valid for this launch
  const int32_t* pages;  // device page table of the session (slot/P -> page id)
};

// One CTA's work: q tile (tokens [q_tok0, q_tok0+q_ntok) of segment `seg`, all
// G query heads of KV head `kv_head`) over key tiles [tile_lo, tile_hi) of the
// segment's tile list (pool tiles first, then tail tiles).
struct WorkUnit {
  int32_t seg;
  int32_t kv_head;
  int32_t q_tok0;
  int32_t q_ntok;
  int32_t tile_lo;
  int32_t tile_hi;
  int32_t group;   // combine group (partial output) or -1 (write O directly)
  int32_t split;   // index of this unit within its group
};

// Output group: the splits of one (segment, kv head, q tile) to be merged.
struct Group {
  int32_t seg;
  int32_t kv_head;
  int32_t q_tok0;
  int32_t q_ntok;
  int32_t unit0;     // first unit index (units of a group are contiguous)
  int32_t n_splits;
};

// tcgen05 CTA = up to two work units ("slots") run by two softmax warpgroups.
// The first n_shared key tiles of both slots are the same keys: each TMA load
// feeds both slots (256 query rows per K/V tile: the q tiles of one append, or
// Flash Queries over one cached pool).  Later tiles are private to a slot and
// loaded separately (own-token tails; the two halves of a split).  same_q: both
// slots use one q tile (a split pair), so only one Q buffer is needed.
// The host fills the copies below before the upload: a CTA reads its units, their
// segments and their groups' split counts in one round of independent loads (no
// pairs -> units -> segments / groups dependency chain in the kernel prologue).
struct TcPair {
  int32_t ua, ub;     // unit indices (ub = -1: single slot)
  int32_t n_shared;   // leading tiles shared by both slots
  int32_t same_q;
  int32_t splits_a, splits_b;   // Group::n_splits of the units' groups (0: no group)
  int32_t unit0_a, unit0_b;     // Group::unit0 of the units' groups
  WorkUnit wa, wb;              // units[ua], units[ub] (wb = wa for a single slot)
  SegDesc sa, sb;               // segs[wa.seg], segs[wb.seg]
};

struct AttnParams {
  const void* Q;         // [n_layers_in][rows_per_layer][Hq][D]
  const void* Kt;        // [n_layers_in][rows_per_layer][Hkv][D]  (segment "tail" keys)
  const void* Vt;
  void* O;               // like Q
  int64_t rows_per_layer;
  int32_t layer0;        // pool layer of grid.y == 0
  int32_t in_layer_stride;  // 1 if inputs carry a layer dimension per grid.y, else 0
  const void* poolK;     // [L][num_pages][Hkv][P][D]
  const void* poolV;
  int64_t num_pages;
  int32_t Hq, Hkv, D, P, G;
  float scale_log2;      // softmax_scale * log2(e)
  const SegDesc* segs;
  const WorkUnit* units;
  int32_t n_units;       // per layer
  const Group* groups;
  int32_t n_groups;      // per layer
  float* part_o;         // [layers][n_units][rows_tile][D]
  float* part_lse;       // [layers][n_units][rows_tile]
  int32_t rows_tile;     // rows per unit (q tile tokens * G)
  int32_t key_tile;      // keys per tile (SIMT 64, tcgen05 128)
  int32_t fault;         // SSA_OPT_FAULT_INJECT
  const TcPair* pairs;   // tcgen05 CTAs (per layer)
  int32_t n_pairs;
  // Cluster merge (tcgen05 path, kernels_tc.cu "CM"): cm_C = cluster size (CTAs
  // per cluster, consecutive blockIdx.x), 0 = off (partials + combine kernel).
  // In CM every unit has a group; Group::n_splits = K clusters per group and
  // WorkUnit::split = the unit's cluster index in [0, K); groups with K > 1 leave
  // K block partials for cm_merge_kernel.
  int32_t cm_C;
  // 1: the previous grid in the stream does not write the KV pool, so pool tiles may
  // be loaded before griddepcontrol.wait (programmatic dependent launch)
  int32_t pool_early;
  // groups over K > 1 clusters: merge tickets [layers][n_groups][cm_C] (zero between
  // launches) for the in-kernel last-arriver merge, or null: cm_merge_kernel
  int32_t* cm_tickets;
  // 1: group-barrier merge (cm_C == 1, one wave): groups over K > 1 CTAs write global
  // partials, meet at a barrier in cm_tickets ([layers][n_groups][2]: arrivals,
  // generation; zero at allocation) and merge in the same kernel (gm_reduce)
  int32_t cm_gbar;
  // 1: as cm_gbar, but no barrier: the CTAs exit after writing their partials and
  // gm_merge_kernel (a programmatic launch right behind) merges the groups
  int32_t cm_gsplit;
  // pool tiles are loaded with an L2 evict-first hint (read once per launch)
  int32_t l2_evict_first;
  // FP8 KV variant (reading R-22): pools and Kt/Vt hold E4M3 codes; scale_log2
  // already includes k_scale, o_scale = v_scale multiplies 1/l
  int32_t kv_fp8;
  float o_scale;
};

struct QuantParams {
  const void* K;         // bf16 [n] (flattened [layers][rows][Hkv][D])
  const void* V;
  uint8_t* K8;           // E4M3 codes [n]
  uint8_t* V8;
  int64_t n;             // elements per tensor (multiple of 16)
  float k_scale, v_scale;
};

// Append scatter (KA): copy new K/V rows into pages, bit-exact.
struct ScatterParams {
  const void* K;         // [n_layers][rows_per_layer][Hkv][D]
  const void* V;
  int64_t rows_per_layer;
  int32_t layer0;
  int32_t in_layer_stride;
  void* poolK;
  void* poolV;
  int64_t num_pages;
  int32_t Hkv, D, P, elem_bytes;
  const SegDesc* segs;   // segments with append_slot0 >= 0
  const int32_t* tok_prefix;  // [n_segs+1] prefix sums of m over segs
  int32_t n_segs;
  int64_t total_tokens;
};

// Gather (read-back) of tokens [start, start+count) of one layer.
struct GatherParams {
  const void* poolK;
  const void* poolV;
  void* K;               // [count][Hkv][D]
  void* V;
  int64_t num_pages;
  int32_t layer, Hkv, D, P, elem_bytes;
  int64_t start, count;
  int32_t n_prefix_slots_pad;  // slot of token n_prefix (R0 padded) or -1
  int64_t n_prefix;
  const int32_t* pages;
};

// Merge of split partials into O.
struct CombineParams {
  int32_t combine_rows;  // rows of a group per CTA (set by launch_combine)
  const float* part_o;
  const float* part_lse;
  void* O;
  float* lse_out;        // optional lse (log2 units) in O layout [rows][Hq]
  float* o_f32;          // optional: write fp32 O here (O layout) instead of O
  const SegDesc* segs;
  const Group* groups;
  int32_t n_groups;
  int32_t n_units;
  int32_t rows_tile;
  int64_t rows_per_layer;
  int32_t in_layer_stride;
  int32_t Hq, G, D;
  int32_t write_o;
  // peer push (A9 over peer memory): when n_peers > 0 the fp32 O / lse rows are
  // written to every peer's gathered buffer (chunk base peer_chunk[q]; lse at
  // +lse_off floats) instead of o_f32 / lse_out
  const uint64_t* peer_chunk;
  int32_t n_peers;
  int64_t lse_off;
};

// On-device greedy sampling (kernels_sample.cu).
struct SampleParams {
  const void* logits;      // [n_rows][row_stride] fp32 or bf16
  int64_t row_stride;      // elements
  int32_t vocab;
  int32_t n_rows;
  int32_t splits;          // CTAs per row
  void* partials;          // [n_rows][splits] reduction triples (scratch)
  int32_t* row_counters;   // [n_rows + 1], zero between calls
  int32_t* out_ids;        // [n_rows] device
  float* out_gap;          // [n_rows] device or null
  float* out_top;          // [n_rows][2] (l1, l2) device or null
  const int32_t* draft;    // [n_rows] device or null
  int32_t* out_n_accept;   // device, used when draft != null
};

// cudaFuncSetAttribute(func, MaxDynamicSharedMemorySize, bytes) once per (device,
// function): the attribute is per device, so a process with stores on several
// devices sets it on each (store.cpp; thread-safe).
cudaError_t set_smem_attr_once(const void* func, int bytes);

// Kernel launchers (kernels_*.cu).  Return cudaGetLastError() after launch.
// Fused data-plane projection (kernels_qkv.cu).
struct QkvParams {
  const void* X;          // [m][hidden] bf16 token rows
  const void* W;          // [(Hq + 2 Hkv) D][hidden] bf16 (nn.Linear weight: Q, K, V head rows)
  void* Q;                // [m][Hq][D] bf16
  void* K;                // [m][Hkv][D] bf16, or null (paged destination only)
  void* V;
  int32_t m, hidden, Hq, Hkv, D;
  int64_t pos0;           // absolute position of token row 0 (never re-based, R-8)
  double rope_theta;      // <= 0: no rotary embedding
  void* poolK;            // optional paged destination: [L][num_pages][Hkv][P][D]
  void* poolV;
  const int32_t* pages;   // device page table of the session (slot / P -> page)
  int64_t page_base;      // layer * num_pages
  int32_t slot0, P;       // slot of token row 0
  int32_t kv_fp8;         // paged destination holds E4M3 codes of x / k_scale, x / v_scale (R-22)
  float k_scale, v_scale;
  int32_t splits;         // split-K factor = thread-block cluster size
  int32_t debug;          // experiments (SSA_QKV_DEBUG): 1 = skip the reduce / RoPE / store epilogue
  uint64_t* trace;        // experiments: per-CTA %globaltimer stamps [grid][8], or null
};

cudaError_t launch_attn_simt(const AttnParams& p, int n_layers, bool bf16, cudaStream_t s);
cudaError_t launch_combine(const CombineParams& p, int n_layers, bool bf16, cudaStream_t s, int max_splits);
cudaError_t launch_scatter(const ScatterParams& p, int n_layers, cudaStream_t s);
cudaError_t launch_quant_e4m3(const QuantParams& p, cudaStream_t s);
cudaError_t launch_gather(const GatherParams& p, cudaStream_t s);
cudaError_t launch_qkv_rope(const QkvParams& p, cudaStream_t s, bool pdl);
bool qkv_supported(int D, int hidden);
int qkv_choose_splits(int m, int n_heads, int hidden, int num_sms);
int qkv_max_active_clusters(int splits);
cudaError_t launch_greedy(const SampleParams& p, bool bf16, cudaStream_t s);
size_t sample_partial_bytes();
// Merge `world` rank partials (packed chunks [O fp32 rows*Hq*D | lse rows*Hq]) into O.
cudaError_t launch_merge_ranks(const float* parts, int world, int64_t rows, int Hq, int D, void* O, bool bf16,
                               cudaStream_t s);
// Release `epoch` into flag slot `slot` of every peer (after the stream's prior work).
cudaError_t launch_signal_peers(const uint64_t* peer_flags, int n_peers, int slot, uint32_t epoch, cudaStream_t s);
// One block waits until flags[i] >= epoch for i < n (acquire, system scope).
cudaError_t launch_wait_flags(const uint32_t* flags, int n, uint32_t epoch, cudaStream_t s);
int simt_rows_tile(int G, int D);     // rows per SIMT unit
int simt_key_tile();                  // keys per SIMT tile

// ---------------------------------------------------------------------------
// Host-side helpers
// ---------------------------------------------------------------------------

// Pinned host ring with a device mirror for per-call uploads (work lists,
// page-table deltas).  Regions are reused only after the event recorded
// behind their consumers has completed.
class UploadRing {
 public:
  ~UploadRing();
  cudaError_t init(size_t cap);
  // Reserve n bytes (256-aligned); returns offset or SIZE_MAX on failure.
  size_t alloc(size_t n);
  char* host(size_t off) { return h_ + off; }
  char* dev(size_t off) { return d_ + off; }
  cudaError_t to_device(size_t off, size_t n, cudaStream_t s) {
    return cudaMemcpyAsync(d_ + off, h_ + off, n, cudaMemcpyHostToDevice, s);
  }
  // Mark [lo, hi) busy until work now enqueued on `s` completes.
  cudaError_t fence(size_t lo, size_t hi, cudaStream_t s);
  size_t capacity() const { return cap_; }

 private:
  struct Span { size_t lo, hi; cudaEvent_t ev; };
  char* h_ = nullptr;
  char* d_ = nullptr;
  size_t cap_ = 0, head_ = 0;
  std::deque<Span> busy_;
  std::vector<cudaEvent_t> free_events_;
  cudaError_t retire_overlapping(size_t lo, size_t hi);
};

}  // namespace ssa
