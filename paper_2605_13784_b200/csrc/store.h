// store.h — the store and session objects behind the opaque ssa_store_t.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <functional>
#include <queue>
#include <string>
#include <vector>

#include "ssa.h"
#include "plan.h"
#include "ssa_internal.h"

namespace ssa {

void set_error(const char* fmt, ...);

struct Session {
  bool live = false;
  int64_t n_prefix = 0;   // Region 0 length
  int64_t n_tokens = 0;   // retained tokens (R0 + R1)
  uint64_t version = 0;   // data version t
  // Region-1 FIFO eviction (Alg. 1): evicted R1 slots at the start of
  // the first retained R1 page (0..P-1; whole evicted pages leave the table),
  // total evicted tokens (positions are never re-based) and the retention cap.
  int64_t r1_skip = 0;
  int64_t n_evicted = 0;
  int64_t retention = 0;  // 0 = unlimited
  std::vector<int32_t> pages;   // host page table: slot / P -> page id
  int32_t* d_pages = nullptr;   // device mirror
  int64_t d_cap = 0;
  int64_t d_valid = 0;
  // open append (per-layer ticket or per-layer batch)
  bool ticket_open = false;
  bool batch_ticket = false;
  int32_t ticket_id = 0;
  int32_t ticket_n_new = 0;
  int64_t ticket_pages = 0;
  std::vector<uint8_t> ticket_done;
};

struct IoBuf {
  const void* user = nullptr;  // caller pointer
  size_t bytes = 0;
  void* dev = nullptr;         // device pointer the kernels use
  void* host = nullptr;        // non-null when `user` is host memory
  size_t stage_off = 0;
  IoBuf() = default;
  IoBuf(const void* u, size_t b) : user(u), bytes(b) {}
};

struct IoSet {
  IoBuf q, k, v, o;
};

struct RunOpts {
  bool force_groups = false;   // all outputs as partials through the combine
  float* o_f32 = nullptr;      // combine writes fp32 O here (O layout)
  float* lse_out = nullptr;    // combine writes lse (log2) here, [rows][Hq]
  const uint64_t* peer_chunk = nullptr;   // device: combine pushes fp32 O / lse to these peer chunks
  int32_t n_peers = 0;
  int64_t lse_off = 0;
  bool skip_scatter = false;   // K/V of the appended segments are already in their pages
};

// tcgen05 path (kernels_tc.cu)
int tc_key_tile();
int tc_debug_trace(void* host, size_t bytes);
int tc_rows_tile();
cudaError_t launch_attn_tc(const AttnParams& p, int n_layers, bool pdl, cudaStream_t s);
size_t tc_smem_bytes();
cudaError_t launch_cm_merge(const AttnParams& p, int n_layers, int max_split, bool pdl, cudaStream_t s);
cudaError_t launch_gm_merge(const AttnParams& p, int n_layers, int max_split, bool pdl, cudaStream_t s);
cudaError_t tc_configure(bool f8);
int tc_max_active_clusters(int c, bool f8);
bool tc_supported_shape(int D, int G, bool bf16);
// bf16 tensor map, 128-byte swizzle (kernels_tc.cu); false if the driver entry point is missing.
bool encode_bf16_map(CUtensorMap* m, const void* base, int rank, const cuuint64_t* dims,
                     const cuuint64_t* strides_bytes, const cuuint32_t* box);

}  // namespace ssa

struct CommState;

// Public calls that enqueue device work are ordered after the store's previous call.
#define SSA_ORDERED(st, stream)                     \
  ssa_store::Ordered ssa_ordered_((st), (stream)); \
  if (!ssa_ordered_.ok) return SSA_ERR_CUDA

struct ssa_store {
  ssa_store_config cfg{};
  int elem = 2;            // bytes per Q/K/V/O element at the ABI
  int pelem = 2;           // bytes per pool element (1: E4M3 codes)
  bool kv_fp8 = false;     // SSA_KV_E4M3 (reading R-22)
  uint8_t* kv8 = nullptr;  // E4M3 codes of the current call's K and V (tails + scatter source)
  size_t kv8_cap = 0;
  float scale = 1.f;
  int num_sms = 148;
  bool sm100 = false;
  void* poolK = nullptr;
  void* poolV = nullptr;
  bool pool_owned = true;   // false: ssa_store_config::pool_ptr (caller-owned)
  size_t pool_half_bytes = 0;
  std::vector<ssa::Session> sessions;
  std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> free_pages;
  std::vector<int32_t> page_ref;   // referers per page (aliased prefixes share pages)
  bool failed = false;
  std::string fail_msg;
  ssa::UploadRing ring;
  // Plans of recent calls (planner + CTA pairing are pure functions of the segment
  // shapes and options): per-layer calls of one step, repeated queries between
  // appends and Flash Query cycles skip the LPT search.
  // Each entry keeps the device copy of its work lists (segments, units, groups,
  // scatter segments, CTA pairs), so a repeated call shape launches without an
  // upload.  Entries read by a captured CUDA graph are pinned (never evicted).
  struct PlanCacheEntry {
    std::vector<int64_t> key;
    ssa::Plan plan;
    std::vector<ssa::TcPair> pairs;
    int32_t cm_C = 0;          // cluster-merge launch (AttnParams::cm_C), 0 = combine kernel / SIMT
    int32_t max_split = 0;     // largest Group::n_splits
    bool gbar = false;         // group-barrier plan (AttnParams::cm_gbar, or cm_gsplit when gsplit)
    bool gsplit = false;       // merged by gm_merge_kernel instead of the in-kernel barrier
    bool l2_hint = false;      // every key tile is read by one CTA (no reuse in L2 to keep)
    int32_t n_app = 0;         // scatter segments
    int32_t app_tokens = 0;
    std::vector<char> image;   // host copy of the lists
    size_t off[6] = {};
    size_t bytes = 0;
    char* dev = nullptr;
    bool pinned = false;
    int64_t last_use = 0;
  };
  std::vector<PlanCacheEntry> plan_cache;   // at most 16 unpinned entries
  int64_t plan_cache_hits = 0, plan_clock = 0;
  int max_clusters_[2][17];   // [E4M3][C]: co-resident clusters of C CTAs (-1 = not queried)
  int max_clusters(int C);
  // CUDA-graph capture (query plane): work lists of captured calls live in this
  // arena (pinned host + device, bump-allocated, never recycled while the store
  // lives) so the captured H2D copy node reads the same bytes at every replay.
  char* arena_h = nullptr;
  char* arena_d = nullptr;
  size_t arena_cap = 0, arena_used = 0;
  float* part_o = nullptr;
  size_t part_o_cap = 0;
  float* part_lse = nullptr;
  size_t part_lse_cap = 0;
  void* stage = nullptr;
  // pipelined host staging (all-layer calls with host buffers): copy streams and events
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  std::vector<cudaEvent_t> pipe_events;
  void* qkv_scratch = nullptr;   // fused projection: dense Q/K/V of the current call
  size_t qkv_scratch_cap = 0;
  size_t stage_cap = 0;
  void* sample_part = nullptr;   // greedy sampling: per-(row, split) partials
  size_t sample_part_cap = 0;
  int32_t* sample_cnt = nullptr; // per-row tickets (zero between launches)
  size_t sample_cnt_cap = 0;
  int64_t opt_backend = 0, opt_max_splits = 0, opt_fault = 0, opt_tc_qtiles = 0;
  int64_t opt_cluster = 0;       // SSA_OPT_CLUSTER
  int64_t opt_pdl = 1;           // SSA_OPT_PDL
  int64_t opt_cm_merge = 2;      // SSA_OPT_CM_MERGE
  int64_t opt_l2_hint = 0;       // SSA_OPT_L2_HINT
  int32_t* tickets = nullptr;    // CM merge tickets (zero between launches)
  size_t tickets_cap = 0;
  int32_t* gb_tickets = nullptr; // group-barrier counters (arrivals reset by the last arriver)
  size_t gb_tickets_cap = 0;
  int64_t opt_pipe_chunks = 0;   // SSA_OPT_PIPE_CHUNKS
  int64_t opt_qkv_debug = 0;     // SSA_OPT_QKV_DEBUG
  // Cross-stream ordering: the device work of a call waits for the previous
  // call's work when it runs on another stream (event recorded at each call's
  // end), so pages, scratch, staging and work lists are reused in call order.
  // The store's last kernel launch: its stream and whether it wrote the KV pool
  // (scatter, fused projection into pages) -- a programmatic launch right behind
  // such a grid must not read the pool before griddepcontrol.wait.
  cudaStream_t last_kernel_stream = nullptr;
  bool pool_writer_last = false;
  void note_kernel(cudaStream_t st, bool writes_pool) {
    last_kernel_stream = st;
    pool_writer_last = writes_pool;
  }
  cudaEvent_t order_ev = nullptr;
  cudaStream_t order_stream = nullptr;
  bool order_valid = false;
  ssa_status enter(cudaStream_t st);
  void leave(cudaStream_t st);
  // enter() / leave() around a public call that enqueues device work
  struct Ordered {
    ssa_store* st;
    cudaStream_t s;
    bool ok;
    Ordered(ssa_store* st_, void* s_) : st(st_), s(static_cast<cudaStream_t>(s_)) { ok = st->enter(s) == SSA_OK; }
    ~Ordered() { st->leave(s); }
  };
  ssa_stats stats{};
  int32_t ticket_seq = 0;
  int64_t last_plan_units = 0, last_plan_groups = 0, last_n_ctas = 0;
  int32_t last_cm_C = 0, last_max_split = 0, last_gbar = 0;
  bool last_used_tc = false;
  CommState* comm = nullptr;
  // SSA_OPT_TIMING
  int64_t opt_timing = 0;
  struct TimedLaunch { int kind; cudaEvent_t a, b; };
  std::vector<TimedLaunch> timed;
  std::vector<cudaEvent_t> spare_events;
  double timing_ms[SSA_TIMING_KINDS] = {};
  int64_t timing_n[SSA_TIMING_KINDS] = {};
  cudaEvent_t tick(cudaStream_t st);
  void timed_push(int kind, cudaEvent_t a, cudaEvent_t b) { timed.push_back({kind, a, b}); }
  ssa_status drain_timing();

  ~ssa_store();
  ssa_status cuda_fail(cudaError_t e, const char* what, int line);
  int64_t pad_prefix(int64_t n_prefix) const;
  int64_t slot_of(const ssa::Session& s, int64_t t) const;
  int64_t slots_for(const ssa::Session& s, int64_t n) const;
  int64_t pages_for(const ssa::Session& s, int64_t n) const;
  ssa::Session* get(ssa_session_t id);
  ssa_status reserve(ssa::Session& s, int64_t n_total, std::vector<int32_t>* got);
  void release(const std::vector<int32_t>& pages);
  ssa_status push_pages(ssa::Session& s, const std::vector<int32_t>& pages, cudaStream_t st, bool force = false);
  ssa_status upload_pages_from(ssa::Session& s, int64_t from, cudaStream_t st);
  ssa_status evict(ssa::Session& s, int64_t n, cudaStream_t st);
  ssa_status evict_for_append(ssa::Session& s, int64_t n_new, cudaStream_t st);
  int64_t pages_freed_by_evict(const ssa::Session& s, int64_t n) const;
  ssa_status retention_plan(const ssa::Session& s, int64_t n_new, int64_t* n_evict, int64_t* need_pages,
                            int64_t* freed_pages) const;
  void fill_cached(const ssa::Session& s, ssa::SegDesc* sg) const;
  ssa_status ensure_scratch(size_t part_o_floats, size_t part_lse_floats, cudaStream_t st);
  ssa_status stage_inputs(ssa::IoSet* io, cudaStream_t st);
  ssa_status query_segments(ssa::Session& s, int32_t layer, int32_t k, const int32_t* q_lens, bool include_tail,
                            std::vector<ssa::SegDesc>* segs, int64_t* total);
  ssa_status unstage_output(ssa::IoSet* io, cudaStream_t st);
  ssa_status stage_plan(ssa::IoSet* io, cudaStream_t st);   // stage_inputs without the copies
  ssa_status run_pipelined(std::vector<ssa::SegDesc>& segs, ssa::IoSet& io, int64_t rows_per_layer, int32_t n_layers,
                           bool query_plane, cudaStream_t st);
  ssa_status run(std::vector<ssa::SegDesc>& segs, const ssa::IoSet& io, int64_t rows_per_layer, int32_t layer0,
                 int32_t n_layers, int32_t in_layer_stride, bool compute_o, bool query_plane, cudaStream_t st,
                 const ssa::RunOpts& opts = ssa::RunOpts());
  bool tc_eligible(const std::vector<ssa::SegDesc>& segs) const;
  void destroy_comm();
};
