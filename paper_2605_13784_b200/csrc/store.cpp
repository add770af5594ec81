// store.cpp — host core of libssa: KV pool, deterministic page allocator,
// sessions (Region 0 / Region 1 bookkeeping, data version t), call planning
// and the C ABI of include/ssa.h.  All device work is enqueued on the
// caller's stream; no computation of attention happens on the host.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <queue>
#include <string>
#include <vector>

#include "plan.h"
#include "ssa.h"
#include "ssa_internal.h"
#include "store.h"

namespace ssa {

thread_local std::string g_last_error;

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

cudaError_t set_smem_attr_once(const void* func, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;   // (function, device)
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& d : done)
    if (d.first == func && d.second == dev) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.push_back({func, dev});
  return e;
}

// ---------------------------------------------------------------- UploadRing
UploadRing::~UploadRing() {
  for (auto& s : busy_) cudaEventDestroy(s.ev);
  for (auto e : free_events_) cudaEventDestroy(e);
  if (h_) cudaFreeHost(h_);
  if (d_) cudaFree(d_);
}

cudaError_t UploadRing::init(size_t cap) {
  cap_ = cap;
  cudaError_t e = cudaMallocHost(&h_, cap);
  if (e != cudaSuccess) return e;
  return cudaMalloc(&d_, cap);
}

cudaError_t UploadRing::retire_overlapping(size_t lo, size_t hi) {
  while (!busy_.empty()) {
    Span& f = busy_.front();
    if (f.hi <= lo || f.lo >= hi) break;
    cudaError_t e = cudaEventSynchronize(f.ev);
    if (e != cudaSuccess) return e;
    free_events_.push_back(f.ev);
    busy_.pop_front();
  }
  return cudaSuccess;
}

size_t UploadRing::alloc(size_t n) {
  n = (n + 255) & ~size_t(255);
  if (n > cap_) return SIZE_MAX;
  if (head_ + n > cap_) head_ = 0;
  // Retire every older span that overlaps [head_, head_+n) (in ring order).
  while (!busy_.empty()) {
    bool overlap = false;
    for (auto& s : busy_)
      if (!(s.hi <= head_ || s.lo >= head_ + n)) { overlap = true; break; }
    if (!overlap) break;
    Span f = busy_.front();
    if (cudaEventSynchronize(f.ev) != cudaSuccess) return SIZE_MAX;
    free_events_.push_back(f.ev);
    busy_.pop_front();
  }
  const size_t off = head_;
  head_ += n;
  return off;
}

cudaError_t UploadRing::fence(size_t lo, size_t hi, cudaStream_t s) {
  cudaEvent_t ev;
  if (!free_events_.empty()) {
    ev = free_events_.back();
    free_events_.pop_back();
  } else {
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = cudaEventRecord(ev, s);
  if (e != cudaSuccess) return e;
  busy_.push_back({lo, hi, ev});
  return cudaSuccess;
}

}  // namespace ssa

using namespace ssa;

// ============================================================================
// helpers
// ============================================================================
#define SSA_CHECK_STORE(st)                                       \
  do {                                                            \
    if (!(st)) { set_error("null store"); return SSA_ERR_INVALID_ARG; } \
    if ((st)->failed) { set_error("store failed earlier: %s", (st)->fail_msg.c_str()); return SSA_ERR_STATE; } \
  } while (0)

#define SSA_CUDA(st, expr)                                                   \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess) return (st)->cuda_fail(_e, #expr, __LINE__);      \
  } while (0)

ssa_status ssa_store::cuda_fail(cudaError_t e, const char* what, int line) {
  failed = true;
  char buf[512];
  snprintf(buf, sizeof(buf), "CUDA error %s (%s) at store.cpp:%d in %s", cudaGetErrorName(e),
           cudaGetErrorString(e), line, what);
  fail_msg = buf;
  set_error("%s", buf);
  return SSA_ERR_CUDA;
}

static int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

cudaEvent_t ssa_store::tick(cudaStream_t st) {
  if (!opt_timing) return nullptr;
  cudaEvent_t e = nullptr;
  if (!spare_events.empty()) {
    e = spare_events.back();
    spare_events.pop_back();
  } else if (cudaEventCreate(&e) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  cudaEventRecord(e, st);
  return e;
}

ssa_status ssa_store::drain_timing() {
  for (auto& t : timed) {
    if (t.a && t.b) {
      SSA_CUDA(this, cudaEventSynchronize(t.b));
      float ms = 0.f;
      SSA_CUDA(this, cudaEventElapsedTime(&ms, t.a, t.b));
      timing_ms[t.kind] += ms;
      timing_n[t.kind] += 1;
    }
    if (t.a) spare_events.push_back(t.a);
    if (t.b) spare_events.push_back(t.b);
  }
  timed.clear();
  return SSA_OK;
}

int64_t ssa_store::pad_prefix(int64_t n_prefix) const { return ceil_div64(n_prefix, cfg.page_size) * cfg.page_size; }

// Planner cost of a split tcgen05 unit beyond its tiles (the partial write,
// the merge, and the CTA prologue a longer unit would amortise), in K/V tiles.
#ifndef SSA_TC_SPLIT_OVERHEAD
#define SSA_TC_SPLIT_OVERHEAD 4.0
#endif
static constexpr double kTcSplitOverheadTiles = SSA_TC_SPLIT_OVERHEAD;

// Slot of retained token t of a session (reading R-9: R0 padded to a page
// boundary; R-8: R1 tokens evicted from the front leave r1_skip empty slots
// at the start of the first retained R1 page).
int64_t ssa_store::slot_of(const Session& s, int64_t t) const {
  return t < s.n_prefix ? t : pad_prefix(s.n_prefix) + s.r1_skip + (t - s.n_prefix);
}
int64_t ssa_store::slots_for(const Session& s, int64_t n) const {
  return n <= s.n_prefix ? n : pad_prefix(s.n_prefix) + s.r1_skip + (n - s.n_prefix);
}
int64_t ssa_store::pages_for(const Session& s, int64_t n) const {
  return ceil_div64(slots_for(s, n), cfg.page_size);
}

Session* ssa_store::get(ssa_session_t id) {
  if (id < 0 || id >= (int)sessions.size() || !sessions[id].live) return nullptr;
  return &sessions[id];
}

// Reserve pages so that the session can hold n_total tokens; all-or-none.
ssa_status ssa_store::reserve(Session& s, int64_t n_total, std::vector<int32_t>* got) {
  const int64_t need = pages_for(s, n_total) - (int64_t)s.pages.size();
  got->clear();
  if (need <= 0) return SSA_OK;
  if (need > (int64_t)free_pages.size()) {
    set_error("pool exhausted: need %lld pages, %zu free", (long long)need, free_pages.size());
    return SSA_ERR_POOL_EXHAUSTED;
  }
  for (int64_t i = 0; i < need; ++i) {
    got->push_back(free_pages.top());
    page_ref[free_pages.top()] = 1;
    free_pages.pop();
  }
  stats.pages_reserved += need;
  return SSA_OK;
}

// Drop one reference per page; a page returns to the free list when its last
// referer (donor or alias, SPEC kv-store design decision) releases it.
void ssa_store::release(const std::vector<int32_t>& pages) {
  for (int32_t p : pages)
    if (--page_ref[p] == 0) free_pages.push(p);
}

// Re-upload the device page table from entry `from` (after entries shifted).
ssa_status ssa_store::upload_pages_from(Session& s, int64_t from, cudaStream_t st) {
  s.d_valid = std::min<int64_t>(s.d_valid, from);
  std::vector<int32_t> none;
  const int64_t n = (int64_t)s.pages.size();
  if (s.d_valid >= n) return SSA_OK;
  // push_pages uploads [min(old, d_valid), n) where old = n: i.e. [d_valid, n)
  return push_pages(s, none, st, true);
}

// Region-1 FIFO eviction of the n oldest retained R1 tokens (Alg. 1
// L279-281; R0 frozen).  Host metadata + page-table upload on `st`.
ssa_status ssa_store::evict(Session& s, int64_t n, cudaStream_t st) {
  if (n <= 0) return SSA_OK;
  const int64_t P = cfg.page_size;
  const int64_t r0_pages = pad_prefix(s.n_prefix) / P;
  s.r1_skip += n;
  s.n_tokens -= n;
  s.n_evicted += n;
  int64_t drop = s.r1_skip / P;
  if (s.n_tokens == s.n_prefix) drop = (int64_t)s.pages.size() - r0_pages;   // R1 empty: release all its pages
  std::vector<int32_t> gone(s.pages.begin() + r0_pages, s.pages.begin() + r0_pages + drop);
  s.pages.erase(s.pages.begin() + r0_pages, s.pages.begin() + r0_pages + drop);
  s.r1_skip = s.n_tokens == s.n_prefix ? 0 : s.r1_skip - drop * P;
  release(gone);
  s.version += 1;
  return upload_pages_from(s, r0_pages, st);
}

// Pages the eviction of n R1 tokens would return to the free list (the
// pages it drops that no alias still references).
int64_t ssa_store::pages_freed_by_evict(const Session& s, int64_t n) const {
  if (n <= 0) return 0;
  const int64_t P = cfg.page_size;
  const int64_t r0_pages = pad_prefix(s.n_prefix) / P;
  int64_t drop = (s.r1_skip + n) / P;
  if (s.n_tokens - n == s.n_prefix) drop = (int64_t)s.pages.size() - r0_pages;
  int64_t freed = 0;
  for (int64_t i = 0; i < drop; ++i) freed += page_ref[s.pages[r0_pages + i]] == 1;
  return freed;
}

// The retention guard of Alg. 1: if the session would exceed its
// retention, evict |tokens| oldest R1 tokens first.  Computes, without
// changing state, how many tokens that evicts, how many new pages the append
// then needs and how many pages the eviction returns to the free list.
ssa_status ssa_store::retention_plan(const Session& s, int64_t n_new, int64_t* n_evict, int64_t* need_pages,
                                     int64_t* freed_pages) const {
  *n_evict = 0;
  if (s.retention > 0 && s.n_tokens + n_new > s.retention) {
    if (n_new > s.n_tokens - s.n_prefix) {
      set_error("retention: %lld new tokens but only %lld evictable Region-1 tokens", (long long)n_new,
                (long long)(s.n_tokens - s.n_prefix));
      return SSA_ERR_INVALID_ARG;
    }
    *n_evict = n_new;
  }
  Session after = s;
  after.pages.clear();
  const int64_t P = cfg.page_size;
  const int64_t r0_pages = pad_prefix(s.n_prefix) / P;
  int64_t drop = 0;
  if (*n_evict > 0) {
    drop = (s.r1_skip + *n_evict) / P;
    after.r1_skip = s.r1_skip + *n_evict - drop * P;
    after.n_tokens = s.n_tokens - *n_evict;
    if (after.n_tokens == s.n_prefix) {
      drop = (int64_t)s.pages.size() - r0_pages;
      after.r1_skip = 0;
    }
  }
  *need_pages = std::max<int64_t>(0, pages_for(after, after.n_tokens + n_new) - ((int64_t)s.pages.size() - drop));
  *freed_pages = pages_freed_by_evict(s, *n_evict);
  return SSA_OK;
}

// Apply the retention guard before an append of n_new tokens: all-or-none
// (fails without state change if the eviction or the append cannot happen).
ssa_status ssa_store::evict_for_append(Session& s, int64_t n_new, cudaStream_t st) {
  int64_t n_ev = 0, need = 0, freed = 0;
  ssa_status rc = retention_plan(s, n_new, &n_ev, &need, &freed);
  if (rc != SSA_OK) return rc;
  if (need > (int64_t)free_pages.size() + freed) {
    set_error("pool exhausted: need %lld pages, %zu free", (long long)need, free_pages.size());
    return SSA_ERR_POOL_EXHAUSTED;
  }
  return n_ev ? evict(s, n_ev, st) : SSA_OK;
}

// Append page ids to the session's host table and upload the delta.
ssa_status ssa_store::push_pages(Session& s, const std::vector<int32_t>& pages, cudaStream_t st, bool force) {
  if (pages.empty() && !force) return SSA_OK;
  const int64_t old = (int64_t)s.pages.size();
  s.pages.insert(s.pages.end(), pages.begin(), pages.end());
  const int64_t n = (int64_t)s.pages.size();
  if (n > s.d_cap) {
    int64_t cap = std::max<int64_t>(64, s.d_cap);
    while (cap < n) cap *= 2;
    int32_t* nd = nullptr;
    SSA_CUDA(this, cudaMallocAsync((void**)&nd, cap * sizeof(int32_t), st));
    if (s.d_pages) {
      SSA_CUDA(this, cudaMemcpyAsync(nd, s.d_pages, s.d_valid * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
      SSA_CUDA(this, cudaFreeAsync(s.d_pages, st));
    }
    s.d_pages = nd;
    s.d_cap = cap;
  }
  // Entries [min(old, d_valid), n) are (re)uploaded: truncate may have lowered d_valid.
  const int64_t lo = std::min<int64_t>(old, s.d_valid);
  const size_t bytes = (n - lo) * sizeof(int32_t);
  const size_t off = ring.alloc(bytes);
  if (off == SIZE_MAX) return cuda_fail(cudaErrorMemoryAllocation, "ring.alloc(page table)", __LINE__);
  memcpy(ring.host(off), s.pages.data() + lo, bytes);
  SSA_CUDA(this, cudaMemcpyAsync(s.d_pages + lo, ring.host(off), bytes, cudaMemcpyHostToDevice, st));
  SSA_CUDA(this, ring.fence(off, off + bytes, st));
  s.d_valid = n;
  return SSA_OK;
}

void ssa_store::fill_cached(const Session& s, SegDesc* sg) const {
  sg->n_slots = (int32_t)slots_for(s, s.n_tokens);
  if (s.n_tokens > s.n_prefix) {
    // one hole: R0's page pad and the evicted head of the first R1 page
    sg->hole_lo = (int32_t)s.n_prefix;
    sg->hole_hi = (int32_t)(pad_prefix(s.n_prefix) + s.r1_skip);
  } else {
    sg->hole_lo = sg->hole_hi = 0;
  }
  sg->pages = s.d_pages;
  sg->n_pages = (int32_t)s.pages.size();
}

static bool capturing(void* stream);

// Scratch grows in stream order (cudaMallocAsync / cudaFreeAsync on the call's
// stream): earlier calls on other streams are ordered before it by enter().
ssa_status ssa_store::ensure_scratch(size_t part_o_floats, size_t part_lse_floats, cudaStream_t st) {
  if (part_o_floats > part_o_cap || part_lse_floats > part_lse_cap) {
    if (capturing(st)) {
      ssa::set_error("CUDA-graph capture: warm up the call once before capturing (split-KV scratch)");
      return SSA_ERR_STATE;
    }
    if (part_o) SSA_CUDA(this, cudaFreeAsync(part_o, st));
    if (part_lse) SSA_CUDA(this, cudaFreeAsync(part_lse, st));
    part_o = nullptr;
    part_lse = nullptr;
    part_o_cap = std::max(part_o_floats, part_o_cap * 2);
    part_lse_cap = std::max(part_lse_floats, part_lse_cap * 2);
    SSA_CUDA(this, cudaMallocAsync(reinterpret_cast<void**>(&part_o), part_o_cap * sizeof(float), st));
    SSA_CUDA(this, cudaMallocAsync(reinterpret_cast<void**>(&part_lse), part_lse_cap * sizeof(float), st));
  }
  return SSA_OK;
}

// Cross-stream ordering of the store's device work (one dispatch order).
ssa_status ssa_store::enter(cudaStream_t st) {
  if (capturing(st)) return SSA_OK;
  if (order_valid && st != order_stream) SSA_CUDA(this, cudaStreamWaitEvent(st, order_ev, 0));
  return SSA_OK;
}
void ssa_store::leave(cudaStream_t st) {
  if (capturing(st) || failed) return;
  if (!order_ev && cudaEventCreateWithFlags(&order_ev, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  if (cudaEventRecord(order_ev, st) == cudaSuccess) {
    order_stream = st;
    order_valid = true;
  } else {
    cudaGetLastError();
  }
}

// --------------------------------------------------------------- staging
static bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// cudaPointerGetAttributes is not allowed while a stream is being captured into
// a CUDA graph (it invalidates a global-mode capture); captured calls must pass
// device pointers anyway.
static bool capturing(void* stream) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing((cudaStream_t)stream, &cs) != cudaSuccess) { cudaGetLastError(); return false; }
  return cs != cudaStreamCaptureStatusNone;
}

ssa_status ssa_store::stage_inputs(IoSet* io, cudaStream_t st) {
  ssa_status rc = stage_plan(io, st);
  if (rc != SSA_OK) return rc;
  for (IoBuf* b : {&io->q, &io->k, &io->v}) {
    if (!b->host) continue;
    SSA_CUDA(this, cudaMemcpyAsync(b->dev, b->host, b->bytes, cudaMemcpyHostToDevice, st));
    stats.h2d_bytes += (int64_t)b->bytes;
  }
  return SSA_OK;
}

ssa_status ssa_store::stage_plan(IoSet* io, cudaStream_t st) {
  // Place every host pointer of the call in one device staging buffer.  A call
  // being captured into a CUDA graph must pass device pointers (pointer queries
  // would invalidate a global-mode capture), so they are taken as such.
  const bool cap = capturing(st);
  size_t need = 0;
  auto plan_one = [&](IoBuf& b) {
    b.dev = nullptr;
    b.host = nullptr;
    if (!b.user || b.bytes == 0) return;
    if (cap || is_device_ptr(b.user)) { b.dev = const_cast<void*>(b.user); return; }
    b.host = const_cast<void*>(b.user);
    b.stage_off = need;
    need += (b.bytes + 255) & ~size_t(255);
  };
  plan_one(io->q); plan_one(io->k); plan_one(io->v); plan_one(io->o);
  if (need > stage_cap) {
    if (stage) SSA_CUDA(this, cudaFreeAsync(stage, st));
    stage = nullptr;
    stage_cap = std::max(need, stage_cap * 2);
    SSA_CUDA(this, cudaMallocAsync(&stage, stage_cap, st));
  }
  for (IoBuf* b : {&io->q, &io->k, &io->v, &io->o})
    if (b->host) b->dev = static_cast<char*>(stage) + b->stage_off;
  return SSA_OK;
}

// All-layer call with host buffers: the layers run in chunks so that the
// host->device copy of chunk c+1 (h2d_stream) and the device->host copy of
// chunk c-1's O (d2h_stream) overlap chunk c's kernels on the call's stream.
// The call's stream waits for the last O copy, so "synchronize `stream`, then
// read O" still holds.
ssa_status ssa_store::run_pipelined(std::vector<SegDesc>& segs, IoSet& io, int64_t rows_per_layer, int32_t n_layers,
                                    bool query_plane, cudaStream_t st) {
  ssa_status rc = stage_plan(&io, st);
  if (rc != SSA_OK) return rc;
  // 2 chunks measured best on the 32-layer 32k query (1.01 vs 1.09 ms unpipelined;
  // 4 and 8 chunks were slower: smaller launches, more per-chunk overhead)
  int chunks = std::min(opt_pipe_chunks > 0 ? (int)opt_pipe_chunks : 2, n_layers);
  if (!h2d_stream) {
    SSA_CUDA(this, cudaStreamCreateWithFlags(&h2d_stream, cudaStreamNonBlocking));
    SSA_CUDA(this, cudaStreamCreateWithFlags(&d2h_stream, cudaStreamNonBlocking));
  }
  while ((int)pipe_events.size() < 2 * chunks + 2) {
    cudaEvent_t e;
    SSA_CUDA(this, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    pipe_events.push_back(e);
  }
  cudaEvent_t ev_start = pipe_events[0], ev_end = pipe_events[1];
  // the staging buffer may still be in use by earlier work on `st`
  SSA_CUDA(this, cudaEventRecord(ev_start, st));
  SSA_CUDA(this, cudaStreamWaitEvent(h2d_stream, ev_start, 0));
  SSA_CUDA(this, cudaStreamWaitEvent(d2h_stream, ev_start, 0));
  for (int c = 0; c < chunks; ++c) {
    const int32_t l0 = (int32_t)((int64_t)c * n_layers / chunks), l1 = (int32_t)((int64_t)(c + 1) * n_layers / chunks);
    IoSet ioc = io;
    for (IoBuf* b : {&ioc.q, &ioc.k, &ioc.v, &ioc.o}) {
      if (!b->dev) continue;
      const size_t per_layer = b->bytes / n_layers;
      b->dev = static_cast<char*>(b->dev) + per_layer * l0;
      if (b->host) b->host = static_cast<char*>(b->host) + per_layer * l0;
      b->bytes = per_layer * (l1 - l0);
      if (b != &ioc.o && b->host) {
        SSA_CUDA(this, cudaMemcpyAsync(b->dev, b->host, b->bytes, cudaMemcpyHostToDevice, h2d_stream));
        stats.h2d_bytes += (int64_t)b->bytes;
      }
    }
    cudaEvent_t ev_in = pipe_events[2 + 2 * c], ev_out = pipe_events[3 + 2 * c];
    SSA_CUDA(this, cudaEventRecord(ev_in, h2d_stream));
    SSA_CUDA(this, cudaStreamWaitEvent(st, ev_in, 0));
    if ((rc = run(segs, ioc, rows_per_layer, l0, l1 - l0, 1, true, query_plane, st)) != SSA_OK) return rc;
    if (ioc.o.host) {
      SSA_CUDA(this, cudaEventRecord(ev_out, st));
      SSA_CUDA(this, cudaStreamWaitEvent(d2h_stream, ev_out, 0));
      SSA_CUDA(this, cudaMemcpyAsync(ioc.o.host, ioc.o.dev, ioc.o.bytes, cudaMemcpyDeviceToHost, d2h_stream));
      stats.d2h_bytes += (int64_t)ioc.o.bytes;
    }
  }
  SSA_CUDA(this, cudaEventRecord(ev_end, d2h_stream));
  SSA_CUDA(this, cudaStreamWaitEvent(st, ev_end, 0));
  return SSA_OK;
}

ssa_status ssa_store::unstage_output(IoSet* io, cudaStream_t st) {
  if (io->o.host) {
    SSA_CUDA(this, cudaMemcpyAsync(io->o.host, io->o.dev, io->o.bytes, cudaMemcpyDeviceToHost, st));
    stats.d2h_bytes += (int64_t)io->o.bytes;
  }
  return SSA_OK;
}

// --------------------------------------------------------------- one launch
// Cluster size of a CM plan for a single-layer tcgen05 launch (kernels_tc.cu
// "CM"): the planner is run for C in 1..8 and 16 (or the forced SSA_OPT_CLUSTER
// size) against the device's co-resident cluster count and the cheapest plan wins.
int ssa_store::max_clusters(int C) {
  if (C < 1 || C > 16) return 0;
  if (max_clusters_[kv_fp8][C] < 0) {
    const int n = C == 1 ? num_sms : tc_max_active_clusters(C, kv_fp8);
    max_clusters_[kv_fp8][C] = n > 0 ? n : 0;
  }
  return max_clusters_[kv_fp8][C];
}

// Runs KA (scatter of appended segments) and the attention kernels for `segs`
// over input layers [0, n_layers) mapped to pool layers layer0 + y.
//
// Work lists (segments, units, groups, CTA pairs, scatter segments) are a pure
// function of the call shape; the store keeps the device copy of the last 16
// shapes' lists, so a repeated call (per-layer queries, the steps of a session,
// Flash Query cycles) launches with no planning and no host->device copy.
ssa_status ssa_store::run(std::vector<SegDesc>& segs, const IoSet& io, int64_t rows_per_layer,
                          int32_t layer0, int32_t n_layers, int32_t in_layer_stride, bool compute_o,
                          bool query_plane, cudaStream_t st, const RunOpts& opts) {
  const int G = cfg.num_q_heads / cfg.num_kv_heads;
  const int D = cfg.head_dim;
  const bool use_tc = compute_o && tc_eligible(segs);
  if (kv_fp8 && compute_o && !use_tc) {
    ssa::set_error("E4M3 KV cache: attention needs the tcgen05 path (sm_100, default backend)");
    return SSA_ERR_UNSUPPORTED;
  }
  // sharded partial outputs (fp32 O / lse / peer push) go through the combine kernel
  const bool special = opts.force_groups || opts.o_f32 || opts.lse_out || opts.n_peers > 0;
  const bool cm = use_tc && !special;
  const bool cap = capturing(st);
  // ---- cache key: every input of the planner and of the uploaded lists
  std::vector<int64_t> key = {compute_o, use_tc, cm, opt_cluster, opt_cm_merge, n_layers, opt_max_splits, opt_fault,
                              opts.force_groups, (int64_t)segs.size()};
  for (const SegDesc& sg : segs)
    key.insert(key.end(), {sg.row0, sg.m, sg.tail_m, sg.n_slots, sg.hole_lo, sg.hole_hi, sg.append_slot0,
                           sg.n_pages, (int64_t)(uintptr_t)sg.pages});
  PlanCacheEntry* ent = nullptr;
  for (size_t e = 0; e < plan_cache.size(); ++e)
    if (plan_cache[e].key == key) {
      ent = &plan_cache[e];
      ent->last_use = ++plan_clock;
      ++plan_cache_hits;
      break;
    }
  PlanCacheEntry fresh;
  if (!ent) {
    fresh.key = std::move(key);
    Plan& plan = fresh.plan;
    if (compute_o) {
      PlanConfig pc;
      pc.Hkv = cfg.num_kv_heads;
      pc.key_tile = use_tc ? tc_key_tile() : simt_key_tile();
      pc.q_tile_tokens = std::max(1, (use_tc ? tc_rows_tile() : simt_rows_tile(G, D)) / G);
      pc.n_layers = n_layers;
      pc.num_sms = num_sms;
      pc.ctas_per_sm = 2;   // SIMT: 2 CTAs/SM; tcgen05: 2 slots per CTA
      pc.max_splits = (int)opt_max_splits;
      pc.min_tiles_per_unit = 2;
      pc.unit_overhead_tiles = use_tc ? 2.0 : 1.0;
      pc.split_overhead_tiles = use_tc ? kTcSplitOverheadTiles : 1.0;
      pc.fault = (int)opt_fault;
      pc.force_groups = opts.force_groups;
      pc.pair_slots = use_tc;
      fresh.cm_C = 0;
      if (cm && n_layers == 1 && opt_cluster >= 0) {
        double best = -1.0;
        // candidates: clusters of C CTAs (DSMEM merge + merge kernel for groups over
        // several clusters), and the group-barrier merge (C = 1, one wave, gm_reduce)
        // (the group plan, when it applies, is taken without comparing costs: measured
        // faster on the per-layer query; its groups are merged by gm_merge_kernel right
        // behind the attention grid (SSA_OPT_CM_MERGE 2 / 3: the next layer's CTAs take
        // the SMs while it runs; 30.7 / 33.0 vs 32.3 / 33.6 us/layer for the 1- / 32-token
        // query with the in-kernel group barrier, 4 / 5).  The per-layer append (SHARED
        // pairs) is faster on the cluster plans: 141-143 vs 148 us/layer,
        // scripts/append_ab.py)
        for (int C : {0, 1, 2, 3, 4, 5, 6, 7, 8, 16}) {
          const bool gb = C == 0;
          // SSA_OPT_CM_MERGE 2 / 4: query plane only; 3 / 5: both planes
          if (gb && (opt_cm_merge < 2 || opt_cluster > 0 || ((opt_cm_merge == 2 || opt_cm_merge == 4) && !query_plane)))
            continue;
          if (!gb && fresh.gbar) break;
          const int Ck = gb ? 1 : C;
          if (opt_cluster > 0 && Ck != opt_cluster) continue;
          Plan pl;
          std::vector<TcPair> prs;
          const double cost = plan_cm(segs, pc, Ck, max_clusters(Ck), &pl, &prs, gb);
          if (cost >= 0.0 && (best < 0.0 || cost < best)) {
            best = cost;
            plan = std::move(pl);
            fresh.pairs = std::move(prs);
            fresh.cm_C = Ck;
            fresh.gbar = gb;
            fresh.gsplit = gb && (opt_cm_merge == 2 || opt_cm_merge == 3);
          }
        }
      }
      if (fresh.cm_C == 0) {
        plan_units(segs, pc, &plan);
        if (use_tc) pair_units(segs, plan, pc.key_tile, &fresh.pairs);
        if (cm) {
          cm_regroup(&plan, fresh.pairs);
          fresh.cm_C = 1;
        }
      }
      for (auto& g : plan.groups) fresh.max_split = std::max(fresh.max_split, g.n_splits);
      // per-CTA copies of the units, segments and group split counts (TcPair)
      for (TcPair& pr : fresh.pairs) {
        pr.wa = plan.units[pr.ua];
        pr.wb = pr.ub >= 0 ? plan.units[pr.ub] : pr.wa;
        pr.sa = segs[pr.wa.seg];
        pr.sb = segs[pr.wb.seg];
        pr.splits_a = pr.wa.group >= 0 ? plan.groups[pr.wa.group].n_splits : 0;
        pr.splits_b = pr.wb.group >= 0 ? plan.groups[pr.wb.group].n_splits : 0;
        pr.unit0_a = pr.wa.group >= 0 ? plan.groups[pr.wa.group].unit0 : 0;
        pr.unit0_b = pr.wb.group >= 0 ? plan.groups[pr.wb.group].unit0 : 0;
      }
      // L2 evict-first pays only when no key tile of the launch is read twice: one q-tile
      // group per (cached pool, KV head) -- not appends, multi-tile queries or Flash batches
      {
        std::vector<std::pair<const int32_t*, int>> seen;
        bool once = !plan.groups.empty();
        for (auto& g : plan.groups) {
          const std::pair<const int32_t*, int> kk{segs[g.seg].pages, g.kv_head};
          if (std::find(seen.begin(), seen.end(), kk) != seen.end()) { once = false; break; }
          seen.push_back(kk);
        }
        fresh.l2_hint = once;
      }
    }
    // ---- host image of the lists: segments, units, groups, scatter segments + prefix, CTA pairs
    std::vector<SegDesc> app_segs;
    std::vector<int32_t> prefix(1, 0);
    for (const SegDesc& sg : segs)
      if (sg.append_slot0 >= 0) {
        app_segs.push_back(sg);
        prefix.push_back(prefix.back() + sg.m);
      }
    fresh.n_app = (int32_t)app_segs.size();
    fresh.app_tokens = prefix.back();
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    const std::pair<const void*, size_t> parts[6] = {
        {segs.data(), segs.size() * sizeof(SegDesc)},
        {plan.units.data(), plan.units.size() * sizeof(WorkUnit)},
        {plan.groups.data(), plan.groups.size() * sizeof(Group)},
        {app_segs.data(), app_segs.size() * sizeof(SegDesc)},
        {prefix.data(), prefix.size() * sizeof(int32_t)},
        {fresh.pairs.data(), fresh.pairs.size() * sizeof(TcPair)}};
    size_t total = 0;
    for (int i = 0; i < 6; ++i) {
      fresh.off[i] = total;
      total += al(parts[i].second);
    }
    fresh.bytes = total;
    fresh.image.resize(total);
    for (int i = 0; i < 6; ++i)
      if (parts[i].second) memcpy(fresh.image.data() + fresh.off[i], parts[i].first, parts[i].second);
    // ---- device copy: the graph arena for a call being captured (the captured copy
    // node writes it at every replay; not cached), else a cached allocation
    if (cap) {
      if (arena_used + total > arena_cap) {
        ssa::set_error("CUDA-graph capture: graph arena exhausted (%zu of %zu bytes used)", arena_used, arena_cap);
        return SSA_ERR_STATE;
      }
      memcpy(arena_h + arena_used, fresh.image.data(), total);
      SSA_CUDA(this, cudaMemcpyAsync(arena_d + arena_used, arena_h + arena_used, total, cudaMemcpyHostToDevice, st));
      fresh.dev = arena_d + arena_used;
      arena_used += total;
    } else {
      const size_t off = ring.alloc(total);
      if (off == SIZE_MAX) return cuda_fail(cudaErrorMemoryAllocation, "ring.alloc(work list)", __LINE__);
      memcpy(ring.host(off), fresh.image.data(), total);
      SSA_CUDA(this, cudaMallocAsync(reinterpret_cast<void**>(&fresh.dev), total, st));
      SSA_CUDA(this, cudaMemcpyAsync(fresh.dev, ring.host(off), total, cudaMemcpyHostToDevice, st));
      SSA_CUDA(this, ring.fence(off, off + total, st));
      // evict the least recently used unpinned entry beyond 16 (freed in stream order)
      int n_unpinned = 0, lru = -1;
      for (size_t e = 0; e < plan_cache.size(); ++e)
        if (!plan_cache[e].pinned) {
          ++n_unpinned;
          if (lru < 0 || plan_cache[e].last_use < plan_cache[lru].last_use) lru = (int)e;
        }
      if (n_unpinned >= 16 && lru >= 0) {
        SSA_CUDA(this, cudaFreeAsync(plan_cache[lru].dev, st));
        plan_cache.erase(plan_cache.begin() + lru);
      }
      fresh.last_use = ++plan_clock;
      plan_cache.push_back(std::move(fresh));
      ent = &plan_cache.back();
    }
    stats.plan_uploads += 1;
  } else if (cap) {
    ent->pinned = true;   // a captured graph reads this entry's device copy at every replay
  }
  const PlanCacheEntry& E = ent ? *ent : fresh;
  const Plan& plan = E.plan;
  const auto d_segs = reinterpret_cast<const SegDesc*>(E.dev + E.off[0]);
  const auto d_units = reinterpret_cast<const WorkUnit*>(E.dev + E.off[1]);
  const auto d_groups = reinterpret_cast<const Group*>(E.dev + E.off[2]);
  const auto d_app = reinterpret_cast<const SegDesc*>(E.dev + E.off[3]);
  const auto d_pre = reinterpret_cast<const int32_t*>(E.dev + E.off[4]);
  const auto d_pairs = reinterpret_cast<const TcPair*>(E.dev + E.off[5]);
  if (cap && opt_timing) {
    ssa::set_error("CUDA-graph capture: not with SSA_OPT_TIMING");
    return SSA_ERR_STATE;
  }

  // ---- E4M3 KV (R-22): codes of the call's K/V, the tails' and the scatter's source
  const void* k_src = io.k.dev;
  const void* v_src = io.v.dev;
  if (kv_fp8 && io.k.dev && (compute_o || (E.n_app > 0 && !opts.skip_scatter))) {
    QuantParams qp{};
    qp.n = (int64_t)(in_layer_stride ? n_layers : 1) * rows_per_layer * cfg.num_kv_heads * D;
    if ((size_t)(2 * qp.n) > kv8_cap) {
      if (cap) { ssa::set_error("CUDA-graph capture: warm up the call once before capturing (E4M3 scratch)"); return SSA_ERR_STATE; }
      if (kv8) SSA_CUDA(this, cudaFreeAsync(kv8, st));
      kv8 = nullptr;
      kv8_cap = std::max((size_t)(2 * qp.n), 2 * kv8_cap);
      SSA_CUDA(this, cudaMallocAsync(reinterpret_cast<void**>(&kv8), kv8_cap, st));
    }
    qp.K = io.k.dev;
    qp.V = io.v.dev;
    qp.K8 = kv8;
    qp.V8 = kv8 + qp.n;
    qp.k_scale = cfg.k_scale;
    qp.v_scale = cfg.v_scale;
    cudaEvent_t t0 = tick(st);
    SSA_CUDA(this, launch_quant_e4m3(qp, st));
    note_kernel(st, false);
    if (t0) timed_push(6, t0, tick(st));
    stats.kernel_launches++;
    k_src = qp.K8;
    v_src = qp.V8;
  }

  // ---- KA: scatter new K/V into pages
  if (E.n_app > 0 && !opts.skip_scatter) {
    ScatterParams sp{};
    sp.K = k_src;
    sp.V = v_src;
    sp.rows_per_layer = rows_per_layer;
    sp.layer0 = layer0;
    sp.in_layer_stride = in_layer_stride;
    sp.poolK = poolK;
    sp.poolV = poolV;
    sp.num_pages = cfg.num_pages;
    sp.Hkv = cfg.num_kv_heads;
    sp.D = D;
    sp.P = cfg.page_size;
    sp.elem_bytes = pelem;
    sp.segs = d_app;
    sp.tok_prefix = d_pre;
    sp.n_segs = E.n_app;
    sp.total_tokens = E.app_tokens;
    cudaEvent_t t0 = tick(st);
    SSA_CUDA(this, launch_scatter(sp, n_layers, st));
    if (t0) timed_push(4, t0, tick(st));
    stats.kernel_launches++;
    note_kernel(st, true);
  }
  // ---- attention (+ combine)
  if (compute_o && !plan.units.empty()) {
    const int rows_tile = use_tc ? tc_rows_tile() : simt_rows_tile(G, D);
    const bool combine = !plan.groups.empty() && E.cm_C == 0;
    const bool partials = combine || E.max_split > 1;
    if (partials) {
      const size_t n_po = (size_t)n_layers * plan.units.size() * rows_tile * D;
      const size_t n_pl = (size_t)n_layers * plan.units.size() * rows_tile;
      ssa_status s = ensure_scratch(n_po, n_pl, st);
      if (s != SSA_OK) return s;
    }
    AttnParams ap{};
    ap.Q = io.q.dev;
    ap.Kt = k_src;
    ap.Vt = v_src;
    ap.O = io.o.dev;
    ap.rows_per_layer = rows_per_layer;
    ap.layer0 = layer0;
    ap.in_layer_stride = in_layer_stride;
    ap.poolK = poolK;
    ap.poolV = poolV;
    ap.num_pages = cfg.num_pages;
    ap.Hq = cfg.num_q_heads;
    ap.Hkv = cfg.num_kv_heads;
    ap.D = D;
    ap.P = cfg.page_size;
    ap.G = G;
    ap.scale_log2 = scale * 1.4426950408889634f * (kv_fp8 ? cfg.k_scale : 1.f);
    ap.kv_fp8 = kv_fp8 ? 1 : 0;
    ap.o_scale = kv_fp8 ? cfg.v_scale : 1.f;
    ap.segs = d_segs;
    ap.units = d_units;
    ap.n_units = (int32_t)plan.units.size();
    ap.groups = d_groups;
    ap.n_groups = (int32_t)plan.groups.size();
    ap.part_o = part_o;
    ap.part_lse = part_lse;
    ap.rows_tile = rows_tile;
    ap.key_tile = use_tc ? tc_key_tile() : simt_key_tile();
    ap.fault = (int32_t)opt_fault;
    ap.pairs = d_pairs;
    ap.n_pairs = (int32_t)E.pairs.size();
    ap.cm_C = E.cm_C;
    // pool tiles may be prefetched before griddepcontrol.wait unless the grid right
    // before this one on the stream is one of the store's pool writers
    ap.pool_early = (opt_pdl != 0 && !opt_timing && !(pool_writer_last && last_kernel_stream == st)) ? 1 : 0;
    ap.l2_evict_first = opt_l2_hint == 2 || (opt_l2_hint == 0 && E.l2_hint) ? 1 : 0;
    const bool gsplit = E.gsplit && E.max_split > 1;
    const bool gbar = E.gbar && !E.gsplit && E.max_split > 1;
    const bool merge_in_kernel = E.cm_C > 0 && E.max_split > 1 && (opt_cm_merge == 0 || gbar);
    ap.cm_gbar = gbar ? 1 : 0;
    ap.cm_gsplit = gsplit ? 1 : 0;
    if (merge_in_kernel) {
      // zeroed counters: [layers][groups][C] tickets, or [layers][groups][2] group barriers
      int32_t*& buf = gbar ? gb_tickets : tickets;
      size_t& buf_cap = gbar ? gb_tickets_cap : tickets_cap;
      const size_t need = (size_t)n_layers * plan.groups.size() * (gbar ? 2 : E.cm_C);
      if (need > buf_cap) {
        if (cap) { ssa::set_error("CUDA-graph capture: warm up the call once before capturing (merge tickets)"); return SSA_ERR_STATE; }
        if (buf) SSA_CUDA(this, cudaFreeAsync(buf, st));
        buf = nullptr;
        buf_cap = std::max(need, buf_cap * 2);
        SSA_CUDA(this, cudaMallocAsync(reinterpret_cast<void**>(&buf), buf_cap * sizeof(int32_t), st));
        SSA_CUDA(this, cudaMemsetAsync(buf, 0, buf_cap * sizeof(int32_t), st));
      }
      ap.cm_tickets = buf;
    }
    cudaEvent_t t0 = tick(st);
    if (use_tc) {
      SSA_CUDA(this, launch_attn_tc(ap, n_layers, opt_pdl != 0 && !t0, st));
      stats.tc_launches++;
      if (E.cm_C > 0) stats.cm_launches++;
    } else {
      SSA_CUDA(this, launch_attn_simt(ap, n_layers, cfg.dtype == SSA_BF16, st));
    }
    if (t0) timed_push(query_plane ? 1 : 0, t0, tick(st));
    stats.kernel_launches++;
    note_kernel(st, false);
    if (E.cm_C > 0 && E.max_split > 1 && !merge_in_kernel) {   // groups over several clusters: merge kernel
      cudaEvent_t t1 = tick(st);
      if (gsplit)
        SSA_CUDA(this, launch_gm_merge(ap, n_layers, E.max_split, opt_pdl != 0 && !t1, st));
      else
        SSA_CUDA(this, launch_cm_merge(ap, n_layers, E.max_split, opt_pdl != 0 && !t1, st));
      if (t1) timed_push(query_plane ? 3 : 2, t1, tick(st));
      stats.kernel_launches++;
    }
    if (combine) {
      CombineParams cp{};
      cp.part_o = part_o;
      cp.part_lse = part_lse;
      cp.O = io.o.dev;
      cp.lse_out = opts.lse_out;
      cp.o_f32 = opts.o_f32;
      cp.segs = d_segs;
      cp.groups = d_groups;
      cp.n_groups = (int32_t)plan.groups.size();
      cp.n_units = (int32_t)plan.units.size();
      cp.rows_tile = rows_tile;
      cp.rows_per_layer = rows_per_layer;
      cp.in_layer_stride = in_layer_stride;
      cp.Hq = cfg.num_q_heads;
      cp.G = G;
      cp.D = D;
      cp.write_o = 1;
      cp.peer_chunk = opts.peer_chunk;
      cp.n_peers = opts.n_peers;
      cp.lse_off = opts.lse_off;
      cudaEvent_t t1 = tick(st);
      SSA_CUDA(this, launch_combine(cp, n_layers, cfg.dtype == SSA_BF16, st, std::max(1, E.max_split)));
      if (t1) timed_push(query_plane ? 3 : 2, t1, tick(st));
      stats.kernel_launches++;
    }
    int64_t rows = 0;
    for (auto& sg : segs) rows += (int64_t)sg.m * cfg.num_q_heads * n_layers;
    stats.rows_computed += rows;
    if (query_plane) stats.query_rows += rows;
  }
  last_plan_units = (int64_t)plan.units.size();
  last_plan_groups = (int64_t)plan.groups.size();
  last_used_tc = use_tc;
  last_cm_C = E.cm_C;
  last_gbar = E.gbar ? 1 : 0;
  last_max_split = E.max_split;
  last_n_ctas = (int64_t)E.pairs.size();
  return SSA_OK;
}

bool ssa_store::tc_eligible(const std::vector<SegDesc>& segs) const {
  (void)segs;
  if (opt_backend == 1 || !sm100) return false;   // SIMT backend forced, or not an sm_100 device
  const int G = cfg.num_q_heads / cfg.num_kv_heads;
  // bf16 with head_dim 128 always runs on tcgen05: even a 1-token GQA query
  // (4 of 128 rows used) is HBM-bound there — per 128-key tile the two MMAs
  // (~1k clk) and the softmax fit under the ~2.9k clk it takes an SM to stream
  // the 64 KB of K/V at its share of HBM bandwidth.
  return tc_supported_shape(cfg.head_dim, G, cfg.dtype == SSA_BF16);
}

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

int32_t ssa_abi_version(void) { return SSA_ABI_VERSION; }

int32_t ssa_debug_trace(void* host, size_t bytes) {
  return ssa::tc_debug_trace(host, bytes);
}

const char* ssa_status_str(ssa_status s) {
  switch (s) {
    case SSA_OK: return "SSA_OK";
    case SSA_ERR_INVALID_ARG: return "SSA_ERR_INVALID_ARG";
    case SSA_ERR_UNKNOWN_SESSION: return "SSA_ERR_UNKNOWN_SESSION";
    case SSA_ERR_POOL_EXHAUSTED: return "SSA_ERR_POOL_EXHAUSTED";
    case SSA_ERR_SESSION_LIMIT: return "SSA_ERR_SESSION_LIMIT";
    case SSA_ERR_CUDA: return "SSA_ERR_CUDA";
    case SSA_ERR_NCCL: return "SSA_ERR_NCCL";
    case SSA_ERR_UNSUPPORTED: return "SSA_ERR_UNSUPPORTED";
    case SSA_ERR_STATE: return "SSA_ERR_STATE";
  }
  return "SSA_ERR_?";
}

const char* ssa_last_error(void) { return g_last_error.c_str(); }

static bool valid_config(const ssa_store_config* c) {
  if (!c) return false;
  if (c->num_layers <= 0 || c->num_q_heads <= 0 || c->num_kv_heads <= 0) return false;
  if (c->num_q_heads % c->num_kv_heads) return false;
  if (c->page_size < 16 || c->page_size > 256 || (c->page_size & (c->page_size - 1))) return false;
  if (c->num_pages <= 0 || c->max_sessions <= 0) return false;
  if (c->dtype != SSA_BF16 && c->dtype != SSA_FP32) return false;
  const int d = c->head_dim;
  if (d != 16 && d != 32 && d != 64 && d != 128) return false;
  if ((int64_t)c->num_pages * c->num_kv_heads * c->page_size >= (1LL << 31)) return false;
  if (c->kv_format != SSA_KV_SAME && c->kv_format != SSA_KV_E4M3) return false;
  if (c->kv_format == SSA_KV_E4M3 &&
      (c->dtype != SSA_BF16 || d != 128 || !(c->k_scale > 0.f) || !(c->v_scale > 0.f) ||
       !std::isfinite(c->k_scale) || !std::isfinite(c->v_scale)))
    return false;
  return true;
}

size_t ssa_store_pool_bytes(const ssa_store_config* c) {
  if (!valid_config(c)) return 0;
  const size_t elem = c->kv_format == SSA_KV_E4M3 ? 1 : c->dtype == SSA_BF16 ? 2 : 4;
  return 2 * (size_t)c->num_layers * c->num_pages * c->num_kv_heads * c->page_size * c->head_dim * elem;
}

ssa_status ssa_store_create(const ssa_store_config* cfg, ssa_store_t* out) {
  if (!out || !valid_config(cfg)) {
    set_error("invalid store config");
    return SSA_ERR_INVALID_ARG;
  }
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) {
    cudaGetLastError();
    set_error("CUDA device %d not available (%d devices)", cfg->device, ndev);
    return SSA_ERR_CUDA;
  }
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) { set_error("cudaSetDevice: %s", cudaGetErrorString(e)); return SSA_ERR_CUDA; }
  ssa_store* st = new ssa_store();
  st->cfg = *cfg;
  st->elem = cfg->dtype == SSA_BF16 ? 2 : 4;
  st->kv_fp8 = cfg->kv_format == SSA_KV_E4M3;
  st->pelem = st->kv_fp8 ? 1 : st->elem;
  st->scale = cfg->softmax_scale > 0.f ? cfg->softmax_scale : (float)(1.0 / std::sqrt((double)cfg->head_dim));
  cudaDeviceGetAttribute(&st->num_sms, cudaDevAttrMultiProcessorCount, cfg->device);
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, cfg->device);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, cfg->device);
  st->sm100 = (major == 10 && minor == 0);
  const size_t half = ssa_store_pool_bytes(cfg) / 2;
  st->pool_half_bytes = half;
  st->arena_cap = 4u << 20;
  if (cfg->pool_ptr) {
    // borrowed pool (caller-owned device memory of this device, big enough, aligned)
    cudaPointerAttributes a{};
    const bool ok = cudaPointerGetAttributes(&a, cfg->pool_ptr) == cudaSuccess && a.type == cudaMemoryTypeDevice &&
                    a.device == cfg->device && cfg->pool_bytes >= 2 * half &&
                    (reinterpret_cast<uintptr_t>(cfg->pool_ptr) & 255) == 0;
    cudaGetLastError();
    if (!ok) {
      set_error("pool_ptr: not 256-byte aligned device memory of device %d with >= %zu bytes", cfg->device, 2 * half);
      delete st;
      return SSA_ERR_INVALID_ARG;
    }
    st->pool_owned = false;
    st->poolK = cfg->pool_ptr;
    st->poolV = static_cast<char*>(cfg->pool_ptr) + half;
  }
  if ((!cfg->pool_ptr && ((e = cudaMalloc(&st->poolK, half)) != cudaSuccess ||
                          (e = cudaMalloc(&st->poolV, half)) != cudaSuccess)) ||
      (e = cudaMemset(st->poolK, 0, half)) != cudaSuccess || (e = cudaMemset(st->poolV, 0, half)) != cudaSuccess ||
      (e = st->ring.init(8u << 20)) != cudaSuccess ||
      (e = cudaMallocHost(reinterpret_cast<void**>(&st->arena_h), 4u << 20)) != cudaSuccess ||
      (e = cudaMalloc(reinterpret_cast<void**>(&st->arena_d), 4u << 20)) != cudaSuccess ||
      (e = cudaDeviceSynchronize()) != cudaSuccess) {
    set_error("store allocation failed: %s", cudaGetErrorString(e));
    delete st;
    return SSA_ERR_CUDA;
  }
  for (int64_t p = 0; p < cfg->num_pages; ++p) st->free_pages.push((int32_t)p);
  st->page_ref.assign(cfg->num_pages, 0);
  for (auto& row : st->max_clusters_) for (int& c : row) c = -1;
  st->sessions.reserve(std::min(cfg->max_sessions, 4096));
  *out = st;
  return SSA_OK;
}

ssa_store::~ssa_store() {
  cudaDeviceSynchronize();
  for (auto& t : timed) { if (t.a) cudaEventDestroy(t.a); if (t.b) cudaEventDestroy(t.b); }
  for (auto e : spare_events) cudaEventDestroy(e);
  for (auto& s : sessions)
    if (s.d_pages) cudaFree(s.d_pages);
  if (pool_owned) {
    if (poolK) cudaFree(poolK);
    if (poolV) cudaFree(poolV);
  }
  if (part_o) cudaFree(part_o);
  if (part_lse) cudaFree(part_lse);
  if (stage) cudaFree(stage);
  if (qkv_scratch) cudaFree(qkv_scratch);
  if (kv8) cudaFree(kv8);
  if (arena_h) cudaFreeHost(arena_h);
  if (arena_d) cudaFree(arena_d);
  for (auto e : pipe_events) cudaEventDestroy(e);
  if (h2d_stream) cudaStreamDestroy(h2d_stream);
  if (d2h_stream) cudaStreamDestroy(d2h_stream);
  for (auto& e : plan_cache)
    if (e.dev) cudaFree(e.dev);
  if (tickets) cudaFree(tickets);
  if (gb_tickets) cudaFree(gb_tickets);
  if (order_ev) cudaEventDestroy(order_ev);
  if (sample_part) cudaFree(sample_part);
  if (sample_cnt) cudaFree(sample_cnt);
  destroy_comm();
}

ssa_status ssa_store_destroy(ssa_store_t st) {
  if (!st) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  delete st;
  return SSA_OK;
}

ssa_status ssa_store_occupancy(ssa_store_t st, int64_t* used, int64_t* total) {
  if (!st) return SSA_ERR_INVALID_ARG;
  if (used) *used = st->cfg.num_pages - (int64_t)st->free_pages.size();
  if (total) *total = st->cfg.num_pages;
  return SSA_OK;
}

ssa_status ssa_store_stats(ssa_store_t st, ssa_stats* out, int32_t reset) {
  if (!st) return SSA_ERR_INVALID_ARG;
  if (out) *out = st->stats;
  if (reset) st->stats = ssa_stats{};
  return SSA_OK;
}

ssa_status ssa_debug_last_plan(ssa_store_t st, int64_t out[6]) {
  if (!st || !out) return SSA_ERR_INVALID_ARG;
  out[0] = st->last_plan_units;
  out[1] = st->last_plan_groups;
  out[2] = st->last_n_ctas;
  out[3] = st->last_cm_C;
  out[4] = st->last_max_split;
  out[5] = st->last_gbar;
  return SSA_OK;
}

ssa_status ssa_store_set_option(ssa_store_t st, int32_t option, int64_t value) {
  if (!st) return SSA_ERR_INVALID_ARG;
  switch (option) {
    case SSA_OPT_ATTN_BACKEND: if (value < 0 || value > 2) return SSA_ERR_INVALID_ARG; st->opt_backend = value; break;
    case SSA_OPT_MAX_SPLITS: if (value < 0) return SSA_ERR_INVALID_ARG; st->opt_max_splits = value; break;
    case SSA_OPT_FAULT_INJECT: if (value < 0 || value > 2) return SSA_ERR_INVALID_ARG; st->opt_fault = value; break;
    case SSA_OPT_TC_Q_TILES: if (value < 0 || value > 2) return SSA_ERR_INVALID_ARG; st->opt_tc_qtiles = value; break;
    case SSA_OPT_TIMING: if (value < 0 || value > 1) return SSA_ERR_INVALID_ARG; st->opt_timing = value; break;
    case SSA_OPT_GRAPH_ARENA_RESET:
      if (value != 1) return SSA_ERR_INVALID_ARG;
      st->arena_used = 0;
      for (auto& e : st->plan_cache) e.pinned = false;   // old graphs are dropped
      break;
    case SSA_OPT_CLUSTER:
      if (value < -1 || value > 16 || (value > 8 && value != 16)) return SSA_ERR_INVALID_ARG;
      st->opt_cluster = value;
      break;
    case SSA_OPT_PDL: if (value < 0 || value > 1) return SSA_ERR_INVALID_ARG; st->opt_pdl = value; break;
    case SSA_OPT_CM_MERGE: if (value < 0 || value > 5) return SSA_ERR_INVALID_ARG; st->opt_cm_merge = value; break;
    case SSA_OPT_L2_HINT: if (value < 0 || value > 2) return SSA_ERR_INVALID_ARG; st->opt_l2_hint = value; break;
    case SSA_OPT_PIPE_CHUNKS: if (value < -1 || value > 64) return SSA_ERR_INVALID_ARG; st->opt_pipe_chunks = value; break;
    case SSA_OPT_QKV_DEBUG: if (value < 0 || value > 3) return SSA_ERR_INVALID_ARG; st->opt_qkv_debug = value; break;
    default: return SSA_ERR_INVALID_ARG;
  }
  return SSA_OK;
}

ssa_status ssa_store_timing(ssa_store_t st, double ms[SSA_TIMING_KINDS], int64_t count[SSA_TIMING_KINDS], int32_t reset) {
  if (!st) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  ssa_status rc = st->drain_timing();
  if (rc != SSA_OK) return rc;
  for (int i = 0; i < SSA_TIMING_KINDS; ++i) {
    if (ms) ms[i] = st->timing_ms[i];
    if (count) count[i] = st->timing_n[i];
    if (reset) { st->timing_ms[i] = 0; st->timing_n[i] = 0; }
  }
  return SSA_OK;
}

static size_t tensor_bytes(const ssa_store* st, int64_t layers, int64_t rows, int heads) {
  return (size_t)layers * rows * heads * st->cfg.head_dim * st->elem;
}

// Create / append share this path: reserve, upload pages, scatter + attention, commit.
// Calls that change the store cannot be captured into a CUDA graph (their page
// reservation and version bump happen at call time, once): rejected up front.
#define SSA_NO_CAPTURE(stream)                                                              \
  do {                                                                                      \
    if (capturing(stream)) {                                                                \
      set_error("CUDA-graph capture: only query-plane calls can be captured");              \
      return SSA_ERR_STATE;                                                                 \
    }                                                                                       \
  } while (0)

static ssa_status do_append(ssa_store* st, Session& s, int32_t n_new, const void* Q, const void* K,
                            const void* V, void* O, cudaStream_t stream) {
  SSA_NO_CAPTURE(stream);
  const int L = st->cfg.num_layers;
  std::vector<int32_t> got;
  ssa_status rc = st->evict_for_append(s, n_new, stream);
  if (rc != SSA_OK) return rc;
  if ((rc = st->reserve(s, s.n_tokens + n_new, &got)) != SSA_OK) return rc;
  IoSet io;
  io.q = {Q, tensor_bytes(st, L, n_new, st->cfg.num_q_heads)};
  io.k = {K, tensor_bytes(st, L, n_new, st->cfg.num_kv_heads)};
  io.v = {V, tensor_bytes(st, L, n_new, st->cfg.num_kv_heads)};
  io.o = {O, tensor_bytes(st, L, n_new, st->cfg.num_q_heads)};
  if (!O) io.q.user = nullptr;  // Q unused when no rows are requested
  if ((rc = st->stage_inputs(&io, stream)) != SSA_OK) return rc;
  if ((rc = st->push_pages(s, got, stream)) != SSA_OK) return rc;
  SegDesc sg{};
  sg.row0 = 0;
  sg.m = n_new;
  sg.tail_m = sg.m;
  st->fill_cached(s, &sg);
  sg.append_slot0 = (int32_t)st->slot_of(s, s.n_tokens);
  std::vector<SegDesc> segs{sg};
  if ((rc = st->run(segs, io, n_new, 0, L, 1, O != nullptr, false, stream)) != SSA_OK) return rc;
  if ((rc = st->unstage_output(&io, stream)) != SSA_OK) return rc;
  s.n_tokens += n_new;
  s.version += 1;
  st->stats.tokens_appended += n_new;
  return SSA_OK;
}

ssa_status ssa_session_create(ssa_store_t st, int32_t n_prefix, const void* Q, const void* K, const void* V,
                              void* O, void* stream, ssa_session_t* out) {
  SSA_CHECK_STORE(st);
  if (!out || n_prefix <= 0 || !K || !V || (O && !Q)) {
    set_error("session_create: invalid arguments");
    return SSA_ERR_INVALID_ARG;
  }
  SSA_NO_CAPTURE(stream);
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  int live = 0;
  int32_t id = -1;
  for (int i = 0; i < (int)st->sessions.size(); ++i) {
    if (st->sessions[i].live) live++;
    else if (id < 0) id = i;
  }
  if (live >= st->cfg.max_sessions) {
    set_error("session limit %d reached", st->cfg.max_sessions);
    return SSA_ERR_SESSION_LIMIT;
  }
  if (id < 0) {
    id = (int32_t)st->sessions.size();
    st->sessions.emplace_back();
  }
  Session& s = st->sessions[id];
  int32_t* keep_d = s.d_pages;
  int64_t keep_cap = s.d_cap;
  s = Session();
  s.d_pages = keep_d;      // reuse the device table allocation of a dead slot
  s.d_cap = keep_cap;
  s.d_valid = 0;
  s.n_prefix = n_prefix;
  s.live = true;
  ssa_status rc = do_append(st, s, n_prefix, Q, K, V, O, (cudaStream_t)stream);
  if (rc != SSA_OK) {
    s.live = false;
    st->release(s.pages);
    s.pages.clear();
    return rc;
  }
  s.version = 1;
  *out = id;
  return SSA_OK;
}

ssa_status ssa_session_append(ssa_store_t st, ssa_session_t id, int32_t n_new, const void* Q, const void* K,
                              const void* V, void* O, void* stream, uint64_t* new_version) {
  SSA_CHECK_STORE(st);
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (n_new <= 0 || !K || !V || (O && !Q)) { set_error("append: invalid arguments"); return SSA_ERR_INVALID_ARG; }
  if (s->ticket_open) { set_error("append: a per-layer append is open"); return SSA_ERR_STATE; }
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  ssa_status rc = do_append(st, *s, n_new, Q, K, V, O, (cudaStream_t)stream);
  if (rc == SSA_OK && new_version) *new_version = s->version;
  return rc;
}

// ---- per-layer append tickets
ssa_status ssa_append_begin(ssa_store_t st, ssa_session_t id, int32_t n_new, int32_t* ticket) {
  SSA_CHECK_STORE(st);
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (n_new <= 0 || !ticket) return SSA_ERR_INVALID_ARG;
  if (s->ticket_open) { set_error("append_begin: ticket already open"); return SSA_ERR_STATE; }
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, nullptr);
  std::vector<int32_t> got;
  ssa_status rc = st->evict_for_append(*s, n_new, nullptr);
  if (rc != SSA_OK) return rc;
  if ((rc = st->reserve(*s, s->n_tokens + n_new, &got)) != SSA_OK) return rc;
  const size_t before = s->pages.size();
  if ((rc = st->push_pages(*s, got, nullptr)) != SSA_OK) return rc;
  s->ticket_open = true;
  s->ticket_id = ++st->ticket_seq;
  s->ticket_n_new = n_new;
  s->ticket_pages = (int64_t)(s->pages.size() - before);
  s->ticket_done.assign(st->cfg.num_layers, 0);
  *ticket = s->ticket_id;
  return SSA_OK;
}

static Session* check_ticket(ssa_store* st, ssa_session_t id, int32_t ticket, ssa_status* rc) {
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); *rc = SSA_ERR_UNKNOWN_SESSION; return nullptr; }
  if (!s->ticket_open || s->ticket_id != ticket) { set_error("bad ticket"); *rc = SSA_ERR_STATE; return nullptr; }
  return s;
}

ssa_status ssa_append_layer(ssa_store_t st, ssa_session_t id, int32_t ticket, int32_t layer, const void* Q,
                            const void* K, const void* V, void* O, void* stream) {
  SSA_CHECK_STORE(st);
  ssa_status rc = SSA_OK;
  Session* s = check_ticket(st, id, ticket, &rc);
  if (!s) return rc;
  if (layer < 0 || layer >= st->cfg.num_layers || !K || !V || (O && !Q)) return SSA_ERR_INVALID_ARG;
  if (s->ticket_done[layer]) { set_error("layer %d already appended", layer); return SSA_ERR_STATE; }
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  const int32_t n_new = s->ticket_n_new;
  IoSet io;
  io.q = {O ? Q : nullptr, tensor_bytes(st, 1, n_new, st->cfg.num_q_heads)};
  io.k = {K, tensor_bytes(st, 1, n_new, st->cfg.num_kv_heads)};
  io.v = {V, tensor_bytes(st, 1, n_new, st->cfg.num_kv_heads)};
  io.o = {O, tensor_bytes(st, 1, n_new, st->cfg.num_q_heads)};
  cudaStream_t cs = (cudaStream_t)stream;
  if ((rc = st->stage_inputs(&io, cs)) != SSA_OK) return rc;
  SegDesc sg{};
  sg.m = n_new;
  sg.tail_m = sg.m;
  st->fill_cached(*s, &sg);
  sg.append_slot0 = (int32_t)st->slot_of(*s, s->n_tokens);
  std::vector<SegDesc> segs{sg};
  if ((rc = st->run(segs, io, n_new, layer, 1, 0, O != nullptr, false, cs)) != SSA_OK) return rc;
  if ((rc = st->unstage_output(&io, cs)) != SSA_OK) return rc;
  s->ticket_done[layer] = 1;
  return SSA_OK;
}

ssa_status ssa_append_commit(ssa_store_t st, ssa_session_t id, int32_t ticket, uint64_t* new_version) {
  SSA_CHECK_STORE(st);
  ssa_status rc = SSA_OK;
  Session* s = check_ticket(st, id, ticket, &rc);
  if (!s) return rc;
  for (auto d : s->ticket_done)
    if (!d) { set_error("append_commit: not every layer was appended"); return SSA_ERR_STATE; }
  s->n_tokens += s->ticket_n_new;
  s->version += 1;
  st->stats.tokens_appended += s->ticket_n_new;
  s->ticket_open = false;
  if (new_version) *new_version = s->version;
  return SSA_OK;
}

ssa_status ssa_append_abort(ssa_store_t st, ssa_session_t id, int32_t ticket) {
  SSA_CHECK_STORE(st);
  ssa_status rc = SSA_OK;
  Session* s = check_ticket(st, id, ticket, &rc);
  if (!s) return rc;
  std::vector<int32_t> back(s->pages.end() - s->ticket_pages, s->pages.end());
  s->pages.resize(s->pages.size() - s->ticket_pages);
  s->d_valid = std::min<int64_t>(s->d_valid, (int64_t)s->pages.size());
  st->release(back);
  s->ticket_open = false;
  return SSA_OK;
}

ssa_status ssa_session_truncate(ssa_store_t st, ssa_session_t id, int64_t p, uint64_t* new_version) {
  SSA_CHECK_STORE(st);
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (s->ticket_open) return SSA_ERR_STATE;
  if (p < s->n_prefix || p > s->n_tokens) {
    set_error("truncate: p=%lld outside [n_prefix=%lld, n_tokens=%lld]", (long long)p, (long long)s->n_prefix,
              (long long)s->n_tokens);
    return SSA_ERR_INVALID_ARG;
  }
  if (p < s->n_tokens) {
    const int64_t keep = st->pages_for(*s, p);
    std::vector<int32_t> back(s->pages.begin() + keep, s->pages.end());
    s->pages.resize(keep);
    s->d_valid = std::min<int64_t>(s->d_valid, keep);
    st->release(back);
    s->n_tokens = p;
    if (p == s->n_prefix) s->r1_skip = 0;   // Region 1 empty: its layout restarts at the R0 pad
    s->version += 1;
  }
  if (new_version) *new_version = s->version;
  return SSA_OK;
}

ssa_status ssa_session_evict_oldest(ssa_store_t st, ssa_session_t id, int64_t n, void* stream,
                                    uint64_t* new_version) {
  SSA_CHECK_STORE(st);
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (s->ticket_open) return SSA_ERR_STATE;
  SSA_NO_CAPTURE(stream);
  if (n < 0 || n > s->n_tokens - s->n_prefix) {
    set_error("evict_oldest: n=%lld but %lld Region-1 tokens retained", (long long)n,
              (long long)(s->n_tokens - s->n_prefix));
    return SSA_ERR_INVALID_ARG;
  }
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  ssa_status rc = st->evict(*s, n, (cudaStream_t)stream);
  if (rc == SSA_OK && new_version) *new_version = s->version;
  return rc;
}

ssa_status ssa_session_set_retention(ssa_store_t st, ssa_session_t id, int64_t max_tokens) {
  SSA_CHECK_STORE(st);
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (max_tokens < 0) return SSA_ERR_INVALID_ARG;
  s->retention = max_tokens;
  return SSA_OK;
}

ssa_status ssa_session_alias_prefix(ssa_store_t st, ssa_session_t donor_id, int64_t len, void* stream,
                                    ssa_session_t* out) {
  SSA_CHECK_STORE(st);
  Session* d = st->get(donor_id);
  if (!d) { set_error("unknown session %d", donor_id); return SSA_ERR_UNKNOWN_SESSION; }
  SSA_NO_CAPTURE(stream);
  if (!out || len < 0 || len > d->n_tokens || (len > d->n_prefix && d->n_evicted > 0)) {
    set_error("alias_prefix: len=%lld invalid for a donor of %lld tokens (%lld evicted)", (long long)len,
              (long long)d->n_tokens, (long long)d->n_evicted);
    return SSA_ERR_INVALID_ARG;
  }
  if (d->ticket_open) return SSA_ERR_STATE;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  const int64_t P = st->cfg.page_size;
  const int64_t end_slot = st->slots_for(*d, len);
  const int64_t full = end_slot / P;                 // pages shared whole
  const bool partial = (end_slot % P) != 0;          // the page holding token len-1 is copied
  if (partial && st->free_pages.empty()) {
    set_error("alias_prefix: pool exhausted");
    return SSA_ERR_POOL_EXHAUSTED;
  }
  int live = 0;
  int32_t id = -1;
  for (int i = 0; i < (int)st->sessions.size(); ++i) {
    if (st->sessions[i].live) live++;
    else if (id < 0) id = i;
  }
  if (live >= st->cfg.max_sessions) {
    set_error("session limit %d reached", st->cfg.max_sessions);
    return SSA_ERR_SESSION_LIMIT;
  }
  if (id < 0) {
    id = (int32_t)st->sessions.size();
    st->sessions.emplace_back();
    d = st->get(donor_id);   // the vector may have moved
  }
  Session& s = st->sessions[id];
  int32_t* keep_d = s.d_pages;
  int64_t keep_cap = s.d_cap;
  s = Session();
  s.d_pages = keep_d;
  s.d_cap = keep_cap;
  s.d_valid = 0;
  s.live = true;
  s.n_prefix = std::min(len, d->n_prefix);
  s.n_tokens = len;
  s.version = 1;
  std::vector<int32_t> pages(d->pages.begin(), d->pages.begin() + full);
  for (int32_t pg : pages) st->page_ref[pg]++;
  cudaStream_t cs = (cudaStream_t)stream;
  if (partial) {
    const int32_t dst = st->free_pages.top();   // lowest free id (R-9)
    st->free_pages.pop();
    st->page_ref[dst] = 1;
    st->stats.pages_reserved += 1;
    const int32_t src = d->pages[full];
    // one page = [Hkv][P][d] contiguous per layer; layers are num_pages pages apart
    const size_t blk = (size_t)st->cfg.num_kv_heads * P * st->cfg.head_dim * st->pelem;
    const size_t pitch = blk * (size_t)st->cfg.num_pages;
    for (void* pool : {st->poolK, st->poolV}) {
      char* b = static_cast<char*>(pool);
      SSA_CUDA(st, cudaMemcpy2DAsync(b + (size_t)dst * blk, pitch, b + (size_t)src * blk, pitch, blk,
                                     st->cfg.num_layers, cudaMemcpyDeviceToDevice, cs));
    }
    pages.push_back(dst);
  }
  ssa_status rc = st->push_pages(s, pages, cs, true);
  if (rc != SSA_OK) return rc;
  *out = id;
  return SSA_OK;
}

ssa_status ssa_session_destroy(ssa_store_t st, ssa_session_t id) {
  if (!st) return SSA_ERR_INVALID_ARG;
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  st->release(s->pages);
  s->pages.clear();
  s->d_valid = 0;
  s->live = false;
  s->ticket_open = false;
  return SSA_OK;
}

// ---- query plane
ssa_status ssa_session_query(ssa_store_t st, ssa_session_t id, int32_t layer, int32_t n_q, const void* Q,
                             const void* K, const void* V, void* O, void* stream) {
  int32_t len = n_q;
  return ssa_flash_query_batch(st, id, layer, 1, &len, Q, K, V, O, stream);
}

ssa_status ssa_flash_query_batch(ssa_store_t st, ssa_session_t id, int32_t layer, int32_t k,
                                 const int32_t* q_lens, const void* Q, const void* K, const void* V, void* O,
                                 void* stream) {
  SSA_CHECK_STORE(st);
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (k <= 0 || !q_lens || !Q || !K || !V || !O || layer < -1 || layer >= st->cfg.num_layers) {
    set_error("query: invalid arguments");
    return SSA_ERR_INVALID_ARG;
  }
  int64_t total = 0;
  for (int i = 0; i < k; ++i) {
    if (q_lens[i] <= 0) { set_error("query: q_lens[%d] <= 0", i); return SSA_ERR_INVALID_ARG; }
    total += q_lens[i];
  }
  if (total >= (1LL << 31)) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  const int64_t Lin = layer < 0 ? st->cfg.num_layers : 1;
  IoSet io;
  io.q = {Q, tensor_bytes(st, Lin, total, st->cfg.num_q_heads)};
  io.k = {K, tensor_bytes(st, Lin, total, st->cfg.num_kv_heads)};
  io.v = {V, tensor_bytes(st, Lin, total, st->cfg.num_kv_heads)};
  io.o = {O, tensor_bytes(st, Lin, total, st->cfg.num_q_heads)};
  cudaStream_t cs = (cudaStream_t)stream;
  // host buffers with all layers: chunked copies overlapped with the kernels
  const bool pipelined = layer < 0 && Lin >= 4 && st->opt_pipe_chunks >= 0 && !capturing(stream) &&
                         (!is_device_ptr(Q) || !is_device_ptr(K) || !is_device_ptr(V) || !is_device_ptr(O));
  ssa_status rc = pipelined ? SSA_OK : st->stage_inputs(&io, cs);
  if (rc != SSA_OK) return rc;
  std::vector<SegDesc> segs;
  int64_t row = 0;
  for (int i = 0; i < k; ++i) {
    SegDesc sg{};
    sg.row0 = row;
    sg.m = q_lens[i];
    sg.tail_m = sg.m;
    st->fill_cached(*s, &sg);
    sg.append_slot0 = -1;
    segs.push_back(sg);
    row += q_lens[i];
  }
  if (pipelined) return st->run_pipelined(segs, io, total, (int32_t)Lin, true, cs);
  if ((rc = st->run(segs, io, total, layer < 0 ? 0 : layer, (int32_t)Lin, 1, true, true, cs)) != SSA_OK) return rc;
  return st->unstage_output(&io, cs);
}

// ---- multi-tenant batch
ssa_status ssa_batch_run(ssa_store_t st, int32_t layer, int32_t n_items, const ssa_work_item* items, const void* Q,
                         const void* K, const void* V, void* O, void* stream) {
  SSA_CHECK_STORE(st);
  const int L = st->cfg.num_layers;
  if (n_items <= 0 || !items || !Q || !K || !V || !O || layer < -1 || layer >= L) {
    set_error("batch_run: invalid arguments");
    return SSA_ERR_INVALID_ARG;
  }
  for (int32_t i = 0; i < n_items; ++i)
    if (items[i].kind == SSA_WORK_APPEND) { SSA_NO_CAPTURE(stream); break; }
  int64_t n_rows = 0;
  std::vector<int32_t> app_sessions;
  for (int i = 0; i < n_items; ++i) {
    const ssa_work_item& it = items[i];
    if (it.n_tokens <= 0 || it.row_offset < 0 || it.kind < 0 || it.kind > 2) return SSA_ERR_INVALID_ARG;
    n_rows = std::max<int64_t>(n_rows, it.row_offset + it.n_tokens);
    if (it.kind != SSA_WORK_STATELESS) {
      Session* s = st->get(it.session);
      if (!s) { set_error("batch_run: unknown session %d", it.session); return SSA_ERR_UNKNOWN_SESSION; }
      if (it.kind == SSA_WORK_APPEND) {
        if (std::find(app_sessions.begin(), app_sessions.end(), it.session) != app_sessions.end()) {
          set_error("batch_run: two APPEND items for session %d", it.session);
          return SSA_ERR_INVALID_ARG;
        }
        app_sessions.push_back(it.session);
        const bool first = layer <= 0;
        if (first && s->ticket_open) { set_error("batch_run: append already open"); return SSA_ERR_STATE; }
        if (!first && (!s->ticket_open || s->ticket_n_new != it.n_tokens || !s->batch_ticket)) {
          set_error("batch_run: per-layer batch must start at layer 0 with the same items");
          return SSA_ERR_STATE;
        }
      }
    }
  }
  if (n_rows >= (1LL << 31)) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  cudaStream_t cs = (cudaStream_t)stream;
  // Reserve pages for every APPEND item, in item order, all-or-none (R-7).
  ssa_status rc = SSA_OK;
  if (layer <= 0) {
    // Retention guard for every APPEND item (Alg. 1), checked for the
    // whole batch before any state changes: evictions, then reservations.
    {
      int64_t need = 0, freed = 0;
      std::vector<std::pair<Session*, int64_t>> ev;
      for (int i = 0; i < n_items; ++i) {
        if (items[i].kind != SSA_WORK_APPEND) continue;
        Session* s = st->get(items[i].session);
        int64_t n_ev = 0, nd = 0, fr = 0;
        if ((rc = st->retention_plan(*s, items[i].n_tokens, &n_ev, &nd, &fr)) != SSA_OK) return rc;
        need += nd;
        freed += fr;
        if (n_ev) ev.push_back({s, n_ev});
      }
      if (need > (int64_t)st->free_pages.size() + freed) {
        set_error("batch_run: pool exhausted (need %lld pages)", (long long)need);
        return SSA_ERR_POOL_EXHAUSTED;
      }
      for (auto& e : ev)
        if ((rc = st->evict(*e.first, e.second, cs)) != SSA_OK) return rc;
    }
    std::vector<std::pair<Session*, std::vector<int32_t>>> res;
    for (int i = 0; i < n_items; ++i) {
      if (items[i].kind != SSA_WORK_APPEND) continue;
      Session* s = st->get(items[i].session);
      std::vector<int32_t> got;
      rc = st->reserve(*s, s->n_tokens + items[i].n_tokens, &got);
      if (rc != SSA_OK) {
        for (auto& r : res) st->release(r.second);
        return rc;
      }
      res.push_back({s, got});
    }
    for (auto& r : res) {
      Session* s = r.first;
      const size_t before = s->pages.size();
      if ((rc = st->push_pages(*s, r.second, cs)) != SSA_OK) return rc;
      s->ticket_open = true;
      s->batch_ticket = true;
      s->ticket_id = ++st->ticket_seq;
      s->ticket_pages = (int64_t)(s->pages.size() - before);
      s->ticket_done.assign(L, 0);
    }
    for (int i = 0; i < n_items; ++i)
      if (items[i].kind == SSA_WORK_APPEND) st->get(items[i].session)->ticket_n_new = items[i].n_tokens;
  }
  const int64_t Lin = layer < 0 ? L : 1;
  IoSet io;
  io.q = {Q, tensor_bytes(st, Lin, n_rows, st->cfg.num_q_heads)};
  io.k = {K, tensor_bytes(st, Lin, n_rows, st->cfg.num_kv_heads)};
  io.v = {V, tensor_bytes(st, Lin, n_rows, st->cfg.num_kv_heads)};
  io.o = {O, tensor_bytes(st, Lin, n_rows, st->cfg.num_q_heads)};
  if ((rc = st->stage_inputs(&io, cs)) != SSA_OK) return rc;
  std::vector<SegDesc> segs;
  for (int i = 0; i < n_items; ++i) {
    const ssa_work_item& it = items[i];
    SegDesc sg{};
    sg.row0 = it.row_offset;
    sg.m = it.n_tokens;
    sg.tail_m = sg.m;
    sg.append_slot0 = -1;
    if (it.kind == SSA_WORK_STATELESS) {
      sg.n_slots = 0;
      sg.pages = nullptr;
    } else {
      Session* s = st->get(it.session);
      st->fill_cached(*s, &sg);  // snapshot: n_tokens of version t
      if (it.kind == SSA_WORK_APPEND) sg.append_slot0 = (int32_t)st->slot_of(*s, s->n_tokens);
    }
    segs.push_back(sg);
  }
  if ((rc = st->run(segs, io, n_rows, layer < 0 ? 0 : layer, (int32_t)Lin, 1, true, false, cs)) != SSA_OK) return rc;
  if ((rc = st->unstage_output(&io, cs)) != SSA_OK) return rc;
  // Commit appends after the last layer (snapshot semantics).
  if (layer < 0 || layer == L - 1) {
    for (int i = 0; i < n_items; ++i) {
      if (items[i].kind != SSA_WORK_APPEND) continue;
      Session* s = st->get(items[i].session);
      s->n_tokens += items[i].n_tokens;
      s->version += 1;
      s->ticket_open = false;
      s->batch_ticket = false;
      st->stats.tokens_appended += items[i].n_tokens;
    }
  }
  return SSA_OK;
}

// ---- introspection
ssa_status ssa_session_get_info(ssa_store_t st, ssa_session_t id, ssa_session_info* out) {
  if (!st || !out) return SSA_ERR_INVALID_ARG;
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  out->n_tokens = s->n_tokens;
  out->n_prefix = s->n_prefix;
  out->n_pages = (int64_t)s->pages.size();
  out->version = s->version;
  out->n_evicted = s->n_evicted;
  out->retention = s->retention;
  return SSA_OK;
}

ssa_status ssa_session_page_table(ssa_store_t st, ssa_session_t id, int32_t* out, int64_t cap, int64_t* n_out) {
  if (!st) return SSA_ERR_INVALID_ARG;
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  const int64_t n = (int64_t)s->pages.size();
  if (n_out) *n_out = n;
  if (out) {
    if (cap < n) return SSA_ERR_INVALID_ARG;
    std::copy(s->pages.begin(), s->pages.end(), out);
  }
  return SSA_OK;
}

ssa_status ssa_session_read_kv(ssa_store_t st, ssa_session_t id, int32_t layer, int64_t start, int64_t count,
                               void* K_out, void* V_out) {
  SSA_CHECK_STORE(st);
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (layer < 0 || layer >= st->cfg.num_layers || start < 0 || count < 0 || start + count > s->n_tokens || !K_out ||
      !V_out)
    return SSA_ERR_INVALID_ARG;
  if (count == 0) return SSA_OK;
  cudaSetDevice(st->cfg.device);
  const size_t bytes = (size_t)count * st->cfg.num_kv_heads * st->cfg.head_dim * st->pelem;
  const bool kdev = is_device_ptr(K_out), vdev = is_device_ptr(V_out);
  void* dk = K_out;
  void* dv = V_out;
  void* tmp = nullptr;
  if (!kdev || !vdev) {
    SSA_CUDA(st, cudaMalloc(&tmp, 2 * bytes));
    dk = tmp;
    dv = static_cast<char*>(tmp) + bytes;
  }
  GatherParams gp{};
  gp.poolK = st->poolK;
  gp.poolV = st->poolV;
  gp.K = dk;
  gp.V = dv;
  gp.num_pages = st->cfg.num_pages;
  gp.layer = layer;
  gp.Hkv = st->cfg.num_kv_heads;
  gp.D = st->cfg.head_dim;
  gp.P = st->cfg.page_size;
  gp.elem_bytes = st->pelem;
  gp.start = start;
  gp.count = count;
  gp.n_prefix = s->n_prefix;
  gp.n_prefix_slots_pad = (int32_t)(st->pad_prefix(s->n_prefix) + s->r1_skip);
  gp.pages = s->d_pages;
  SSA_CUDA(st, cudaDeviceSynchronize());
  SSA_CUDA(st, launch_gather(gp, nullptr));
  st->stats.kernel_launches++;
  SSA_CUDA(st, cudaDeviceSynchronize());
  if (tmp) {
    SSA_CUDA(st, cudaMemcpy(K_out, dk, bytes, kdev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
    SSA_CUDA(st, cudaMemcpy(V_out, dv, bytes, vdev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
    cudaFree(tmp);
  }
  return SSA_OK;
}

ssa_status ssa_session_load_kv(ssa_store_t st, ssa_session_t id, int64_t count, const void* K, const void* V,
                               void* stream) {
  SSA_CHECK_STORE(st);
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (count <= 0 || count >= (1LL << 31) || !K || !V) return SSA_ERR_INVALID_ARG;
  if (s->ticket_open) return SSA_ERR_STATE;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  return do_append(st, *s, (int32_t)count, nullptr, K, V, nullptr, (cudaStream_t)stream);
}

// ---- on-device greedy sampling
ssa_status ssa_greedy_sample(ssa_store_t st, ssa_dtype dtype, int32_t n_rows, int32_t vocab, int64_t row_stride,
                             const void* logits, int32_t* out_ids, float* out_gap, float* out_top2,
                             const int32_t* draft, int32_t* out_n_accept, void* stream) {
  SSA_CHECK_STORE(st);
  if (n_rows <= 0 || n_rows > 65535 || vocab <= 0 || row_stride < vocab || !logits || !out_ids ||
      (dtype != SSA_FP32 && dtype != SSA_BF16) || (draft && !out_n_accept)) {
    set_error("greedy_sample: invalid arguments");
    return SSA_ERR_INVALID_ARG;
  }
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  cudaStream_t cs = (cudaStream_t)stream;
  // about four CTAs per SM over all rows, at least 4096 logits per CTA
  int splits = std::max(1, (4 * st->num_sms + n_rows - 1) / n_rows);
  splits = std::min(splits, std::max(1, vocab / 4096));
  const size_t part = (size_t)n_rows * splits * sample_partial_bytes();
  if ((part > st->sample_part_cap || (size_t)n_rows + 1 > st->sample_cnt_cap) && capturing(stream)) {
    set_error("CUDA-graph capture: warm up the call once before capturing (sampling scratch)");
    return SSA_ERR_STATE;
  }
  if (part > st->sample_part_cap) {   // stream-ordered growth (enter() ordered earlier calls)
    if (st->sample_part) SSA_CUDA(st, cudaFreeAsync(st->sample_part, cs));
    st->sample_part = nullptr;
    st->sample_part_cap = std::max(part, 2 * st->sample_part_cap);
    SSA_CUDA(st, cudaMallocAsync(&st->sample_part, st->sample_part_cap, cs));
  }
  if ((size_t)n_rows + 1 > st->sample_cnt_cap) {
    if (st->sample_cnt) SSA_CUDA(st, cudaFreeAsync(st->sample_cnt, cs));
    st->sample_cnt = nullptr;
    st->sample_cnt_cap = std::max<size_t>(n_rows + 1, 2 * st->sample_cnt_cap);
    SSA_CUDA(st, cudaMallocAsync(reinterpret_cast<void**>(&st->sample_cnt), st->sample_cnt_cap * sizeof(int32_t), cs));
    SSA_CUDA(st, cudaMemsetAsync(st->sample_cnt, 0, st->sample_cnt_cap * sizeof(int32_t), cs));
  }
  SampleParams sp{};
  sp.logits = logits;
  sp.row_stride = row_stride;
  sp.vocab = vocab;
  sp.n_rows = n_rows;
  sp.splits = splits;
  sp.partials = st->sample_part;
  sp.row_counters = st->sample_cnt;
  sp.out_ids = out_ids;
  sp.out_gap = out_gap;
  sp.out_top = out_top2;
  sp.draft = draft;
  sp.out_n_accept = out_n_accept;
  SSA_CUDA(st, launch_greedy(sp, dtype == SSA_BF16, cs));
  st->stats.kernel_launches++;
  return SSA_OK;
}

// FNV-1a 64 over the session's records (library's own implementation; the
// oracle has an independent one).
static uint64_t fnv1a(const uint8_t* p, size_t n, uint64_t h) {
  for (size_t i = 0; i < n; ++i) { h ^= p[i]; h *= 0x100000001b3ULL; }
  return h;
}

ssa_status ssa_session_digest(ssa_store_t st, ssa_session_t id, uint64_t* out) {
  SSA_CHECK_STORE(st);
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (!out) return SSA_ERR_INVALID_ARG;
  uint64_t h = 0xcbf29ce484222325ULL;
  const int64_t n = s->n_tokens;
  const size_t row = (size_t)st->cfg.num_kv_heads * st->cfg.head_dim * st->pelem;
  std::vector<uint8_t> k(n * row), v(n * row);
  for (int32_t l = 0; l < st->cfg.num_layers; ++l) {
    if (n) {
      ssa_status rc = ssa_session_read_kv(st, id, l, 0, n, k.data(), v.data());
      if (rc != SSA_OK) return rc;
    }
    for (int64_t t = 0; t < n; ++t) {
      uint8_t hdr[12];
      const int32_t l32 = l;
      const int64_t pos = t < s->n_prefix ? t : t + s->n_evicted;   // positions never re-based (R-8)
      memcpy(hdr, &l32, 4);       // little-endian host (x86-64)
      memcpy(hdr + 4, &pos, 8);
      h = fnv1a(hdr, 12, h);
      h = fnv1a(k.data() + t * row, row, h);
      h = fnv1a(v.data() + t * row, row, h);
    }
  }
  *out = h;
  return SSA_OK;
}

// Planner introspection for host-logic tests (no GPU needed).
int32_t ssa_debug_plan(int32_t n_segs, const int32_t* seg_m, const int32_t* seg_slots, int32_t Hkv,
                       int32_t q_tile_tokens, int32_t key_tile, int32_t n_layers, int32_t num_sms,
                       int32_t ctas_per_sm, int32_t max_splits, int32_t* units_out, int32_t cap_units) {
  std::vector<SegDesc> segs(n_segs);
  for (int i = 0; i < n_segs; ++i) {
    segs[i] = SegDesc{};
    segs[i].m = seg_m[i];
    segs[i].tail_m = seg_m[i];
    segs[i].n_slots = seg_slots[i];
  }
  PlanConfig pc;
  pc.Hkv = Hkv;
  pc.q_tile_tokens = q_tile_tokens;
  pc.key_tile = key_tile;
  pc.n_layers = n_layers;
  pc.num_sms = num_sms;
  pc.ctas_per_sm = ctas_per_sm;
  pc.max_splits = max_splits;
  pc.pair_slots = key_tile == tc_key_tile();   // the tcgen05 key tile selects two-slot CTAs
  if (pc.pair_slots) {                          // mirror run()'s tcgen05 cost model
    pc.min_tiles_per_unit = 2;
    pc.unit_overhead_tiles = 2.0;
    pc.split_overhead_tiles = kTcSplitOverheadTiles;
  }
  Plan plan;
  plan_units(segs, pc, &plan);
  const int32_t n = (int32_t)plan.units.size();
  if (units_out) {
    for (int i = 0; i < n && i < cap_units; ++i) {
      const WorkUnit& u = plan.units[i];
      int32_t* o = units_out + 8 * i;
      o[0] = u.seg; o[1] = u.kv_head; o[2] = u.q_tok0; o[3] = u.q_ntok;
      o[4] = u.tile_lo; o[5] = u.tile_hi; o[6] = u.group; o[7] = u.split;
    }
  }
  return n;
}

}  // extern "C"

// ---- fused data-plane projection (Alg. 1 L282 `Forward`)

static bool dev_ok(const void* p, void* stream) { return p && (capturing(stream) || is_device_ptr(p)); }

static uint64_t* g_qkv_trace = nullptr;   // ssa_debug_qkv_trace
static bool qkv_args_ok(ssa_store* st, int32_t n, int32_t hidden, const void* X, const void* W, void* stream) {
  if (n <= 0 || !X || !W || st->cfg.dtype != SSA_BF16 || !st->sm100 || !qkv_supported(st->cfg.head_dim, hidden)) {
    set_error("qkv: needs bf16, head_dim 128, hidden %% 64 == 0, sm_100 and n > 0");
    return false;
  }
  if (!dev_ok(X, stream) || !dev_ok(W, stream)) {
    set_error("qkv: X and W must be device pointers");
    return false;
  }
  return true;
}

static ssa_status qkv_launch(ssa_store* st, int32_t n, int32_t hidden, int64_t pos0, float rope_theta,
                             const void* X, const void* W, void* Q, void* K, void* V, const Session* paged,
                             int32_t layer, int64_t slot0, cudaStream_t cs) {
  QkvParams qp{};
  qp.X = X;
  qp.W = W;
  qp.Q = Q;
  qp.K = K;
  qp.V = V;
  qp.m = n;
  qp.hidden = hidden;
  qp.Hq = st->cfg.num_q_heads;
  qp.Hkv = st->cfg.num_kv_heads;
  qp.D = st->cfg.head_dim;
  qp.pos0 = pos0;
  qp.rope_theta = rope_theta;
  if (paged) {
    qp.poolK = st->poolK;
    qp.poolV = st->poolV;
    qp.pages = paged->d_pages;
    qp.page_base = (int64_t)layer * st->cfg.num_pages;
    qp.slot0 = (int32_t)slot0;
    qp.P = st->cfg.page_size;
    qp.kv_fp8 = st->kv_fp8 ? 1 : 0;
    qp.k_scale = st->cfg.k_scale;
    qp.v_scale = st->cfg.v_scale;
  }
  qp.splits = qkv_choose_splits(n, qp.Hq + 2 * qp.Hkv, hidden, st->num_sms);
  qp.debug = (int32_t)st->opt_qkv_debug;
  qp.trace = g_qkv_trace;
  cudaEvent_t t0 = st->tick(cs);
  SSA_CUDA(st, launch_qkv_rope(qp, cs, st->opt_pdl != 0 && !t0));
  if (t0) st->timed_push(5, t0, st->tick(cs));
  st->stats.kernel_launches++;
  st->note_kernel(cs, qp.poolK != nullptr);   // K/V written straight into pages
  return SSA_OK;
}

ssa_status ssa_qkv_rope(ssa_store_t st, int32_t n, int32_t hidden, int64_t pos0, float rope_theta, const void* X,
                        const void* W, void* Q, void* K, void* V, void* stream) {
  SSA_CHECK_STORE(st);
  if (!qkv_args_ok(st, n, hidden, X, W, stream) || !Q || !K || !V || pos0 < 0) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  return qkv_launch(st, n, hidden, pos0, rope_theta, X, W, Q, K, V, nullptr, 0, 0, (cudaStream_t)stream);
}

static ssa_status qkv_scratch(ssa_store* st, int64_t n, void** q, void** k, void** v, cudaStream_t cs) {
  const size_t eq = (size_t)n * st->cfg.num_q_heads * st->cfg.head_dim * 2;
  const size_t ek = (size_t)n * st->cfg.num_kv_heads * st->cfg.head_dim * 2;
  const size_t need = eq + 2 * ek;
  if (need > st->qkv_scratch_cap) {
    if (capturing(cs)) {
      set_error("CUDA-graph capture: warm up the call once before capturing (projection scratch)");
      return SSA_ERR_STATE;
    }
    if (st->qkv_scratch) SSA_CUDA(st, cudaFreeAsync(st->qkv_scratch, cs));
    st->qkv_scratch = nullptr;
    st->qkv_scratch_cap = std::max(need, 2 * st->qkv_scratch_cap);
    SSA_CUDA(st, cudaMallocAsync(&st->qkv_scratch, st->qkv_scratch_cap, cs));
  }
  *q = st->qkv_scratch;
  *k = static_cast<uint8_t*>(st->qkv_scratch) + eq;
  *v = static_cast<uint8_t*>(st->qkv_scratch) + eq + ek;
  return SSA_OK;
}

ssa_status ssa_append_layer_fused(ssa_store_t st, ssa_session_t id, int32_t ticket, int32_t layer, int32_t hidden,
                                  float rope_theta, const void* X, const void* W, void* O, void* stream) {
  SSA_CHECK_STORE(st);
  ssa_status rc = SSA_OK;
  Session* s = check_ticket(st, id, ticket, &rc);
  if (!s) return rc;
  SSA_NO_CAPTURE(stream);
  if (layer < 0 || layer >= st->cfg.num_layers || !dev_ok(O, stream)) return SSA_ERR_INVALID_ARG;
  if (!qkv_args_ok(st, s->ticket_n_new, hidden, X, W, stream)) return SSA_ERR_INVALID_ARG;
  if (s->ticket_done[layer]) { set_error("layer %d already appended", layer); return SSA_ERR_STATE; }
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  const int32_t n_new = s->ticket_n_new;
  void *q, *k, *v;
  if ((rc = qkv_scratch(st, n_new, &q, &k, &v, (cudaStream_t)stream)) != SSA_OK) return rc;
  cudaStream_t cs = (cudaStream_t)stream;
  const int64_t slot0 = st->slot_of(*s, s->n_tokens);
  // positions never re-based (R-8): the next token's position counts evicted tokens
  const int64_t pos0 = s->n_tokens + s->n_evicted;
  if ((rc = qkv_launch(st, n_new, hidden, pos0, rope_theta, X, W, q, k, v, s, layer, slot0, cs)) != SSA_OK) return rc;
  IoSet io;
  io.q = {q, tensor_bytes(st, 1, n_new, st->cfg.num_q_heads)};
  io.k = {k, tensor_bytes(st, 1, n_new, st->cfg.num_kv_heads)};
  io.v = {v, tensor_bytes(st, 1, n_new, st->cfg.num_kv_heads)};
  io.o = {O, tensor_bytes(st, 1, n_new, st->cfg.num_q_heads)};
  if ((rc = st->stage_inputs(&io, cs)) != SSA_OK) return rc;
  SegDesc sg{};
  sg.m = n_new;
  sg.tail_m = sg.m;
  st->fill_cached(*s, &sg);
  sg.append_slot0 = (int32_t)slot0;
  std::vector<SegDesc> segs{sg};
  RunOpts ro;
  ro.skip_scatter = true;   // the projection epilogue wrote K/V into the pages
  if ((rc = st->run(segs, io, n_new, layer, 1, 0, true, false, cs, ro)) != SSA_OK) return rc;
  s->ticket_done[layer] = 1;
  return SSA_OK;
}

ssa_status ssa_session_query_fused(ssa_store_t st, ssa_session_t id, int32_t layer, int32_t n_q, int32_t hidden,
                                   float rope_theta, const void* X, const void* W, void* O, void* stream) {
  SSA_CHECK_STORE(st);
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (layer < 0 || layer >= st->cfg.num_layers || !dev_ok(O, stream)) return SSA_ERR_INVALID_ARG;
  if (!qkv_args_ok(st, n_q, hidden, X, W, stream)) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  void *q, *k, *v;
  ssa_status rc = qkv_scratch(st, n_q, &q, &k, &v, (cudaStream_t)stream);
  if (rc != SSA_OK) return rc;
  cudaStream_t cs = (cudaStream_t)stream;
  const int64_t pos0 = s->n_tokens + s->n_evicted;   // query tokens follow the cache (R-8)
  if ((rc = qkv_launch(st, n_q, hidden, pos0, rope_theta, X, W, q, k, v, nullptr, 0, 0, cs)) != SSA_OK) return rc;
  return ssa_session_query(st, id, layer, n_q, q, k, v, O, stream);
}

int32_t ssa_debug_qkv_clusters(int32_t splits) { return qkv_max_active_clusters(splits); }
int32_t ssa_debug_tc_clusters(int32_t size, int32_t e4m3) { return tc_max_active_clusters(size, e4m3 != 0); }

/* experiments: per-CTA %globaltimer stamps of the next fused-projection launches */
int32_t ssa_debug_qkv_trace(void* device_buf) {
  g_qkv_trace = static_cast<uint64_t*>(device_buf);
  return 0;
}
