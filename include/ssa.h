/*
 * ssa.h — C ABI of the B200-native stateful-session attention library
 * (libssa.so), the data-parallel hot path of arXiv 2605.13784 ("stateful
 * sessions").  Citations "P:n" are lines of the paper text;
 * "R-n" are the readings listed in DESIGN.md §3.
 *
 * The paper's problem statement (§2): a context
 *     C = [S; D_1; ...; D_k]
 * of a static prefix S and appended data segments D_i, against which queries
 * Q_j are answered without re-processing C.  The library keeps C as a paged,
 * append-only KV cache per session and computes, on the GPU:
 *   - data plane:  the attention rows of each new segment D_k over all cached
 *                  keys plus D_k itself, causally (Alg. 1), and
 *                  appends D_k's K/V to the cache;
 *   - query plane: the attention rows of a query q (Alg. 2) or of
 *                  a batch of registered Flash Queries f_i (Eq. flash-eval
 *                  P:406, Alg. 3) over the same cache, without
 *                  changing it.
 * Attention is Eq. (attention), softmax(Q K^T / sqrt(d_k)) V, with the
 * cached-context decomposition of Eq. (query-attention) P:150-155.
 *
 * ----------------------------------------------------------------------------
 * Conventions (apply to every call)
 * ----------------------------------------------------------------------------
 * Tensors.  Q/K/V/O are plain pointers to contiguous row-major arrays
 *   [L'][n][H][d] of the store dtype (bf16 as uint16 bit patterns, or fp32),
 *   where L' = num_layers for all-layer calls (layer == -1) and L' = 1 for
 *   single-layer calls, n is the number of new tokens, H = num_q_heads for Q
 *   and O and num_kv_heads for K and V, d = head_dim.  Inputs are post-RoPE
 *   (R-6): positions only define order and causality.  Q head h attends with
 *   KV head h / (num_q_heads / num_kv_heads) (GQA, R-5).
 * Host or device.  Each pointer may be device memory or host memory (pinned
 *   or pageable); the library detects which.  Host inputs are copied to
 *   store-owned staging buffers on `stream`; a host O is copied back on
 *   `stream` — synchronize `stream` before reading it.
 * Streams.  `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *   stream).  All device work of a call is enqueued on it, in call order.  The
 *   store orders its calls across streams: a call on another stream than the
 *   previous call first waits (cudaStreamWaitEvent, no host sync) for the
 *   previous call's work, so pages released by truncate / destroy / evict,
 *   scratch and staging buffers are never reused while an earlier call on
 *   another stream may still read them (one dispatch order).
 * Ownership.  The caller owns Q/K/V/O and `stream` and keeps device buffers
 *   alive until the stream has passed the call.  The store owns the KV pool,
 *   page tables, staging and scratch memory, and its NCCL communicator.
 * Host metadata.  Page reservation, n_tokens and version change at call time
 *   (the device work that fills the pages is stream-ordered after it).
 * Errors.  Validation and capacity errors (INVALID_ARG, UNKNOWN_SESSION,
 *   POOL_EXHAUSTED, SESSION_LIMIT, UNSUPPORTED) return synchronously and leave
 *   NO state change; page reservation is all-or-none.  A CUDA or NCCL failure
 *   marks the store failed (sticky): every later call returns SSA_ERR_STATE.
 *   ssa_last_error() returns a message for the calling thread's last error.
 * CUDA graphs.  Query-plane calls (ssa_session_query, ssa_flash_query_batch,
 *   ssa_batch_run without APPEND items, the sharded partial/push/merge) and the
 *   per-layer data-plane step ssa_append_layer may be captured into a CUDA graph
 *   on a capturing `stream` with DEVICE pointers.  A replay repeats the call as
 *   planned at capture time (cache length, page table and, for
 *   ssa_append_layer, the ticket's destination slots of that moment): replay a
 *   captured ssa_append_layer only inside a ticket of the same session state
 *   (e.g. after truncating back to the captured length, ssa_append_begin
 *   reserves the same pages, lowest id first, R-9); a capture marks the layer
 *   appended for the ticket open at capture time.  Work lists come from the
 *   store's cache of call shapes (entries read by a graph are kept) or, for a
 *   shape never run eagerly, from a persistent 4 MiB arena written by a captured
 *   copy (SSA_OPT_GRAPH_ARENA_RESET recycles it once old graphs are dropped).
 *   Run the call once before capturing (scratch buffers are sized on first
 *   use).  Calls that change host state (create, append, begin, load, evict,
 *   alias) return SSA_ERR_STATE while the stream is capturing, no state change.
 * Threading.  One host thread at a time per store (external serialization —
 *   the paper's single dispatch worker).  Distinct stores are
 *   independent.  Sessions never see each other's keys.
 */
#ifndef SSA_H_
#define SSA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSA_ABI_VERSION 3   /* 3: ssa_debug_last_plan fills out[6]; SSA_OPT_CM_MERGE 2-5 */

typedef enum {
    SSA_OK = 0,
    SSA_ERR_INVALID_ARG = -1,     /* bad shape/pointer/argument; no state change */
    SSA_ERR_UNKNOWN_SESSION = -2, /* session id not live          */
    SSA_ERR_POOL_EXHAUSTED = -3,  /* not enough free pages           */
    SSA_ERR_SESSION_LIMIT = -4,   /* max_sessions live sessions already          */
    SSA_ERR_CUDA = -5,            /* CUDA runtime/launch failure (store failed)  */
    SSA_ERR_NCCL = -6,            /* NCCL failure (store failed)                 */
    SSA_ERR_UNSUPPORTED = -7,     /* shape/dtype not supported by this build     */
    SSA_ERR_STATE = -8            /* store previously failed, or call order bad  */
} ssa_status;

typedef enum { SSA_BF16 = 0, SSA_FP32 = 1 } ssa_dtype;

/* Store configuration.  The KV pool holds num_pages pages per layer; a page
 * is page_size token slots of one (layer, kv head) — see DESIGN.md §5 for the
 * HBM layout [L][num_pages][Hkv][page_size][d] of the K and V pools.
 * softmax_scale <= 0 selects 1/sqrt(head_dim) (Eq. attention; R-1). */
typedef struct {
    int32_t num_layers;
    int32_t num_q_heads;
    int32_t num_kv_heads;   /* must divide num_q_heads */
    int32_t head_dim;       /* fp32: <= 128; bf16: 64 or 128 */
    int32_t page_size;      /* power of two, 16..256 (R-9) */
    int64_t num_pages;      /* pages per layer */
    int32_t max_sessions;
    int32_t device;         /* CUDA device ordinal */
    ssa_dtype dtype;
    float softmax_scale;
    /* KV-cache storage format (FP8 KV is what the paper's
     * TRT-LLM baseline runs).  SSA_KV_E4M3 stores every cached K / V
     * element as the E4M3 code of x / k_scale (x / v_scale), the quotient rounded
     * once in fp32, then to nearest-even E4M3, saturating at +-448 (reading R-22);
     * attention uses code * scale for every key and value, the segment's own
     * tokens included.  Requires dtype SSA_BF16 (Q/K/V/O stay bf16 at the ABI),
     * head_dim 128, an sm_100 GPU, finite scales > 0.  Halves the pool and the
     * query plane's HBM bytes.  0 = SSA_KV_SAME (K/V stored in `dtype`). */
    int32_t kv_format;
    float k_scale;
    float v_scale;
    /* Optional caller-owned KV pool (e.g. a torch allocation, so the
     * framework's allocator owns device memory).  NULL: the store allocates the pool
     * with cudaMalloc.  Otherwise pool_ptr must be device memory of cfg->device, 256-byte
     * aligned, pool_bytes >= ssa_store_pool_bytes(cfg); K takes the first half and V
     * the second half of ssa_store_pool_bytes(cfg).  The store zero-fills it at creation,
     * never frees it, and the caller keeps it alive until ssa_store_destroy returns.
     * A pointer that fails these checks gives SSA_ERR_INVALID_ARG. */
    void *pool_ptr;
    size_t pool_bytes;
} ssa_store_config;

enum { SSA_KV_SAME = 0, SSA_KV_E4M3 = 1 };

typedef struct ssa_store *ssa_store_t;
typedef int32_t ssa_session_t;

/* Bytes of the K+V pools for `cfg`: 2 * L * num_pages * Hkv * page_size * d *
 * sizeof(dtype) (1 byte per element for SSA_KV_E4M3) — the paged form of Eq. (memory), with the GQA
 * KV width Hkv*d in place of the model dimension (R-13). 0 on bad config. */
size_t ssa_store_pool_bytes(const ssa_store_config *cfg);

/* Create a store on cfg->device: allocates and zero-fills the KV pools.
 * *out receives the handle.  INVALID_ARG on a bad config; CUDA on allocation
 * failure (nothing is leaked). */
ssa_status ssa_store_create(const ssa_store_config *cfg, ssa_store_t *out);

/* Synchronizes the device, then frees every resource of the store. */
ssa_status ssa_store_destroy(ssa_store_t store);

/* Pages in use / pages in the pool (per layer).  Occupancy in the paper's
 * "cells" is used_pages * page_size * num_layers slots. */
ssa_status ssa_store_occupancy(ssa_store_t store, int64_t *used_pages, int64_t *total_pages);

/* ----------------------------------------------------------------------------
 * Data plane
 * -------------------------------------------------------------------------- */

/* Create a session whose Region 0 (the static prefix S, processed once at
 * initialization) is the n_prefix tokens given.  Q/K/V: [L][n_prefix]
 * [H][d].  O (may be NULL): [L][n_prefix][Hq][d] — the causal self-attention
 * rows of S.  K/V are written into freshly reserved pages (lowest free page
 * id first; R0 is padded to a page boundary, R-9).  version becomes 1.
 * Errors: INVALID_ARG (n_prefix <= 0, NULL K/V), SESSION_LIMIT,
 * POOL_EXHAUSTED. */
ssa_status ssa_session_create(ssa_store_t store, int32_t n_prefix,
                              const void *Q, const void *K, const void *V, void *O,
                              void *stream, ssa_session_t *out);

/* Append data segment D_k of n_new tokens (Alg. 1 "K.append(Forward(
 * tokens, K))"; "only the delta is processed and appended"):
 * computes the attention rows of D_k over the cached keys and D_k itself
 * (row t sees new tokens 0..t, R-2), writes O (may be NULL), scatters D_k's
 * K/V into the session's pages (bit-exact copy), commits n_tokens += n_new
 * and version += 1.  Q/K/V/O: [L][n_new][H][d].  *new_version may be
 * NULL.  Errors: INVALID_ARG (n_new <= 0), UNKNOWN_SESSION, POOL_EXHAUSTED. */
ssa_status ssa_session_append(ssa_store_t store, ssa_session_t session, int32_t n_new,
                              const void *Q, const void *K, const void *V, void *O,
                              void *stream, uint64_t *new_version);

/* Per-layer form for a model whose layer l+1 input depends on layer l's O:
 * begin reserves the pages for n_new tokens (all-or-none) and returns a
 * ticket; layer(l) computes layer l's rows and scatters its K/V (Q/K/V/O:
 * [1][n_new][H][d]); commit publishes n_tokens/version after every layer was
 * run exactly once.  abort releases the reservation (no state change).
 * Only one open ticket per session; errors: STATE on misuse. */
ssa_status ssa_append_begin(ssa_store_t store, ssa_session_t session, int32_t n_new,
                            int32_t *ticket);
ssa_status ssa_append_layer(ssa_store_t store, ssa_session_t session, int32_t ticket,
                            int32_t layer, const void *Q, const void *K, const void *V,
                            void *O, void *stream);
ssa_status ssa_append_commit(ssa_store_t store, ssa_session_t session, int32_t ticket,
                             uint64_t *new_version);
ssa_status ssa_append_abort(ssa_store_t store, ssa_session_t session, int32_t ticket);

/* SeqRemove(s, p, inf) (Alg. 3 L540/L547): drop tokens at positions
 * >= p (0 <= p <= n_tokens), free pages no longer needed (the first page is
 * kept if any slot of it is still used), version += 1 when tokens were
 * removed.  Host metadata only. */
ssa_status ssa_session_truncate(ssa_store_t store, ssa_session_t session, int64_t p,
                                uint64_t *new_version);

/* Region-1 FIFO eviction, K.evict_oldest(|tokens|) of Alg. 1: drop
 * the n_tokens oldest retained Region-1 tokens (Region 0 is frozen, P:186;
 * SPEC kv-store evict_oldest).  Positions of the remaining tokens are not
 * re-based (R-8); they keep their order and the digest records their original
 * positions.  Pages whose slots are all evicted leave the page table and
 * return to the pool once no alias references them; the device page table is
 * updated on `stream`.  version += 1 when n_tokens > 0.  Errors (no state
 * change): SSA_ERR_INVALID_ARG if n_tokens < 0 or exceeds the retained
 * Region-1 tokens; SSA_ERR_STATE with an append ticket open. */
ssa_status ssa_session_evict_oldest(ssa_store_t store, ssa_session_t session, int64_t n_tokens,
                                    void *stream, uint64_t *new_version);

/* Retention window of Region 1 ("configurable retention"): with
 * max_tokens > 0 every later append of m tokens (session_append, append_begin,
 * batch APPEND items, load_kv) first evicts m oldest Region-1 tokens when
 * n_tokens + m > max_tokens -- the guard of Alg. 1 L279-281.  The append
 * fails with SSA_ERR_INVALID_ARG and no state change when fewer than m
 * Region-1 tokens are retained.  0 disables the guard. */
ssa_status ssa_session_set_retention(ssa_store_t store, ssa_session_t session, int64_t max_tokens);

/* Metadata-only prefix aliasing (Eq. T_restore; SPEC
 * kv-store alias_prefix): create a new session whose first len_tokens tokens
 * are the donor's first len_tokens tokens, by reference.  Whole pages are
 * shared (reference counted; a page returns to the pool when its last referer
 * releases it); the one page that holds tokens past len_tokens, if any, is
 * copied (one page per layer: constant in len_tokens), so appends to either
 * session never disturb the other.  The new session's Region 0 is
 * min(len_tokens, donor Region 0); version 0.  Requires 0 <= len_tokens <=
 * donor n_tokens and, when len_tokens reaches into Region 1, a donor with no
 * evictions (the prefix must be contiguous from the start).  Errors:
 * SSA_ERR_UNKNOWN_SESSION, SSA_ERR_INVALID_ARG, SSA_ERR_SESSION_LIMIT,
 * SSA_ERR_POOL_EXHAUSTED (no state change); copies are enqueued on `stream`. */
ssa_status ssa_session_alias_prefix(ssa_store_t store, ssa_session_t donor, int64_t len_tokens,
                                    void *stream, ssa_session_t *out);

/* Destroy a session, returning its pages to the pool. */
ssa_status ssa_session_destroy(ssa_store_t store, ssa_session_t session);

/* ----------------------------------------------------------------------------
 * Query plane — never changes pages, page table, n_tokens or version (R-3)
 * -------------------------------------------------------------------------- */

/* Query q of n_q tokens (Alg. 2 "Forward(tokens_q, K)  O(|q|) not
 * O(|K|)") against the session's cache: row t sees every cached token
 * and q's tokens 0..t.  q's own K/V are read from the K/V arguments (Region 2
 * scratch, "cleared between queries") and never written to pages.
 * layer == -1: all layers, Q/K/V/O [L][n_q][H][d]; else that layer only,
 * [1][n_q][H][d]. */
ssa_status ssa_session_query(ssa_store_t store, ssa_session_t session, int32_t layer,
                             int32_t n_q, const void *Q, const void *K, const void *V,
                             void *O, void *stream);

/* Flash Query batch (Eq. flash-eval; Alg. 3): k registered
 * questions f_1..f_k evaluated against cache version t in ONE launch; f_i
 * sees the cache plus its own tokens only, never another f_j (R-4).
 * q_lens (host, k entries > 0); Q/K/V/O are packed varlen over the questions
 * in order: [L'][sum q_lens][H][d], L' as for ssa_session_query. */
ssa_status ssa_flash_query_batch(ssa_store_t store, ssa_session_t session, int32_t layer,
                                 int32_t k, const int32_t *q_lens, const void *Q,
                                 const void *K, const void *V, void *O, void *stream);

/* ----------------------------------------------------------------------------
 * Multi-tenant varlen batch (admit-many / run-few; R-7)
 * -------------------------------------------------------------------------- */
typedef enum {
    SSA_WORK_APPEND = 0,     /* data-plane append D_k of `session`           */
    SSA_WORK_QUERY = 1,      /* query-plane rows of `session`, no state change */
    SSA_WORK_STATELESS = 2   /* stateless prompt: causal prefill over its own
                                tokens only, K/V discarded (R-16) */
} ssa_work_kind;

typedef struct {
    int32_t kind;            /* ssa_work_kind */
    ssa_session_t session;   /* ignored for STATELESS */
    int32_t n_tokens;        /* > 0 */
    int32_t reserved;
    int64_t row_offset;      /* first token row of this item in Q/K/V/O */
} ssa_work_item;

/* Run n_items heterogeneous items in one launch per layer.  Q/K/V/O are packed
 * [L'][n_rows][H][d] with n_rows = max(row_offset + n_tokens) and L' as for
 * ssa_session_query.  Snapshot semantics (R-7): every item reads the cache as
 * of the call; APPEND items reserve their pages in item order (all-or-none
 * over the batch) and publish n_tokens/version when the call returns (layer ==
 * -1) or on the call for layer num_layers-1 (per-layer use: call layers 0..L-1
 * in order with the same items).  At most one APPEND item per session. */
ssa_status ssa_batch_run(ssa_store_t store, int32_t layer, int32_t n_items,
                         const ssa_work_item *items, const void *Q, const void *K,
                         const void *V, void *O, void *stream);

/* ----------------------------------------------------------------------------
 * Fused data-plane projection before attention
 * -------------------------------------------------------------------------- */
/* The `Forward` of Alg. 1 L282 up to the attention inputs, for a
 * Llama-shaped layer (the paper's model):
 *     [Q | K | V] = X W^T,   Q, K <- RoPE(., pos),   V unchanged,
 * with X [n][hidden] bf16 token rows and W the nn.Linear weight
 * [(num_q_heads + 2 num_kv_heads) * head_dim][hidden] bf16 (rows: the Q heads,
 * then the K heads, then the V heads).  RoPE is the rotate-half form (R-21):
 * for pair j < head_dim/2 of a head, angle = pos * rope_theta^(-2j/head_dim),
 *     x'[j]       = x[j] cos - x[j + head_dim/2] sin,
 *     x'[j + d/2] = x[j + d/2] cos + x[j] sin;
 * rope_theta <= 0 disables it.  fp32 accumulation, one bf16 rounding (RNE).
 * Requires a bf16 store with head_dim 128, hidden % 64 == 0, an sm_100 GPU;
 * X, W and all outputs are DEVICE pointers.  One launch (tcgen05 GEMM with
 * split-K over a thread-block cluster and a RoPE / store epilogue).
 *
 * ssa_qkv_rope: token row i has position pos0 + i; writes Q [n][Hq][d] and
 *   K, V [n][Hkv][d].  No store state is read or changed.
 * ssa_append_layer_fused: the per-layer append of an open ticket (as
 *   ssa_append_layer) whose Q/K/V come from X: positions continue the session
 *   (n_tokens + evicted tokens, never re-based, R-8); the projection epilogue
 *   writes K and V straight into the ticket's pages (no scatter launch; E4M3
 *   codes of the bf16-rounded values on an SSA_KV_E4M3 store), then
 *   the data-plane attention writes O [n_new][Hq][d].
 * ssa_session_query_fused: ssa_session_query for one layer with Q/K/V from
 *   X [n_q][hidden] at the positions after the cache; no state change.
 * Errors: SSA_ERR_INVALID_ARG (shape, dtype, host pointers), as
 *   ssa_append_layer / ssa_session_query otherwise.  Q/K/V scratch of the
 *   fused calls is store-owned. */
ssa_status ssa_qkv_rope(ssa_store_t store, int32_t n, int32_t hidden, int64_t pos0,
                        float rope_theta, const void *X, const void *W, void *Q, void *K,
                        void *V, void *stream);
ssa_status ssa_append_layer_fused(ssa_store_t store, ssa_session_t session, int32_t ticket,
                                  int32_t layer, int32_t hidden, float rope_theta,
                                  const void *X, const void *W, void *O, void *stream);
ssa_status ssa_session_query_fused(ssa_store_t store, ssa_session_t session, int32_t layer,
                                   int32_t n_q, int32_t hidden, float rope_theta,
                                   const void *X, const void *W, void *O, void *stream);

/* ----------------------------------------------------------------------------
 * On-device greedy sampling
 * -------------------------------------------------------------------------- */
/* For each of n_rows rows of `vocab` logits (dtype SSA_FP32 or SSA_BF16, row r
 * at logits + r * row_stride elements): out_ids[r] = argmax with ties broken
 * toward the lowest id (SPEC greedy_sample), out_gap[r] = l1 - l2 computed in
 * fp32, the logit gap of Eq. flash-cache / Eq. logit-gap
 * (P:454-457), where l2 is the second-highest VALUE (equal to l1 when the top
 * value occurs twice, so the gap is 0), and optionally out_top2[2r..2r+1] =
 * (l1, l2).  NaN logits are ignored; a row with no non-NaN logit gives id -1
 * and gap 0.  With `draft` (n_rows proposed ids) *out_n_accept = the number of
 * leading rows whose argmax equals the draft (the batched speculative check of
 * P:385).  All pointers are device pointers; out_gap, out_top2, draft may be
 * NULL.  One launch on `stream`, one read of the logits (HBM-bound); the
 * store provides scratch.  Errors: SSA_ERR_INVALID_ARG. */
ssa_status ssa_greedy_sample(ssa_store_t store, ssa_dtype dtype, int32_t n_rows, int32_t vocab,
                             int64_t row_stride, const void *logits, int32_t *out_ids, float *out_gap,
                             float *out_top2, const int32_t *draft, int32_t *out_n_accept, void *stream);

/* ----------------------------------------------------------------------------
 * Introspection (tests, not hot path)
 * -------------------------------------------------------------------------- */
typedef struct {
    int64_t n_tokens;   /* retained tokens */
    int64_t n_prefix;   /* Region 0 length */
    int64_t n_pages;    /* pages held (per layer) */
    uint64_t version;   /* data version t */
    int64_t n_evicted;  /* Region-1 tokens evicted so far (positions are not re-based) */
    int64_t retention;  /* Region-1 retention window (0 = unlimited) */
} ssa_session_info;

ssa_status ssa_session_get_info(ssa_store_t store, ssa_session_t session, ssa_session_info *out);

/* Copy the session's page table (int32 page ids, in slot order) to host
 * `out` (capacity `cap`); *n_out = number of entries. */
ssa_status ssa_session_page_table(ssa_store_t store, ssa_session_t session, int32_t *out,
                                  int64_t cap, int64_t *n_out);

/* Gather tokens [start, start+count) of `layer` from the pages into
 * K_out/V_out [count][Hkv][d] (host or device), bit-exact; synchronous.
 * SSA_KV_E4M3 stores return the E4M3 codes (1 byte per element). */
ssa_status ssa_session_read_kv(ssa_store_t store, ssa_session_t session, int32_t layer,
                               int64_t start, int64_t count, void *K_out, void *V_out);

/* Bulk import of `count` tokens appended to the session without computing
 * attention (building a long session, e.g. the 128k split-KV config):
 * K/V [L][count][Hkv][d].  Reserves pages, scatters, version += 1. */
ssa_status ssa_session_load_kv(ssa_store_t store, ssa_session_t session, int64_t count,
                               const void *K, const void *V, void *stream);

/* FNV-1a-64 digest of the retained K/V: over layers, then tokens, the
 * records int32 LE layer || int64 LE token || K bytes || V bytes (SPEC
 * S:158-166) -- the stored bytes, i.e. E4M3 codes for an
 * SSA_KV_E4M3 store.  Reads the pages back; synchronous. */
ssa_status ssa_session_digest(ssa_store_t store, ssa_session_t session, uint64_t *out);

/* Counters since store creation (or the last reset). */
typedef struct {
    int64_t kernel_launches;     /* kernels this library launched */
    int64_t rows_computed;       /* attention rows = tokens * num_q_heads * layers */
    int64_t query_rows;          /* subset of rows_computed from the query plane */
    int64_t tokens_appended;     /* tokens written to pages (per layer counted once) */
    int64_t pages_reserved;
    int64_t h2d_bytes;           /* host staging copies */
    int64_t d2h_bytes;
    int64_t tc_launches;         /* attention launches on the tcgen05 kernel */
    int64_t cm_launches;         /* of which cluster-merge launches (split-KV merged
                                    in the kernel: no partials in HBM unless a group
                                    spans several clusters, no combine launch) */
    int64_t plan_uploads;        /* work lists planned and copied to the device (a
                                    repeated call shape reuses the device copy) */
} ssa_stats;

ssa_status ssa_store_stats(ssa_store_t store, ssa_stats *out, int32_t reset);

/* Options (tests / benchmarking). */
typedef enum {
    SSA_OPT_ATTN_BACKEND = 1,   /* 0 auto, 1 SIMT kernels only, 2 tcgen05 when eligible */
    SSA_OPT_MAX_SPLITS = 2,     /* cap on split-KV factor (0 = auto) */
    SSA_OPT_FAULT_INJECT = 3,   /* negative controls: 0 none, 1 drop last key tile,
                                   2 causal off-by-one (row t misses its own key) */
    SSA_OPT_TC_Q_TILES = 4,     /* accepted for compatibility; no effect */
    SSA_OPT_TIMING = 5,         /* 1: record CUDA events around every kernel launch
                                   (on the call's stream) for ssa_store_timing */
    /* 6, 7: removed in ABI 2 (in-kernel merge is now the cluster merge below;
       the cta_group::2 kernel was slower than the two-slot kernel) */
    SSA_OPT_GRAPH_ARENA_RESET = 8, /* value 1: recycle the CUDA-graph arena and unpin the
                                   cached work lists (the caller no longer replays
                                   graphs captured before this call) */
    SSA_OPT_CLUSTER = 9,        /* split-KV merge of single-layer tcgen05 calls: 0 (default)
                                   cluster size from the planner's cost model over
                                   C in 1..8 and 16; 1..8 or 16 force C; -1 no cluster
                                   plan (LPT plan, split groups merged across CTAs) */
    SSA_OPT_PDL = 10,           /* 1 (default): tcgen05 attention launches allow
                                   programmatic dependent launch (prologue overlaps
                                   the previous kernel); 0: plain stream order */
    SSA_OPT_PIPE_CHUNKS = 11,   /* all-layer calls with host buffers: -1 no copy/compute
                                   pipelining, 0 default (2 layer chunks), n chunks */
    SSA_OPT_QKV_DEBUG = 12,     /* fused projection experiments: 0 off, 1 skip the epilogue */
    SSA_OPT_CM_MERGE = 13,      /* split-KV merge of single-layer tcgen05 calls: 2 (default)
                                   query-plane calls take the group plan when it fits one
                                   wave of single CTAs: every CTA of a group writes its
                                   partial and exits, a small merge kernel launched right
                                   behind (programmatic launch) merges each group; other
                                   calls as 1; 3 the group plan for data-plane calls too;
                                   4 / 5 as 2 / 3 but the group's CTAs meet at a barrier in
                                   global memory and merge inside the attention kernel;
                                   1 cluster plans, groups over several clusters merged by
                                   a separate kernel; 0 as 1 but the last arriving CTA
                                   merges inside the attention kernel.  With
                                   SSA_OPT_CLUSTER > 0 the cluster plans */
    SSA_OPT_L2_HINT = 14,       /* KV pool tiles loaded with an L2 evict-first hint: 0 (default)
                                   when no key tile of the launch is read by two CTAs, 1 never,
                                   2 always */
} ssa_option;
ssa_status ssa_store_set_option(ssa_store_t store, int32_t option, int64_t value);

/* Shape of the store's last attention launch (a test / tuning aid):
 * out[0] work units, [1] split groups, [2] CTAs per layer, [3] cluster size of a
 * cluster-merge launch (0: combine kernel or SIMT), [4] largest split count
 * (clusters per group for a cluster-merge launch), [5] 1 for a group plan (single CTAs
 * in one wave, SSA_OPT_CM_MERGE 2-5: merged by the merge kernel or the group barrier). */
ssa_status ssa_debug_last_plan(ssa_store_t store, int64_t out[6]);

/* Kernel timing recorded while SSA_OPT_TIMING is on, per kernel class
 * (SSA_TIMING_KINDS entries): [0] data-plane attention (create/append/batch),
 * [1] query-plane attention (query/flash/sharded), [2] data-plane split-KV
 * combine, [3] query-plane combine, [4] KV append scatter, [5] fused QKV
 * projection + RoPE (ssa_qkv_rope and the *_fused calls), [6] E4M3
 * quantization of a call's K/V (SSA_KV_E4M3 stores).
 * ms[i] = summed device time of launches of class i, count[i] = launches.
 * Synchronizes the recorded events; reset != 0 clears the record. */
#define SSA_TIMING_KINDS 7
ssa_status ssa_store_timing(ssa_store_t store, double ms[SSA_TIMING_KINDS],
                            int64_t count[SSA_TIMING_KINDS], int32_t reset);

/* Kernel-internal timestamps of a trace build (compiled with -DSSA_TRACE; a
 * profiling aid, not part of the method): copies the clock64 record of the
 * tcgen05 kernels' softmax / MMA-issuer events for the first CTAs of layer 5
 * into `host` (`bytes` capacity): the two-slot kernel's record, followed by the
 * CTA-pair kernel's if it fits.  Returns the bytes written, 0 in a normal
 * build, -1 if `bytes` is too small or the copy fails.  Synchronous. */
int32_t ssa_debug_trace(void *host, size_t bytes);

/* Occupancy probe of the fused-projection kernel (a tuning aid): the number of
 * thread-block clusters of `splits` CTAs that can be co-resident on the current
 * device (cudaOccupancyMaxActiveClusters), or -1 on error. */
int32_t ssa_debug_qkv_clusters(int32_t splits);

/* Occupancy probe of the tcgen05 attention kernel: co-resident thread-block
 * clusters of `size` CTAs (one CTA per SM) on the current device, for the bf16
 * (e4m3 = 0) or E4M3 variant; what the cluster-merge planner sizes plans by. */
int32_t ssa_debug_tc_clusters(int32_t size, int32_t e4m3);
/* Tuning aid: when `device_buf` is non-NULL the following fused-projection
 * launches write per-CTA %globaltimer stamps (uint64 [grid][8]: start, after
 * setup, accumulator ready, partial dumped, cluster synced, epilogue done,
 * exit) into it; NULL turns it off.  Returns 0. */
int32_t ssa_debug_qkv_trace(void *device_buf);

/* ----------------------------------------------------------------------------
 * Multi-GPU split-KV for one long session (R-12)
 * -------------------------------------------------------------------------- */
/* NCCL unique id (128 bytes) for rank 0 to broadcast through any channel
 * (e.g. a torch.distributed process group). */
ssa_status ssa_comm_unique_id(uint8_t out[128]);

/* Join the store to a `world`-rank NCCL communicator on its device. */
ssa_status ssa_comm_init(ssa_store_t store, int32_t rank, int32_t world, const uint8_t id[128]);

/* Query against a session sharded by contiguous token ranges over the ranks
 * (each rank's store holds its shard as an ordinary session, rank r holding
 * tokens [r*n/G, (r+1)*n/G)).  Each rank computes the partial (O_r, lse_r)
 * of all n_q rows over its shard; the tail owner (rank world-1) also covers
 * q's own tokens; partials are exchanged with one ncclAllGather on `stream`
 * and merged (log-sum-exp) so every rank returns the full O. */
ssa_status ssa_sharded_query(ssa_store_t store, ssa_session_t session, int32_t layer,
                             int32_t n_q, const void *Q, const void *K, const void *V,
                             void *O, void *stream);

ssa_status ssa_comm_destroy(ssa_store_t store);

/* A9 over peer memory instead of NCCL: the rank partial is pushed straight
 * into every rank's gathered buffer by the kernel that produces it (NVLink
 * P2P stores from the split-KV combine epilogue), a system-scope release of a
 * per-rank epoch flag follows on the same stream, and each rank's merge waits
 * (acquire, one spinning block) for all flags of the epoch -- no collective
 * launch, no staging copy.  peer_bufs[q] / peer_flags[q] (host arrays of `world`
 * device addresses valid in this process, e.g. from torch symmetric memory) are
 * rank q's gathered buffer ([2][world][chunk] fp32, buf_bytes each, chunk =
 * rows*Hq*(D+1) as in ssa_sharded_partial; epoch e uses half e & 1) and its
 * uint32 flag array [2][world] (zero-initialised): ready[p] = the last epoch rank
 * p pushed into this buffer, ack[p] = the last epoch rank p finished merging.  A
 * push of epoch e first waits for every peer's ack of e - 2 (the merge that last
 * read that half), so ranks may run any number of push/merge rounds back to back
 * without a barrier; a rank alternates push and merge, and the chunk size is
 * fixed after the first push.  Replaces any NCCL communicator.  After attaching,
 * ssa_sharded_query = ssa_sharded_push + ssa_sharded_merge.  A peer that never
 * signals fails the waiting launch after 10 s (sticky CUDA error) instead of
 * hanging.  Errors: SSA_ERR_INVALID_ARG (null / out-of-range / buffers too
 * small), SSA_ERR_STATE (not attached, push without merge, merge without push). */
ssa_status ssa_comm_attach_peers(ssa_store_t store, int32_t rank, int32_t world, const uint64_t *peer_bufs,
                                 const uint64_t *peer_flags, size_t buf_bytes);
ssa_status ssa_sharded_push(ssa_store_t store, ssa_session_t session, int32_t layer, int32_t n_q,
                            const void *Q, const void *K, const void *V, void *stream);
ssa_status ssa_sharded_merge(ssa_store_t store, int32_t layer, int32_t n_q, void *O, void *stream);

/* Building blocks of ssa_sharded_query, usable without NCCL.
 * ssa_sharded_partial: the rank partial of the n_q query rows over this
 * store's shard of the session (include_tail != 0: this rank also covers the
 * query's own tokens, i.e. it is the tail owner).  Writes one packed chunk of
 * rows*Hq*(d+1) floats to device memory `part`: O fp32 [L'][n_q][Hq][d] (each
 * row normalized over the shard) followed by lse [L'][n_q][Hq] in log2 units
 * (-inf for a row with no visible key on this shard).
 * ssa_merge_rank_partials: merges `world` consecutive chunks (device) into O
 * (log-sum-exp, R-11); rows = L' * n_q. */
ssa_status ssa_sharded_partial(ssa_store_t store, ssa_session_t session, int32_t layer, int32_t n_q,
                               const void *Q, const void *K, const void *V, int32_t include_tail,
                               float *part, void *stream);
ssa_status ssa_merge_rank_partials(ssa_store_t store, int32_t world, int64_t rows, const float *parts,
                                   void *O, void *stream);

/* ----------------------------------------------------------------------------
 * Diagnostics
 * -------------------------------------------------------------------------- */
const char *ssa_status_str(ssa_status s);
const char *ssa_last_error(void);
int32_t ssa_abi_version(void);

/* Host-only planner introspection (tests; no GPU needed): plans the split-KV
 * work units for n_segs segments of seg_m[i] new tokens over seg_slots[i]
 * cached slots and writes up to cap_units units as 8 int32 each
 * (seg, kv_head, q_tok0, q_ntok, tile_lo, tile_hi, group, split) into
 * units_out (may be NULL).  key_tile == 128 (the tcgen05 key tile) plans for
 * two-slot tcgen05 CTAs, where a lone one-q-tile unit is split in two so
 * that its halves share a CTA.  Returns the number of units. */
int32_t ssa_debug_plan(int32_t n_segs, const int32_t *seg_m, const int32_t *seg_slots,
                       int32_t Hkv, int32_t q_tile_tokens, int32_t key_tile, int32_t n_layers,
                       int32_t num_sms, int32_t ctas_per_sm, int32_t max_splits,
                       int32_t *units_out, int32_t cap_units);

#ifdef __cplusplus
}
#endif
#endif /* SSA_H_ */
