// comm.cpp — multi-GPU split-KV query for one long session (§8(a) row A9,
// reading R-12): each rank holds a contiguous token shard of the session in
// its own store; it computes the rank partial (O fp32, lse) of every query row
// over its shard (the last rank also over the query's own tokens), the packed
// partials are exchanged with one ncclAllGather on the caller's stream over
// NVLink/NVSwitch, and every rank merges them (log-sum-exp, reading R-11).
//
// NCCL is loaded with dlopen("libnccl.so.2"): inside a torch process this
// resolves to the NCCL torch already loaded; standalone, to the system one.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "store.h"

using namespace ssa;

typedef ncclResult_t (*GetUniqueIdFn)(ncclUniqueId*);
typedef ncclResult_t (*CommInitRankFn)(ncclComm_t*, int, ncclUniqueId, int);
typedef ncclResult_t (*AllGatherFn)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
typedef ncclResult_t (*CommDestroyFn)(ncclComm_t);
typedef const char* (*ErrStrFn)(ncclResult_t);

namespace {
struct NcclApi {
  void* lib = nullptr;
  GetUniqueIdFn get_unique_id = nullptr;
  CommInitRankFn comm_init_rank = nullptr;
  AllGatherFn all_gather = nullptr;
  CommDestroyFn comm_destroy = nullptr;
  ErrStrFn err_str = nullptr;
  bool ok() const { return get_unique_id && comm_init_rank && all_gather && comm_destroy; }
};

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.lib = dlopen(n, RTLD_NOW | RTLD_LOCAL);
      if (api.lib) break;
    }
    if (api.lib) {
      api.get_unique_id = (GetUniqueIdFn)dlsym(api.lib, "ncclGetUniqueId");
      api.comm_init_rank = (CommInitRankFn)dlsym(api.lib, "ncclCommInitRank");
      api.all_gather = (AllGatherFn)dlsym(api.lib, "ncclAllGather");
      api.comm_destroy = (CommDestroyFn)dlsym(api.lib, "ncclCommDestroy");
      api.err_str = (ErrStrFn)dlsym(api.lib, "ncclGetErrorString");
    }
  }
  return api;
}

ssa_status nccl_fail(ssa_store* st, ncclResult_t r, const char* what) {
  const char* msg = nccl().err_str ? nccl().err_str(r) : "?";
  if (st) {
    st->failed = true;
    st->fail_msg = std::string("NCCL ") + what + ": " + msg;
  }
  set_error("NCCL %s failed: %s", what, msg);
  return SSA_ERR_NCCL;
}
}  // namespace

struct CommState {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  float* buf = nullptr;     // [send chunk | world gathered chunks]
  size_t cap = 0;           // floats
  // peer-memory path (ssa_comm_attach_peers): every rank's gathered buffer
  // [2][world][chunk] floats (halves alternate by epoch parity) and flag array
  // [2][world] uint32 (ready[q]: last epoch rank q pushed here; ack[q]: last
  // epoch rank q finished merging), mapped in this process
  bool peers = false;
  std::vector<uint64_t> peer_buf, peer_flag;
  size_t peer_bytes = 0;
  uint64_t* d_peer_flag = nullptr;   // device copy of peer_flag
  uint64_t* d_peer_chunk = nullptr;  // device: [2][world] this rank's chunk slot in every peer buffer half
  int64_t chunk_for = -1;            // chunk size d_peer_chunk was built for
  uint32_t epoch = 0;                // last pushed epoch
  uint32_t merged = 0;               // last merged epoch
};

void ssa_store::destroy_comm() {
  if (!comm) return;
  if (comm->comm && nccl().comm_destroy) nccl().comm_destroy(comm->comm);
  if (comm->buf) cudaFree(comm->buf);
  if (comm->d_peer_flag) cudaFree(comm->d_peer_flag);
  if (comm->d_peer_chunk) cudaFree(comm->d_peer_chunk);
  delete comm;
  comm = nullptr;
}

static ssa_status check_store(ssa_store* st) {
  if (!st) { set_error("null store"); return SSA_ERR_INVALID_ARG; }
  if (st->failed) { set_error("store failed earlier: %s", st->fail_msg.c_str()); return SSA_ERR_STATE; }
  return SSA_OK;
}

#define COMM_CUDA(st, expr)                                              \
  do {                                                                   \
    cudaError_t _e = (expr);                                             \
    if (_e != cudaSuccess) return (st)->cuda_fail(_e, #expr, __LINE__);  \
  } while (0)

extern "C" {

ssa_status ssa_comm_unique_id(uint8_t out[128]) {
  if (!out) return SSA_ERR_INVALID_ARG;
  if (!nccl().ok()) { set_error("libnccl.so.2 not loadable"); return SSA_ERR_UNSUPPORTED; }
  ncclUniqueId id;
  ncclResult_t r = nccl().get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail(nullptr, r, "ncclGetUniqueId");
  static_assert(sizeof(id.internal) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out, id.internal, 128);
  return SSA_OK;
}

ssa_status ssa_comm_init(ssa_store_t st, int32_t rank, int32_t world, const uint8_t* id) {
  ssa_status rc = check_store(st);
  if (rc != SSA_OK) return rc;
  if (!id || world <= 0 || rank < 0 || rank >= world) return SSA_ERR_INVALID_ARG;
  if (!nccl().ok()) { set_error("libnccl.so.2 not loadable"); return SSA_ERR_UNSUPPORTED; }
  cudaSetDevice(st->cfg.device);
  st->destroy_comm();
  ncclUniqueId uid;
  memcpy(uid.internal, id, 128);
  CommState* cs = new CommState();
  ncclResult_t r = nccl().comm_init_rank(&cs->comm, world, uid, rank);
  if (r != ncclSuccess) {
    delete cs;
    return nccl_fail(st, r, "ncclCommInitRank");
  }
  cs->rank = rank;
  cs->world = world;
  st->comm = cs;
  return SSA_OK;
}

ssa_status ssa_comm_destroy(ssa_store_t st) {
  if (!st) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  st->destroy_comm();
  return SSA_OK;
}

ssa_status ssa_sharded_partial(ssa_store_t st, ssa_session_t id, int32_t layer, int32_t n_q, const void* Q,
                               const void* K, const void* V, int32_t include_tail, float* part, void* stream) {
  ssa_status rc = check_store(st);
  if (rc != SSA_OK) return rc;
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (n_q <= 0 || !Q || !K || !V || !part || layer < -1 || layer >= st->cfg.num_layers) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  cudaStream_t cs = (cudaStream_t)stream;
  const int64_t Lin = layer < 0 ? st->cfg.num_layers : 1;
  const int64_t rows = Lin * n_q;
  const size_t el = st->elem;
  IoSet io;
  io.q = {Q, (size_t)rows * st->cfg.num_q_heads * st->cfg.head_dim * el};
  io.k = {K, (size_t)rows * st->cfg.num_kv_heads * st->cfg.head_dim * el};
  io.v = {V, (size_t)rows * st->cfg.num_kv_heads * st->cfg.head_dim * el};
  if ((rc = st->stage_inputs(&io, cs)) != SSA_OK) return rc;
  SegDesc sg{};
  sg.row0 = 0;
  sg.m = n_q;
  sg.tail_m = include_tail ? n_q : 0;
  st->fill_cached(*s, &sg);
  sg.append_slot0 = -1;
  std::vector<SegDesc> segs{sg};
  RunOpts opts;
  opts.force_groups = true;
  opts.o_f32 = part;
  opts.lse_out = part + rows * st->cfg.num_q_heads * st->cfg.head_dim;
  return st->run(segs, io, n_q, layer < 0 ? 0 : layer, (int32_t)Lin, 1, true, true, cs, opts);
}

ssa_status ssa_merge_rank_partials(ssa_store_t st, int32_t world, int64_t rows, const float* parts, void* O,
                                   void* stream) {
  ssa_status rc = check_store(st);
  if (rc != SSA_OK) return rc;
  if (world <= 0 || rows <= 0 || !parts || !O) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  cudaStream_t cs = (cudaStream_t)stream;
  IoSet io;
  io.o = {O, (size_t)rows * st->cfg.num_q_heads * st->cfg.head_dim * st->elem};
  if ((rc = st->stage_inputs(&io, cs)) != SSA_OK) return rc;
  COMM_CUDA(st, launch_merge_ranks(parts, world, rows, st->cfg.num_q_heads, st->cfg.head_dim, io.o.dev,
                                   st->cfg.dtype == SSA_BF16, cs));
  st->stats.kernel_launches++;
  return st->unstage_output(&io, cs);
}

ssa_status ssa_comm_attach_peers(ssa_store_t st, int32_t rank, int32_t world, const uint64_t* peer_bufs,
                                 const uint64_t* peer_flags, size_t buf_bytes) {
  ssa_status rc = check_store(st);
  if (rc != SSA_OK) return rc;
  if (world <= 0 || rank < 0 || rank >= world || !peer_bufs || !peer_flags || buf_bytes == 0) return SSA_ERR_INVALID_ARG;
  for (int q = 0; q < world; ++q)
    if (!peer_bufs[q] || !peer_flags[q]) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  st->destroy_comm();
  CommState* c = new CommState();
  c->rank = rank;
  c->world = world;
  c->peers = true;
  c->peer_buf.assign(peer_bufs, peer_bufs + world);
  c->peer_flag.assign(peer_flags, peer_flags + world);
  c->peer_bytes = buf_bytes;
  st->comm = c;
  COMM_CUDA(st, cudaMalloc(&c->d_peer_flag, world * sizeof(uint64_t)));
  COMM_CUDA(st, cudaMalloc(&c->d_peer_chunk, 2 * world * sizeof(uint64_t)));
  COMM_CUDA(st, cudaMemcpy(c->d_peer_flag, peer_flags, world * sizeof(uint64_t), cudaMemcpyHostToDevice));
  return SSA_OK;
}

ssa_status ssa_sharded_push(ssa_store_t st, ssa_session_t id, int32_t layer, int32_t n_q, const void* Q,
                            const void* K, const void* V, void* stream) {
  ssa_status rc = check_store(st);
  if (rc != SSA_OK) return rc;
  CommState* c = st->comm;
  if (!c || !c->peers) { set_error("sharded_push: ssa_comm_attach_peers first"); return SSA_ERR_STATE; }
  Session* s = st->get(id);
  if (!s) { set_error("unknown session %d", id); return SSA_ERR_UNKNOWN_SESSION; }
  if (n_q <= 0 || !Q || !K || !V || layer < -1 || layer >= st->cfg.num_layers) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  cudaStream_t cs = (cudaStream_t)stream;
  const int64_t Lin = layer < 0 ? st->cfg.num_layers : 1;
  const int64_t rows = Lin * n_q;
  const int64_t chunk = rows * st->cfg.num_q_heads * (int64_t)(st->cfg.head_dim + 1);
  if ((size_t)(2 * c->world * chunk) * sizeof(float) > c->peer_bytes) {
    set_error("sharded_push: peer buffers hold %zu bytes, need %lld (two halves)", c->peer_bytes,
              (long long)(2 * c->world * chunk * (int64_t)sizeof(float)));
    return SSA_ERR_INVALID_ARG;
  }
  if (c->epoch != c->merged) {
    set_error("sharded_push: merge the previous epoch first");
    return SSA_ERR_STATE;
  }
  if (c->chunk_for != chunk) {   // this rank's chunk slot in both halves of every peer's gathered buffer
    if (c->chunk_for >= 0 && c->epoch > 0) {
      set_error("sharded_push: the chunk size is fixed after the first push (re-attach to change it)");
      return SSA_ERR_STATE;
    }
    std::vector<uint64_t> slot(2 * c->world);
    for (int h = 0; h < 2; ++h)
      for (int q = 0; q < c->world; ++q)
        slot[h * c->world + q] = c->peer_buf[q] + ((uint64_t)h * c->world + c->rank) * chunk * sizeof(float);
    COMM_CUDA(st, cudaMemcpyAsync(c->d_peer_chunk, slot.data(), 2 * c->world * sizeof(uint64_t),
                                  cudaMemcpyHostToDevice, cs));
    COMM_CUDA(st, cudaStreamSynchronize(cs));
    c->chunk_for = chunk;
  }
  const uint32_t e = c->epoch + 1;
  // half e & 1 of every peer buffer was last read by the peers' merges of epoch e - 2:
  // wait for their acks (slots [world, 2 world) of this rank's own flag array)
  if (e >= 3)
    COMM_CUDA(st, launch_wait_flags(reinterpret_cast<const uint32_t*>(c->peer_flag[c->rank]) + c->world, c->world,
                                    e - 2, cs));
  const size_t el = st->elem;
  IoSet io;
  io.q = {Q, (size_t)rows * st->cfg.num_q_heads * st->cfg.head_dim * el};
  io.k = {K, (size_t)rows * st->cfg.num_kv_heads * st->cfg.head_dim * el};
  io.v = {V, (size_t)rows * st->cfg.num_kv_heads * st->cfg.head_dim * el};
  if ((rc = st->stage_inputs(&io, cs)) != SSA_OK) return rc;
  SegDesc sg{};
  sg.row0 = 0;
  sg.m = n_q;
  sg.tail_m = c->rank == c->world - 1 ? n_q : 0;   // the tail owner (R-12)
  st->fill_cached(*s, &sg);
  sg.append_slot0 = -1;
  std::vector<SegDesc> segs{sg};
  RunOpts opts;
  opts.force_groups = true;
  opts.peer_chunk = c->d_peer_chunk + (e & 1) * c->world;
  opts.n_peers = c->world;
  opts.lse_off = rows * st->cfg.num_q_heads * (int64_t)st->cfg.head_dim;
  if ((rc = st->run(segs, io, n_q, layer < 0 ? 0 : layer, (int32_t)Lin, 1, true, true, cs, opts)) != SSA_OK) return rc;
  c->epoch = e;
  COMM_CUDA(st, launch_signal_peers(c->d_peer_flag, c->world, c->rank, e, cs));   // ready[rank] on every peer
  st->stats.kernel_launches += e >= 3 ? 2 : 1;
  return SSA_OK;
}

ssa_status ssa_sharded_merge(ssa_store_t st, int32_t layer, int32_t n_q, void* O, void* stream) {
  ssa_status rc = check_store(st);
  if (rc != SSA_OK) return rc;
  CommState* c = st->comm;
  if (!c || !c->peers) { set_error("sharded_merge: ssa_comm_attach_peers first"); return SSA_ERR_STATE; }
  if (n_q <= 0 || !O || layer < -1 || layer >= st->cfg.num_layers) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  cudaStream_t cs = (cudaStream_t)stream;
  const int64_t rows = (layer < 0 ? st->cfg.num_layers : 1) * (int64_t)n_q;
  IoSet io;
  io.o = {O, (size_t)rows * st->cfg.num_q_heads * st->cfg.head_dim * st->elem};
  if ((rc = st->stage_inputs(&io, cs)) != SSA_OK) return rc;
  if (c->epoch == c->merged) {
    set_error("sharded_merge: no pushed epoch to merge");
    return SSA_ERR_STATE;
  }
  const uint32_t e = c->epoch;
  const int64_t chunk = rows * st->cfg.num_q_heads * (int64_t)(st->cfg.head_dim + 1);
  if (chunk != c->chunk_for) return SSA_ERR_INVALID_ARG;
  const float* gathered = reinterpret_cast<const float*>(c->peer_buf[c->rank]) + (e & 1) * c->world * chunk;
  // every rank's chunk of epoch e has landed (ready slots [0, world) of this rank's flags)
  COMM_CUDA(st, launch_wait_flags(reinterpret_cast<const uint32_t*>(c->peer_flag[c->rank]), c->world, e, cs));
  COMM_CUDA(st, launch_merge_ranks(gathered, c->world, rows, st->cfg.num_q_heads, st->cfg.head_dim, io.o.dev,
                                   st->cfg.dtype == SSA_BF16, cs));
  // this rank is done reading half e & 1: ack[rank] = e on every peer (they may reuse it for e + 2)
  COMM_CUDA(st, launch_signal_peers(c->d_peer_flag, c->world, c->world + c->rank, e, cs));
  c->merged = e;
  st->stats.kernel_launches += 3;
  return st->unstage_output(&io, cs);
}

ssa_status ssa_sharded_query(ssa_store_t st, ssa_session_t id, int32_t layer, int32_t n_q, const void* Q,
                             const void* K, const void* V, void* O, void* stream) {
  ssa_status rc = check_store(st);
  if (rc != SSA_OK) return rc;
  if (!st->comm) { set_error("sharded_query: ssa_comm_init or ssa_comm_attach_peers first"); return SSA_ERR_STATE; }
  if (st->comm->peers) {
    if ((rc = ssa_sharded_push(st, id, layer, n_q, Q, K, V, stream)) != SSA_OK) return rc;
    return ssa_sharded_merge(st, layer, n_q, O, stream);
  }
  if (n_q <= 0 || !O || layer < -1 || layer >= st->cfg.num_layers) return SSA_ERR_INVALID_ARG;
  cudaSetDevice(st->cfg.device);
  SSA_ORDERED(st, stream);
  CommState* c = st->comm;
  cudaStream_t cs = (cudaStream_t)stream;
  const int64_t Lin = layer < 0 ? st->cfg.num_layers : 1;
  const int64_t rows = Lin * n_q;
  const size_t chunk = (size_t)rows * st->cfg.num_q_heads * (st->cfg.head_dim + 1);
  const size_t need = chunk * (1 + c->world);
  if (need > c->cap) {   // stream-ordered growth
    if (c->buf) COMM_CUDA(st, cudaFreeAsync(c->buf, cs));
    c->buf = nullptr;
    c->cap = std::max(need, c->cap * 2);
    COMM_CUDA(st, cudaMallocAsync(reinterpret_cast<void**>(&c->buf), c->cap * sizeof(float), cs));
  }
  rc = ssa_sharded_partial(st, id, layer, n_q, Q, K, V, c->rank == c->world - 1, c->buf, stream);
  if (rc != SSA_OK) return rc;
  ncclResult_t r = nccl().all_gather(c->buf, c->buf + chunk, chunk, ncclFloat32, c->comm, cs);
  if (r != ncclSuccess) return nccl_fail(st, r, "ncclAllGather");
  return ssa_merge_rank_partials(st, c->world, rows, c->buf + chunk, O, stream);
}

}  // extern "C"
