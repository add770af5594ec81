"""Python binding of libssa — B200-native stateful-session attention.

Thin marshalling over the C ABI in ``include/ssa.h`` (same names, minus the
``ssa_`` prefix): every step of the hot path runs in the library's sm_100a
kernels.  Arguments may be torch tensors (CUDA or CPU), numpy arrays or raw
integer pointers.  There is no fallback: if ``libssa.so`` is missing or fails to
load, importing this package raises.

Shapes follow the ABI: Q/O ``[L'][n][Hq][d]``, K/V ``[L'][n][Hkv][d]`` with
L' = num_layers for all-layer calls (``layer=-1``) and 1 for single-layer calls.
"""
from __future__ import annotations

import ctypes
import os

__all__ = ["Store", "SsaError", "lib", "LIB_PATH", "WORK_APPEND", "WORK_QUERY", "WORK_STATELESS",
           "OPT_ATTN_BACKEND", "OPT_MAX_SPLITS", "OPT_FAULT_INJECT", "OPT_TC_Q_TILES", "OPT_TIMING",
           "OPT_GRAPH_ARENA_RESET", "OPT_CLUSTER", "OPT_PDL", "OPT_PIPE_CHUNKS", "OPT_QKV_DEBUG", "OPT_CM_MERGE", "OPT_L2_HINT",
           "debug_plan", "TIMING_KINDS"]
TIMING_KINDS = ("attn_data", "attn_query", "combine_data", "combine_query", "scatter", "qkv_rope", "quant_e4m3")

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libssa.so")

WORK_APPEND, WORK_QUERY, WORK_STATELESS = 0, 1, 2
OPT_ATTN_BACKEND, OPT_MAX_SPLITS, OPT_FAULT_INJECT, OPT_TC_Q_TILES, OPT_TIMING = 1, 2, 3, 4, 5
OPT_GRAPH_ARENA_RESET, OPT_CLUSTER, OPT_PDL, OPT_PIPE_CHUNKS, OPT_QKV_DEBUG, OPT_CM_MERGE = 8, 9, 10, 11, 12, 13
OPT_L2_HINT = 14
BF16, FP32 = 0, 1

_STATUS = {0: "SSA_OK", -1: "SSA_ERR_INVALID_ARG", -2: "SSA_ERR_UNKNOWN_SESSION", -3: "SSA_ERR_POOL_EXHAUSTED",
           -4: "SSA_ERR_SESSION_LIMIT", -5: "SSA_ERR_CUDA", -6: "SSA_ERR_NCCL", -7: "SSA_ERR_UNSUPPORTED",
           -8: "SSA_ERR_STATE"}


class SsaError(RuntimeError):
    def __init__(self, code: int, where: str, msg: str):
        super().__init__(f"{where}: {_STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = _STATUS.get(code, str(code))


class StoreConfig(ctypes.Structure):
    _fields_ = [("num_layers", ctypes.c_int32), ("num_q_heads", ctypes.c_int32),
                ("num_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32),
                ("page_size", ctypes.c_int32), ("num_pages", ctypes.c_int64),
                ("max_sessions", ctypes.c_int32), ("device", ctypes.c_int32),
                ("dtype", ctypes.c_int32), ("softmax_scale", ctypes.c_float),
                ("kv_format", ctypes.c_int32), ("k_scale", ctypes.c_float), ("v_scale", ctypes.c_float),
                ("pool_ptr", ctypes.c_void_p), ("pool_bytes", ctypes.c_size_t)]


KV_SAME, KV_E4M3 = 0, 1


class SessionInfo(ctypes.Structure):
    _fields_ = [("n_tokens", ctypes.c_int64), ("n_prefix", ctypes.c_int64),
                ("n_pages", ctypes.c_int64), ("version", ctypes.c_uint64),
                ("n_evicted", ctypes.c_int64), ("retention", ctypes.c_int64)]


class WorkItem(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("session", ctypes.c_int32), ("n_tokens", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("row_offset", ctypes.c_int64)]


class Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("kernel_launches", "rows_computed", "query_rows",
                                              "tokens_appended", "pages_reserved", "h2d_bytes", "d2h_bytes",
                                              "tc_launches", "cm_launches", "plan_uploads")]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libssa.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    P = ctypes.POINTER
    sig = {
        "ssa_store_pool_bytes": (ctypes.c_size_t, [P(StoreConfig)]),
        "ssa_store_create": (i32, [P(StoreConfig), P(vp)]),
        "ssa_store_destroy": (i32, [vp]),
        "ssa_store_occupancy": (i32, [vp, P(i64), P(i64)]),
        "ssa_session_create": (i32, [vp, i32, vp, vp, vp, vp, vp, P(i32)]),
        "ssa_session_append": (i32, [vp, i32, i32, vp, vp, vp, vp, vp, P(u64)]),
        "ssa_append_begin": (i32, [vp, i32, i32, P(i32)]),
        "ssa_append_layer": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp]),
        "ssa_append_commit": (i32, [vp, i32, i32, P(u64)]),
        "ssa_append_abort": (i32, [vp, i32, i32]),
        "ssa_session_truncate": (i32, [vp, i32, i64, P(u64)]),
        "ssa_session_destroy": (i32, [vp, i32]),
        "ssa_session_evict_oldest": (i32, [vp, i32, i64, vp, P(u64)]),
        "ssa_session_set_retention": (i32, [vp, i32, i64]),
        "ssa_session_alias_prefix": (i32, [vp, i32, i64, vp, P(i32)]),
        "ssa_debug_trace": (i32, [vp, ctypes.c_size_t]),
        "ssa_greedy_sample": (i32, [vp, i32, i32, i32, i64, vp, vp, vp, vp, vp, vp, vp]),
        "ssa_session_query": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp]),
        "ssa_flash_query_batch": (i32, [vp, i32, i32, i32, P(i32), vp, vp, vp, vp, vp]),
        "ssa_batch_run": (i32, [vp, i32, i32, P(WorkItem), vp, vp, vp, vp, vp]),
        "ssa_session_get_info": (i32, [vp, i32, P(SessionInfo)]),
        "ssa_session_page_table": (i32, [vp, i32, P(i32), i64, P(i64)]),
        "ssa_session_read_kv": (i32, [vp, i32, i32, i64, i64, vp, vp]),
        "ssa_session_load_kv": (i32, [vp, i32, i64, vp, vp, vp]),
        "ssa_session_digest": (i32, [vp, i32, P(u64)]),
        "ssa_store_stats": (i32, [vp, P(Stats), i32]),
        "ssa_store_set_option": (i32, [vp, i32, i64]),
        "ssa_store_timing": (i32, [vp, P(ctypes.c_double), P(i64), i32]),
        "ssa_comm_unique_id": (i32, [P(ctypes.c_uint8)]),
        "ssa_comm_init": (i32, [vp, i32, i32, P(ctypes.c_uint8)]),
        "ssa_sharded_query": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp]),
        "ssa_comm_destroy": (i32, [vp]),
        "ssa_comm_attach_peers": (i32, [vp, i32, i32, P(u64), P(u64), ctypes.c_size_t]),
        "ssa_sharded_push": (i32, [vp, i32, i32, i32, vp, vp, vp, vp]),
        "ssa_sharded_merge": (i32, [vp, i32, i32, vp, vp]),
        "ssa_sharded_partial": (i32, [vp, i32, i32, i32, vp, vp, vp, i32, vp, vp]),
        "ssa_merge_rank_partials": (i32, [vp, i32, i64, vp, vp, vp]),
        "ssa_qkv_rope": (i32, [vp, i32, i32, i64, ctypes.c_float, vp, vp, vp, vp, vp, vp]),
        "ssa_append_layer_fused": (i32, [vp, i32, i32, i32, i32, ctypes.c_float, vp, vp, vp, vp]),
        "ssa_session_query_fused": (i32, [vp, i32, i32, i32, i32, ctypes.c_float, vp, vp, vp, vp]),
        "ssa_status_str": (ctypes.c_char_p, [i32]),
        "ssa_last_error": (ctypes.c_char_p, []),
        "ssa_abi_version": (i32, []),
        "ssa_debug_last_plan": (i32, [vp, P(i64)]),
        "ssa_debug_tc_clusters": (i32, [i32, i32]),
        "ssa_debug_plan": (i32, [i32, P(i32), P(i32), i32, i32, i32, i32, i32, i32, i32, P(i32), i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


def _check(rc: int, where: str):
    if rc != 0:
        raise SsaError(rc, where, (lib.ssa_last_error() or b"").decode())


def _ptr(x):
    """Raw address of a torch tensor / numpy array / int / None (no copies)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    raise TypeError(f"unsupported buffer type {type(x)}")


def _stream(stream):
    if stream is None:
        try:
            import torch
            if torch.cuda.is_available() and torch.cuda.is_initialized():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _ntok(x, axis=1):
    return int(x.shape[axis])


class Store:
    """A KV pool on one GPU plus its sessions (see include/ssa.h)."""

    def __init__(self, num_layers, num_q_heads, num_kv_heads, head_dim, page_size=64, num_pages=1024,
                 max_sessions=64, device=0, dtype="bf16", softmax_scale=0.0, kv_format=None,
                 k_scale=1.0, v_scale=1.0, pool=None):
        """kv_format None: K/V stored in `dtype`; "e4m3": E4M3 codes of K/k_scale, V/v_scale
        (include/ssa.h, reading R-22).  pool: optional caller-owned device buffer for the KV
        pool (a contiguous torch tensor of >= pool_bytes(...) bytes on `device`); the store
        keeps a reference to it."""
        self._pool = pool
        pool_ptr, pool_nbytes = (None, 0)
        if pool is not None:
            pool_ptr = _ptr(pool)
            pool_nbytes = pool.numel() * pool.element_size() if hasattr(pool, "numel") else int(pool.nbytes)
        self.cfg = StoreConfig(num_layers, num_q_heads, num_kv_heads, head_dim, page_size, num_pages,
                               max_sessions, device, BF16 if dtype == "bf16" else FP32, softmax_scale,
                               KV_E4M3 if kv_format == "e4m3" else KV_SAME, k_scale, v_scale,
                               pool_ptr, pool_nbytes)
        self.dtype = dtype
        self.kv_format = kv_format
        self.L, self.hq, self.hkv, self.d, self.P = num_layers, num_q_heads, num_kv_heads, head_dim, page_size
        self.device = device
        h = ctypes.c_void_p()
        _check(lib.ssa_store_create(ctypes.byref(self.cfg), ctypes.byref(h)), "store_create")
        self._h = h

    @staticmethod
    def pool_bytes(num_layers, num_q_heads, num_kv_heads, head_dim, page_size, num_pages, dtype="bf16",
                   kv_format=None, k_scale=1.0, v_scale=1.0):
        c = StoreConfig(num_layers, num_q_heads, num_kv_heads, head_dim, page_size, num_pages, 1, 0,
                        BF16 if dtype == "bf16" else FP32, 0.0, KV_E4M3 if kv_format == "e4m3" else KV_SAME,
                        k_scale, v_scale)
        return int(lib.ssa_store_pool_bytes(ctypes.byref(c)))

    def close(self):
        if getattr(self, "_h", None):
            lib.ssa_store_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- data plane ---------------------------------------------------------
    def session_create(self, Q, K, V, O=None, stream=None, n_prefix=None):
        n = n_prefix if n_prefix is not None else _ntok(K)
        sid = ctypes.c_int32()
        _check(lib.ssa_session_create(self._h, n, _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _stream(stream),
                                      ctypes.byref(sid)), "session_create")
        return sid.value

    def session_append(self, sid, Q, K, V, O=None, stream=None, n_new=None):
        n = n_new if n_new is not None else _ntok(K)
        ver = ctypes.c_uint64()
        _check(lib.ssa_session_append(self._h, sid, n, _ptr(Q), _ptr(K), _ptr(V), _ptr(O), _stream(stream),
                                      ctypes.byref(ver)), "session_append")
        return ver.value

    def append_begin(self, sid, n_new):
        t = ctypes.c_int32()
        _check(lib.ssa_append_begin(self._h, sid, n_new, ctypes.byref(t)), "append_begin")
        return t.value

    def append_layer(self, sid, ticket, layer, Q, K, V, O=None, stream=None):
        _check(lib.ssa_append_layer(self._h, sid, ticket, layer, _ptr(Q), _ptr(K), _ptr(V), _ptr(O),
                                    _stream(stream)), "append_layer")

    # -- fused projection (Alg. 1 L282 `Forward`) ---------
    def qkv_rope(self, X, W, Q, K, V, pos0=0, rope_theta=500000.0, stream=None):
        """[Q|K|V] = X W^T with RoPE on Q and K at positions pos0.. (device tensors;
        X [n][hidden], W [(Hq+2Hkv)*d][hidden], Q [n][Hq][d], K/V [n][Hkv][d], bf16)."""
        _check(lib.ssa_qkv_rope(self._h, X.shape[0], X.shape[1], pos0, rope_theta, _ptr(X), _ptr(W), _ptr(Q),
                                _ptr(K), _ptr(V), _stream(stream)), "qkv_rope")

    def append_layer_fused(self, sid, ticket, layer, X, W, O, rope_theta=500000.0, stream=None):
        """Per-layer append whose Q/K/V come from the fused projection of X; K/V go
        straight into the ticket's pages."""
        _check(lib.ssa_append_layer_fused(self._h, sid, ticket, layer, X.shape[1], rope_theta, _ptr(X), _ptr(W),
                                          _ptr(O), _stream(stream)), "append_layer_fused")

    def session_query_fused(self, sid, layer, X, W, O, rope_theta=500000.0, stream=None):
        _check(lib.ssa_session_query_fused(self._h, sid, layer, X.shape[0], X.shape[1], rope_theta, _ptr(X), _ptr(W),
                                           _ptr(O), _stream(stream)), "session_query_fused")

    def append_commit(self, sid, ticket):
        ver = ctypes.c_uint64()
        _check(lib.ssa_append_commit(self._h, sid, ticket, ctypes.byref(ver)), "append_commit")
        return ver.value

    def append_abort(self, sid, ticket):
        _check(lib.ssa_append_abort(self._h, sid, ticket), "append_abort")

    def session_truncate(self, sid, p):
        ver = ctypes.c_uint64()
        _check(lib.ssa_session_truncate(self._h, sid, p, ctypes.byref(ver)), "session_truncate")
        return ver.value

    def evict_oldest(self, sid, n_tokens, stream=None):
        """Region-1 FIFO eviction (Alg. 1); returns the new version."""
        ver = ctypes.c_uint64()
        _check(lib.ssa_session_evict_oldest(self._h, sid, n_tokens, _stream(stream), ctypes.byref(ver)),
               "session_evict_oldest")
        return ver.value

    def set_retention(self, sid, max_tokens):
        _check(lib.ssa_session_set_retention(self._h, sid, max_tokens), "session_set_retention")

    def alias_prefix(self, donor, len_tokens, stream=None):
        """Metadata-only prefix aliasing; returns the new session id."""
        out = ctypes.c_int32()
        _check(lib.ssa_session_alias_prefix(self._h, donor, len_tokens, _stream(stream), ctypes.byref(out)),
               "session_alias_prefix")
        return out.value

    def greedy_sample(self, logits, out_ids, out_gap=None, out_top2=None, draft=None, out_n_accept=None,
                      stream=None):
        """On-device greedy sampling: per row argmax (lowest id on ties) and logit
        gap l1 - l2 (Eq. logit-gap); optional draft-window acceptance.  `logits` is a
        2-D torch tensor (fp32 or bf16, rows contiguous); outputs are device tensors."""
        import torch
        if logits.dim() != 2 or logits.stride(1) != 1:
            raise ValueError("logits must be [rows][vocab] with unit column stride")
        dt = {torch.float32: FP32, torch.bfloat16: BF16}[logits.dtype]
        _check(lib.ssa_greedy_sample(self._h, dt, logits.shape[0], logits.shape[1], logits.stride(0), logits.data_ptr(),
                                     _ptr(out_ids), _ptr(out_gap), _ptr(out_top2), _ptr(draft), _ptr(out_n_accept),
                                     _stream(stream)), "greedy_sample")

    def session_destroy(self, sid):
        _check(lib.ssa_session_destroy(self._h, sid), "session_destroy")

    # -- query plane ----------------------------------------------------------
    def session_query(self, sid, Q, K, V, O, layer=-1, stream=None, n_q=None):
        n = n_q if n_q is not None else _ntok(K)
        _check(lib.ssa_session_query(self._h, sid, layer, n, _ptr(Q), _ptr(K), _ptr(V), _ptr(O),
                                     _stream(stream)), "session_query")

    def flash_query_batch(self, sid, q_lens, Q, K, V, O, layer=-1, stream=None):
        arr = (ctypes.c_int32 * len(q_lens))(*q_lens)
        _check(lib.ssa_flash_query_batch(self._h, sid, layer, len(q_lens), arr, _ptr(Q), _ptr(K), _ptr(V),
                                         _ptr(O), _stream(stream)), "flash_query_batch")

    def batch_run(self, items, Q, K, V, O, layer=-1, stream=None):
        """items: list of (kind, session, n_tokens, row_offset)."""
        arr = (WorkItem * len(items))(*[WorkItem(k, s, n, 0, r) for (k, s, n, r) in items])
        _check(lib.ssa_batch_run(self._h, layer, len(items), arr, _ptr(Q), _ptr(K), _ptr(V), _ptr(O),
                                 _stream(stream)), "batch_run")

    # -- introspection --------------------------------------------------------
    def info(self, sid):
        i = SessionInfo()
        _check(lib.ssa_session_get_info(self._h, sid, ctypes.byref(i)), "session_get_info")
        return dict(n_tokens=i.n_tokens, n_prefix=i.n_prefix, n_pages=i.n_pages, version=i.version,
                    n_evicted=i.n_evicted, retention=i.retention)

    def page_table(self, sid):
        n = ctypes.c_int64()
        _check(lib.ssa_session_page_table(self._h, sid, None, 0, ctypes.byref(n)), "session_page_table")
        buf = (ctypes.c_int32 * max(1, n.value))()
        _check(lib.ssa_session_page_table(self._h, sid, buf, n.value, ctypes.byref(n)), "session_page_table")
        return list(buf[:n.value])

    def read_kv(self, sid, layer, start, count):
        import numpy as np
        dt = np.uint8 if self.kv_format == "e4m3" else np.uint16 if self.dtype == "bf16" else np.float32
        K = np.zeros((count, self.hkv, self.d), dtype=dt)
        V = np.zeros_like(K)
        _check(lib.ssa_session_read_kv(self._h, sid, layer, start, count, _ptr(K), _ptr(V)), "session_read_kv")
        return K, V

    def load_kv(self, sid, K, V, stream=None):
        _check(lib.ssa_session_load_kv(self._h, sid, _ntok(K), _ptr(K), _ptr(V), _stream(stream)),
               "session_load_kv")

    def digest(self, sid):
        h = ctypes.c_uint64()
        _check(lib.ssa_session_digest(self._h, sid, ctypes.byref(h)), "session_digest")
        return h.value

    def occupancy(self):
        u, t = ctypes.c_int64(), ctypes.c_int64()
        _check(lib.ssa_store_occupancy(self._h, ctypes.byref(u), ctypes.byref(t)), "store_occupancy")
        return u.value, t.value

    def stats(self, reset=False):
        s = Stats()
        _check(lib.ssa_store_stats(self._h, ctypes.byref(s), int(reset)), "store_stats")
        return {n: getattr(s, n) for n, _ in Stats._fields_}

    def set_option(self, option, value):
        _check(lib.ssa_store_set_option(self._h, option, value), "store_set_option")

    def last_plan(self):
        """Shape of the last attention launch: units, groups, CTAs per layer, cluster size of a
        cluster-merge launch (0: combine kernel / SIMT), largest split count, group-barrier merge."""
        out = (ctypes.c_int64 * 6)()
        _check(lib.ssa_debug_last_plan(self._h, out), "debug_last_plan")
        return dict(zip(("units", "groups", "ctas", "cm_C", "max_split", "gbar"), list(out)))

    def timing(self, reset=False):
        """{kind: (ms_total, launches)} recorded under OPT_TIMING (syncs)."""
        ms = (ctypes.c_double * len(TIMING_KINDS))()
        n = (ctypes.c_int64 * len(TIMING_KINDS))()
        _check(lib.ssa_store_timing(self._h, ms, n, int(reset)), "store_timing")
        return {k: (ms[i], n[i]) for i, k in enumerate(TIMING_KINDS)}

    # -- multi-GPU split-KV ---------------------------------------------------
    @staticmethod
    def comm_unique_id() -> bytes:
        buf = (ctypes.c_uint8 * 128)()
        _check(lib.ssa_comm_unique_id(buf), "comm_unique_id")
        return bytes(buf)

    def comm_init(self, rank, world, uid: bytes):
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
        _check(lib.ssa_comm_init(self._h, rank, world, buf), "comm_init")

    def sharded_partial(self, sid, Q, K, V, part, include_tail, layer=-1, stream=None, n_q=None):
        """Rank partial over this store's shard -> packed fp32 chunk [O | lse] (device `part`)."""
        n = n_q if n_q is not None else _ntok(K)
        _check(lib.ssa_sharded_partial(self._h, sid, layer, n, _ptr(Q), _ptr(K), _ptr(V), int(include_tail),
                                       _ptr(part), _stream(stream)), "sharded_partial")

    def merge_rank_partials(self, world, rows, parts, O, stream=None):
        _check(lib.ssa_merge_rank_partials(self._h, world, rows, _ptr(parts), _ptr(O), _stream(stream)),
               "merge_rank_partials")

    def comm_attach_peers(self, rank, world, peer_bufs, peer_flags, buf_bytes):
        """A9 over peer memory (no NCCL): peer_bufs / peer_flags are `world` device addresses."""
        pb = (ctypes.c_uint64 * world)(*[int(x) for x in peer_bufs])
        pf = (ctypes.c_uint64 * world)(*[int(x) for x in peer_flags])
        _check(lib.ssa_comm_attach_peers(self._h, rank, world, pb, pf, buf_bytes), "comm_attach_peers")

    def sharded_push(self, sid, Q, K, V, layer=-1, stream=None, n_q=None):
        n = n_q if n_q is not None else _ntok(Q)
        _check(lib.ssa_sharded_push(self._h, sid, layer, n, _ptr(Q), _ptr(K), _ptr(V), _stream(stream)),
               "sharded_push")

    def sharded_merge(self, O, layer=-1, stream=None, n_q=None):
        n = n_q if n_q is not None else _ntok(O)
        _check(lib.ssa_sharded_merge(self._h, layer, n, _ptr(O), _stream(stream)), "sharded_merge")

    def comm_destroy(self):
        _check(lib.ssa_comm_destroy(self._h), "comm_destroy")

    def sharded_query(self, sid, Q, K, V, O, layer=-1, stream=None, n_q=None):
        n = n_q if n_q is not None else _ntok(K)
        _check(lib.ssa_sharded_query(self._h, sid, layer, n, _ptr(Q), _ptr(K), _ptr(V), _ptr(O),
                                     _stream(stream)), "sharded_query")


def debug_plan(seg_m, seg_slots, Hkv, q_tile_tokens, key_tile, n_layers=1, num_sms=148, ctas_per_sm=1,
               max_splits=0):
    """Planner introspection (host only): list of units (seg, kvh, tok0, ntok, tile_lo, tile_hi, group, split)."""
    n = len(seg_m)
    m = (ctypes.c_int32 * n)(*seg_m)
    s = (ctypes.c_int32 * n)(*seg_slots)
    cnt = lib.ssa_debug_plan(n, m, s, Hkv, q_tile_tokens, key_tile, n_layers, num_sms, ctas_per_sm, max_splits,
                             None, 0)
    buf = (ctypes.c_int32 * (8 * max(1, cnt)))()
    lib.ssa_debug_plan(n, m, s, Hkv, q_tile_tokens, key_tile, n_layers, num_sms, ctas_per_sm, max_splits, buf, cnt)
    return [tuple(buf[8 * i:8 * i + 8]) for i in range(cnt)]
