"""fp64 CPU oracle for the stateful-session attention hot path (arXiv 2605.13784).

TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  It shares no code with ``paper_2605_13784_b200`` (the CUDA path) and
imports nothing from it; the two meet only in ``streams.py`` (seeded inputs).

What it computes:

* ``attention_rows`` — Eq. (attention) softmax(QK^T/sqrt(d_k))V, PAPER.md
  P:143-148, for explicit rows and visible-key counts (C, ``ssa_oracle.c``).
* ``segment_rows`` — Eq. (query-attention): the rows of a new
  segment X (an append D_k, Alg. 1 L282 P:282; a query q, Alg. 2 L295 P:295;
  a Flash Query f_i, Alg. 3 L542 P:542) attend to the cached keys
  [S; D_1..D_{k-1}] followed by X[0..i] (causal; reading R-2), with the
  GQA head map of reading R-5.
* ``full_recompute`` — the naive approach of P:42: causal attention over the
  whole concatenation [S; D_1..D_k; Q_j] from scratch, no session state.
* ``merge_partials`` — split-KV log-sum-exp merge (reading R-11).
* ``qkv_projection`` / ``rope`` / ``qkv_rope`` / ``round_bf16`` — the fused
  data-plane projection before attention (reading R-21).
* ``e4m3_decode`` / ``e4m3_encode`` — the FP8 (E4M3) KV-cache variant (SURVEY
  §8(f) rank 4, reading R-22): codes per the OCP FP8 E4M3 definition, values
  x / scale rounded once in fp32, then to the nearest E4M3 value (ties to even),
  saturating at +-448.
* ``OracleStore`` — the session model: retained tokens, versions ("data
  version t"), the page allocator replica (lowest free id first, R0 padded to a
  page boundary; reading R-9) and the FNV-1a-64 digest.

Pins: ``tests/test_oracle_pins.py`` (mpmath brute force, closed forms,
invariants, golden fixtures under ``tests/golden/``).
"""
from __future__ import annotations

import ctypes
import copy
import heapq
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build() -> str:
    """Compile ssa_oracle.c with gcc (plain -O2, no fast-math)."""
    import subprocess
    src = os.path.join(_HERE, "ssa_oracle.c")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-std=c11", "-o", _LIB_PATH, src, "-lm"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        L.oracle_attention_rows.argtypes = [i64, i64, i64, dp, i64, i64, dp, i64, dp, i64,
                                            ctypes.POINTER(i64), ctypes.c_double, dp, dp]
        L.oracle_attention_rows.restype = ctypes.c_int
        L.oracle_merge_partials.argtypes = [i64, i64, i64, dp, dp, dp, dp]
        L.oracle_merge_partials.restype = ctypes.c_int
        L.oracle_fnv1a64.argtypes = [ctypes.c_void_p, i64, ctypes.c_uint64]
        L.oracle_fnv1a64.restype = ctypes.c_uint64
        L.oracle_fnv1a64_offset_basis.argtypes = []
        L.oracle_fnv1a64_offset_basis.restype = ctypes.c_uint64
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ----------------------------------------------------------------------------
# exact decode of stored values (reading R-10: inputs are bf16 or fp32 bits)
# ----------------------------------------------------------------------------
def to_f64(x: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (uint16) or float32 -> float64, exactly."""
    x = np.asarray(x)
    if x.dtype == np.uint16:
        return (x.astype(np.uint32) << np.uint32(16)).view(np.float32).astype(np.float64)
    if x.dtype == np.float32:
        return x.astype(np.float64)
    if x.dtype == np.float64:
        return x
    raise TypeError(f"unsupported storage dtype {x.dtype}")


# ----------------------------------------------------------------------------
# FP8 E4M3 KV storage (P:629 names FP8 KV for the TRT-LLM
# baseline; reading R-22)
# ----------------------------------------------------------------------------
E4M3_MAX = 448.0


def e4m3_decode(codes: np.ndarray) -> np.ndarray:
    """E4M3 code (uint8: sign, 4-bit exponent with bias 7, 3-bit mantissa; no
    infinities; S.1111.111 is NaN) -> float64, by the format's definition:
    exponent field 0 -> (-1)^s (m/8) 2^-6, else (-1)^s (1 + m/8) 2^(e-7)."""
    c = np.asarray(codes, dtype=np.uint8).astype(np.int64)
    s = (c >> 7) & 1
    e = (c >> 3) & 15
    m = c & 7
    mag = np.where(e == 0, (m / 8.0) * 2.0 ** -6, (1.0 + m / 8.0) * np.exp2(e - 7.0))
    val = np.where(s == 1, -mag, mag)
    return np.where((e == 15) & (m == 7), np.nan, val)


_E4M3_POS = e4m3_decode(np.arange(127, dtype=np.uint8))   # codes 0..126: the finite values >= 0


def e4m3_encode(x, scale: float) -> np.ndarray:
    """Quantize to E4M3 codes (reading R-22): y = fp32(x) / fp32(scale), one
    IEEE fp32 division (round to nearest), then y is rounded to the nearest
    finite E4M3 value with ties to the even code (even mantissa), |y| > 448
    saturating to 448 (every such y rounds to 448 or overflows); the sign of y
    is kept (a negative y that rounds to 0 gives -0, code 0x80); NaN -> 0x7F.
    x: bf16 bit patterns (uint16) or floats exactly representable in fp32."""
    xf = to_f64(x).astype(np.float32) if np.asarray(x).dtype == np.uint16 else np.asarray(x, dtype=np.float32)
    y = (xf / np.float32(scale)).astype(np.float64)       # fp32 division, exact widening
    a = np.minimum(np.abs(y), E4M3_MAX)
    a = np.where(np.isnan(y), 0.0, a)
    # spacing of the E4M3 grid around a: 2^-9 below 2^-6 (subnormals), else 2^(floor(log2 a) - 3)
    _, ex = np.frexp(np.maximum(a, 2.0 ** -6))            # a = f 2^ex, 0.5 <= f < 1
    ulp = np.exp2(ex - 4.0)
    q = np.round(a / ulp) * ulp                            # numpy rounds halves to even
    code = np.searchsorted(_E4M3_POS, q).astype(np.uint8)  # q is on the grid: exact match
    code = np.where(np.signbit(y), code | np.uint8(0x80), code).astype(np.uint8)
    return np.where(np.isnan(y), np.uint8(0x7F), code).astype(np.uint8)


# ----------------------------------------------------------------------------
# definitions
# ----------------------------------------------------------------------------
def attention_rows(q: np.ndarray, k: np.ndarray, v: np.ndarray, nvis, scale: float):
    """Eq. (attention) P:145 for rows q[r] over keys k[0:nvis[r]], v[0:nvis[r]].

    q: [nr][d], k: [nk][d], v: [nk][dv] (float64).  Returns (o [nr][dv], lse [nr]).
    """
    q = np.ascontiguousarray(q, dtype=np.float64)
    k = np.ascontiguousarray(k, dtype=np.float64)
    v = np.ascontiguousarray(v, dtype=np.float64)
    nr, d = q.shape
    nk = k.shape[0]
    dv = v.shape[1]
    nvis = np.ascontiguousarray(np.broadcast_to(np.asarray(nvis, dtype=np.int64), (nr,)))
    o = np.zeros((nr, dv), dtype=np.float64)
    lse = np.zeros((nr,), dtype=np.float64)
    if nr == 0:
        return o, lse
    kk = k if nk else np.zeros((1, d))
    vv = v if nk else np.zeros((1, dv))
    rc = lib().oracle_attention_rows(nr, d, dv, _dp(q), d, nk, _dp(kk), d, _dp(vv), dv,
                                     nvis.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                     float(scale), _dp(o), _dp(lse))
    if rc != 0:
        raise ValueError("oracle_attention_rows: bad arguments")
    return o, lse


def merge_partials(o_parts: np.ndarray, lse_parts: np.ndarray):
    """Split-KV merge (reading R-11).  o_parts [G][nr][dv], lse_parts [G][nr]."""
    o_parts = np.ascontiguousarray(o_parts, dtype=np.float64)
    lse_parts = np.ascontiguousarray(lse_parts, dtype=np.float64)
    G, nr, dv = o_parts.shape
    o = np.zeros((nr, dv))
    lse = np.zeros((nr,))
    rc = lib().oracle_merge_partials(G, nr, dv, _dp(o_parts), _dp(lse_parts), _dp(o), _dp(lse))
    if rc != 0:
        raise ValueError("oracle_merge_partials: bad arguments")
    return o, lse


def fnv1a64(data: bytes, h: int | None = None) -> int:
    L = lib()
    if h is None:
        h = L.oracle_fnv1a64_offset_basis()
    buf = (ctypes.c_uint8 * len(data)).from_buffer_copy(data) if data else None
    return int(L.oracle_fnv1a64(buf, len(data), ctypes.c_uint64(h)))


def derive_seed(tokens) -> int:
    """Eq. seed(P) = FNV1a(P) mod 2^32; tokens as int32 LE."""
    data = np.asarray(list(tokens), dtype="<i4").tobytes()
    return fnv1a64(data) % (1 << 32)


def default_scale(d: int) -> float:
    """1/sqrt(d_k), Eq. (attention) P:145 (reading R-1)."""
    return 1.0 / math.sqrt(d)


def segment_rows(k_cache, v_cache, q_new, k_new, v_new, num_kv_heads: int, scale: float,
                 tokens=None, heads=None):
    """Rows of a new segment X against cache ++ X (causal), Eq. query-attention P:152.

    k_cache/v_cache: [n][Hkv][d] (any storage dtype; n may be 0)
    q_new: [m][Hq][d], k_new/v_new: [m][Hkv][d]
    Row (t, h) attends to all n cached keys and new keys 0..t of kv head
    h // (Hq/Hkv) (readings R-2, R-5).  ``tokens``/``heads`` select a subset.
    Returns (o [len(tokens)][len(heads)][d], lse [len(tokens)][len(heads)]) fp64.
    """
    kc, vc = to_f64(k_cache), to_f64(v_cache)
    qn, kn, vn = to_f64(q_new), to_f64(k_new), to_f64(v_new)
    m, hq, d = qn.shape
    n = kc.shape[0]
    g = hq // num_kv_heads
    tokens = list(range(m)) if tokens is None else list(tokens)
    heads = list(range(hq)) if heads is None else list(heads)
    dv = vn.shape[2]
    o = np.zeros((len(tokens), len(heads), dv))
    lse = np.zeros((len(tokens), len(heads)))
    for hi, h in enumerate(heads):
        kvh = h // g
        keys = np.concatenate([kc[:, kvh, :].reshape(n, kn.shape[2]), kn[:, kvh, :]], axis=0)
        vals = np.concatenate([vc[:, kvh, :].reshape(n, dv), vn[:, kvh, :]], axis=0)
        qrows = qn[tokens, h, :]
        nvis = np.array([n + t + 1 for t in tokens], dtype=np.int64)
        oh, lh = attention_rows(qrows, keys, vals, nvis, scale)
        o[:, hi, :] = oh
        lse[:, hi] = lh
    return o, lse


def full_recompute(q_all, k_all, v_all, num_kv_heads: int, scale: float, rows=None):
    """Naive approach of P:42: causal attention over the whole sequence, from scratch.

    q_all: [N][Hq][d], k_all/v_all: [N][Hkv][d].  Row i sees keys 0..i.
    Returns o [len(rows)][Hq][d] fp64 (rows default: all).
    """
    q, k, v = to_f64(q_all), to_f64(k_all), to_f64(v_all)
    N, hq, d = q.shape
    g = hq // num_kv_heads
    rows = list(range(N)) if rows is None else list(rows)
    o = np.zeros((len(rows), hq, v.shape[2]))
    for h in range(hq):
        oh, _ = attention_rows(q[rows, h, :], k[:, h // g, :], v[:, h // g, :],
                               np.array([i + 1 for i in rows], dtype=np.int64), scale)
        o[:, h, :] = oh
    return o


# ----------------------------------------------------------------------------
# session model
# ----------------------------------------------------------------------------
class OracleError(Exception):
    def __init__(self, code: str):
        super().__init__(code)
        self.code = code


@dataclass
class _Session:
    n_prefix: int
    k: list = field(default_factory=list)     # per layer: np array [n][Hkv][d]
    v: list = field(default_factory=list)
    n_tokens: int = 0
    version: int = 0
    pages: list = field(default_factory=list)
    pos: list = field(default_factory=list)   # original position of each retained token (never re-based)
    r1_skip: int = 0        # evicted Region-1 slots at the head of the first retained R1 page
    n_evicted: int = 0
    retention: int = 0      # Region-1 retention window, 0 = unlimited


class OracleStore:
    """Session model of DESIGN.md §3.

    * create(S)   — Region 0 processed once; version 1.
    * append(D_k) — "only the delta is processed and appended", Alg. 1;
                    version += 1 ("incremented after each data ingestion batch").
    * query(q)    — Alg. 2; no state change (R2 cleared; reading R-3).
    * flash_query_batch(f_1..f_k) — Eq. flash-eval P:406 for each f_i against K_t, each
                    seeing only the cache and its own tokens (reading R-4); no state change.
    * truncate(p) — SeqRemove(s, p, inf), P:438 / Alg. 3 L540.
    * evict_oldest(n) — Alg. 1 L279-281 FIFO eviction of the n oldest Region-1 tokens
                    (R0 frozen; SPEC kv-store evict_oldest); positions never re-based.
    * set_retention(w) — the Alg. 1 guard: an append of m tokens that would exceed w first
                    evicts m tokens.
    * alias_prefix(donor, m) — metadata-only prefix sharing (SPEC alias_prefix):
                    whole pages shared by reference count, the page holding token m-1 copied.
    * pages       — P-token pages, lowest free id first, R0 padded to a page boundary
                    (reading R-9); the page table is compared bit-exactly with the GPU store.
    """

    def __init__(self, num_layers, num_q_heads, num_kv_heads, head_dim, page_size, num_pages,
                 dtype="bf16", softmax_scale=0.0, max_sessions=1024, kv_format=None,
                 k_scale=1.0, v_scale=1.0):
        self.L, self.hq, self.hkv, self.d = num_layers, num_q_heads, num_kv_heads, head_dim
        self.P, self.num_pages, self.dtype = page_size, num_pages, dtype
        # kv_format "e4m3": the cache holds E4M3 codes of K / k_scale and V / v_scale
        # (reading R-22); every key and value a row attends to -- cached or the
        # segment's own -- is the dequantized code (code value * scale).
        self.kv_format = kv_format
        self.k_scale, self.v_scale = float(np.float32(k_scale)), float(np.float32(v_scale))
        self.scale = softmax_scale if softmax_scale > 0 else default_scale(head_dim)
        self.max_sessions = max_sessions
        self.free = list(range(num_pages))
        heapq.heapify(self.free)
        self.ref = [0] * num_pages      # referers per page (aliases share pages)
        self.sessions: dict[int, _Session] = {}
        self.next_id = 0

    # -- page model (reading R-9) --------------------------------------------
    def slots_for(self, n_prefix: int, n_tokens: int, r1_skip: int = 0) -> int:
        """Slots occupied by n_tokens retained tokens: R0 is padded to a page boundary,
        and r1_skip evicted slots precede the first retained Region-1 token."""
        if n_tokens <= n_prefix:
            return n_tokens
        pad = -(-n_prefix // self.P) * self.P
        return pad + r1_skip + (n_tokens - n_prefix)

    def pages_for(self, n_prefix: int, n_tokens: int, r1_skip: int = 0) -> int:
        return -(-self.slots_for(n_prefix, n_tokens, r1_skip) // self.P)

    def _take_page(self) -> int:
        pg = heapq.heappop(self.free)        # lowest free id first (reading R-9)
        self.ref[pg] = 1
        return pg

    def _release(self, pages) -> None:
        for pg in pages:
            self.ref[pg] -= 1
            if self.ref[pg] == 0:            # last referer gone (SPEC: deferred free)
                heapq.heappush(self.free, pg)

    def _reserve(self, s: _Session, n_new: int) -> list:
        need = self.pages_for(s.n_prefix, s.n_tokens + n_new, s.r1_skip) - len(s.pages)
        if need > len(self.free):
            raise OracleError("POOL_EXHAUSTED")
        return [self._take_page() for _ in range(need)]

    def _snapshot(self):
        return copy.deepcopy((self.sessions, self.free, self.ref, self.next_id))

    def _restore(self, snap):
        self.sessions, self.free, self.ref, self.next_id = snap

    def occupancy(self):
        return self.num_pages - len(self.free), self.num_pages

    # -- helpers ---------------------------------------------------------------
    def _check(self, sid):
        if sid not in self.sessions:
            raise OracleError("UNKNOWN_SESSION")
        return self.sessions[sid]

    def _layers(self, layer):
        return range(self.L) if layer < 0 else [layer]

    def _store_kv(self, K, V):
        """What the cache stores for input K/V: the input bits, or E4M3 codes (R-22)."""
        if self.kv_format == "e4m3":
            return e4m3_encode(K, self.k_scale), e4m3_encode(V, self.v_scale)
        return K, V

    def _kv_values(self, K, V):
        """Stored K/V -> the fp64 values attention uses."""
        if self.kv_format == "e4m3":
            return e4m3_decode(K) * self.k_scale, e4m3_decode(V) * self.v_scale
        return to_f64(K), to_f64(V)

    def _rows(self, s: _Session, layer: int, Q, K, V, tokens=None, heads=None):
        d = self.d
        K, V = self._store_kv(K, V)
        kc = s.k[layer] if s.n_tokens else np.zeros((0, self.hkv, d), dtype=K.dtype)
        vc = s.v[layer] if s.n_tokens else np.zeros((0, self.hkv, d), dtype=V.dtype)
        kc, vc = self._kv_values(kc[:s.n_tokens], vc[:s.n_tokens])
        K, V = self._kv_values(K, V)
        return segment_rows(kc, vc, Q, K, V, self.hkv, self.scale, tokens, heads)

    # -- API -------------------------------------------------------------------
    def session_create(self, n_prefix, Q, K, V, compute=True):
        """Q/K/V: [L][n][H][d] storage arrays.  Returns (sid, O [L][n][Hq][d] or None)."""
        if n_prefix <= 0:
            raise OracleError("INVALID_ARG")
        if len(self.sessions) >= self.max_sessions:
            raise OracleError("SESSION_LIMIT")
        s = _Session(n_prefix=n_prefix)
        s.pages = []
        s.pages = self._reserve(s, n_prefix)
        s.pos = list(range(n_prefix))
        sid = self.next_id
        self.next_id += 1
        O = self._compute(s, Q, K, V, -1) if compute else None
        Ks, Vs = self._store_kv(K, V)
        s.k = [np.array(Ks[l]) for l in range(self.L)]
        s.v = [np.array(Vs[l]) for l in range(self.L)]
        s.n_tokens = n_prefix
        s.version = 1
        self.sessions[sid] = s
        return sid, O

    def _compute(self, s, Q, K, V, layer):
        outs = []
        for l in self._layers(layer):
            li = 0 if layer >= 0 else l
            o, _ = self._rows(s, l, Q[li], K[li], V[li])
            outs.append(o)
        return np.stack(outs)

    def _retention_evict(self, s: _Session, m: int) -> None:
        """Alg. 1: if K.size() + |tokens| > K.capacity(): K.evict_oldest(|tokens|)."""
        if s.retention > 0 and s.n_tokens + m > s.retention:
            self._evict(s, m)

    def _next_position(self, s: _Session) -> int:
        return (s.pos[-1] + 1) if s.pos else 0

    def _commit_append(self, s: _Session, new_pages, K, V) -> None:
        m = K.shape[1]
        K, V = self._store_kv(K, V)
        p0 = self._next_position(s)
        s.pages.extend(new_pages)
        for l in range(self.L):
            li = l if K.shape[0] == self.L else 0
            s.k[l] = np.concatenate([s.k[l][:s.n_tokens], K[li]], axis=0)
            s.v[l] = np.concatenate([s.v[l][:s.n_tokens], V[li]], axis=0)
        s.pos = s.pos[:s.n_tokens] + list(range(p0, p0 + m))
        s.n_tokens += m
        s.version += 1

    def session_append(self, sid, Q, K, V, compute=True):
        s = self._check(sid)
        m = K.shape[1]
        if m <= 0:
            raise OracleError("INVALID_ARG")
        snap = self._snapshot()
        try:
            self._retention_evict(s, m)
            new_pages = self._reserve(s, m)
        except OracleError:
            self._restore(snap)                  # all-or-none
            raise
        O = self._compute(s, Q, K, V, -1) if compute else None
        self._commit_append(s, new_pages, K, V)
        return O, s.version

    # -- Region-1 retention (Alg. 1) and prefix aliasing --
    def _evict(self, s: _Session, n: int) -> None:
        if n < 0 or n > s.n_tokens - s.n_prefix:
            raise OracleError("INVALID_ARG")     # SPEC: insufficient SLIDING tokens
        if n == 0:
            return
        for l in range(self.L):                  # the n lowest-position Region-1 tokens leave
            s.k[l] = np.concatenate([s.k[l][:s.n_prefix], s.k[l][s.n_prefix + n:s.n_tokens]], axis=0)
            s.v[l] = np.concatenate([s.v[l][:s.n_prefix], s.v[l][s.n_prefix + n:s.n_tokens]], axis=0)
        s.pos = s.pos[:s.n_prefix] + s.pos[s.n_prefix + n:s.n_tokens]
        s.n_tokens -= n
        s.n_evicted += n
        s.r1_skip += n
        r0_pages = -(-s.n_prefix // self.P)
        if s.n_tokens == s.n_prefix:             # Region 1 empty: all its pages go
            drop = len(s.pages) - r0_pages
            s.r1_skip = 0
        else:                                    # whole pages of evicted slots go
            drop = s.r1_skip // self.P
            s.r1_skip -= drop * self.P
        gone = s.pages[r0_pages:r0_pages + drop]
        s.pages = s.pages[:r0_pages] + s.pages[r0_pages + drop:]
        self._release(gone)
        s.version += 1

    def evict_oldest(self, sid, n):
        s = self._check(sid)
        self._evict(s, n)
        return s.version

    def set_retention(self, sid, max_tokens):
        if max_tokens < 0:
            raise OracleError("INVALID_ARG")
        self._check(sid).retention = max_tokens

    def alias_prefix(self, donor, m):
        """New session whose first m tokens are the donor's first m, shared by reference."""
        d = self._check(donor)
        if m < 0 or m > d.n_tokens or (m > d.n_prefix and d.n_evicted > 0):
            raise OracleError("INVALID_ARG")
        if len(self.sessions) >= self.max_sessions:
            raise OracleError("SESSION_LIMIT")
        end_slot = self.slots_for(d.n_prefix, m, d.r1_skip)
        full = end_slot // self.P
        if end_slot % self.P and not self.free:
            raise OracleError("POOL_EXHAUSTED")
        t = _Session(n_prefix=min(m, d.n_prefix))
        t.pages = list(d.pages[:full])
        for pg in t.pages:
            self.ref[pg] += 1
        if end_slot % self.P:
            t.pages.append(self._take_page())   # the page holding token m-1 is a private copy
        t.k = [np.array(d.k[l][:m]) for l in range(self.L)]
        t.v = [np.array(d.v[l][:m]) for l in range(self.L)]
        t.pos = list(d.pos[:m])
        t.n_tokens = m
        t.version = 1
        sid = self.next_id
        self.next_id += 1
        self.sessions[sid] = t
        return sid

    def session_query(self, sid, Q, K, V, layer=-1, tokens=None, heads=None):
        """Query plane: Q/K/V [L'][m][H][d] (L' = L, or 1 when layer >= 0). No state change."""
        s = self._check(sid)
        if K.shape[1] <= 0:
            raise OracleError("INVALID_ARG")
        outs = []
        for i, l in enumerate(self._layers(layer)):
            o, _ = self._rows(s, l, Q[i], K[i], V[i], tokens, heads)
            outs.append(o)
        return np.stack(outs)

    def flash_query_batch(self, sid, questions, layer):
        """questions: list of (Q [m_i][Hq][d], K, V [m_i][Hkv][d]) for one layer.

        Each f_i sees cache version t plus its own tokens only (reading R-4)."""
        s = self._check(sid)
        return [self._rows(s, layer, q, k, v)[0] for (q, k, v) in questions]

    def batch_run(self, items, layer=-1):
        """Multi-tenant batch with snapshot semantics (reading R-7).

        items: list of dicts {kind: 'append'|'query'|'stateless', session, Q, K, V}
        with per-layer arrays [L'][m][H][d].  Every item reads version t; appends
        publish t+1 after all items are computed.  Pages for appends are reserved
        in item order.  Returns list of O arrays.
        """
        seen = set()
        for it in items:
            if it["kind"] == "append":
                if it["session"] in seen:
                    raise OracleError("INVALID_ARG")
                seen.add(it["session"])
                self._check(it["session"])
        reserved = {}
        snap = self._snapshot()
        try:
            for it in items:                     # retention evictions apply before any item runs
                if it["kind"] == "append":
                    self._retention_evict(self.sessions[it["session"]], it["K"].shape[1])
            for it in items:
                if it["kind"] == "append":
                    s = self.sessions[it["session"]]
                    reserved[it["session"]] = self._reserve(s, it["K"].shape[1])
        except OracleError:
            self._restore(snap)
            raise
        outs = []
        for it in items:
            Q, K, V = it["Q"], it["K"], it["V"]
            if it["kind"] == "stateless":
                tmp = _Session(n_prefix=0)
                outs.append(np.stack([self._rows(tmp, l, Q[i], K[i], V[i])[0]
                                      for i, l in enumerate(self._layers(layer))]))
            else:
                s = self._check(it["session"])
                outs.append(np.stack([self._rows(s, l, Q[i], K[i], V[i])[0]
                                      for i, l in enumerate(self._layers(layer))]))
        if layer < 0 or layer == self.L - 1:
            for it in items:
                if it["kind"] == "append":
                    s = self.sessions[it["session"]]
                    self._commit_append(s, reserved[it["session"]], it["K"], it["V"])
        return outs

    def truncate(self, sid, p):
        """SeqRemove(s, p, inf) (Alg. 3 L540/L547): drop tokens >= p, free pages."""
        s = self._check(sid)
        if p < s.n_prefix or p > s.n_tokens:      # Region 0 is frozen (reading R-17)
            raise OracleError("INVALID_ARG")
        if p == s.n_tokens:
            return s.version
        s.n_tokens = p
        s.pos = s.pos[:p]
        keep = self.pages_for(s.n_prefix, p, s.r1_skip)
        self._release(s.pages[keep:])
        s.pages = s.pages[:keep]
        if p == s.n_prefix:
            s.r1_skip = 0
        s.version += 1
        return s.version

    def session_destroy(self, sid):
        s = self._check(sid)
        self._release(s.pages)
        del self.sessions[sid]

    def page_table(self, sid):
        return list(self._check(sid).pages)

    def info(self, sid):
        s = self._check(sid)
        return dict(n_tokens=s.n_tokens, n_prefix=s.n_prefix, n_pages=len(s.pages), version=s.version,
                    n_evicted=s.n_evicted, retention=s.retention)

    def digest(self, sid) -> int:
        """FNV-1a-64 over, layer-major then token order, the records
        int32 LE layer || int64 LE position || K bytes || V bytes;
        positions are the tokens' original ones (never re-based after eviction)."""
        s = self._check(sid)
        return session_digest(s.k, s.v, s.n_tokens, s.pos)


def session_digest(k_layers, v_layers, n_tokens, positions=None) -> int:
    h = None
    for l, (K, V) in enumerate(zip(k_layers, v_layers)):
        K = np.ascontiguousarray(K[:n_tokens])
        V = np.ascontiguousarray(V[:n_tokens])
        kb = K.reshape(n_tokens, -1).view(np.uint8)
        vb = V.reshape(n_tokens, -1).view(np.uint8)
        rec = np.empty((n_tokens, 12 + kb.shape[1] + vb.shape[1]), dtype=np.uint8)
        rec[:, 0:4] = np.frombuffer(np.int32(l).astype("<i4").tobytes(), dtype=np.uint8)
        pos = np.arange(n_tokens, dtype="<i8") if positions is None else np.asarray(positions[:n_tokens], dtype="<i8")
        rec[:, 4:12] = pos.view(np.uint8).reshape(n_tokens, 8)
        rec[:, 12:12 + kb.shape[1]] = kb
        rec[:, 12 + kb.shape[1]:] = vb
        h = fnv1a64(rec.tobytes(), h)
    if h is None:
        h = fnv1a64(b"")
    return h


def greedy_sample(logits: np.ndarray):
    """Greedy sampling of P:383-385 with the logit gap of Eq. flash-cache and
    Eq. logit-gap, per SPEC greedy_sample: for each row, the argmax with ties
    toward the lowest token id and gap = l1 - l2, l2 the second-highest value (== l1 on a
    tie at the top).  Rows are fp32 values or bf16 bits (uint16, decoded exactly); the gap
    is one fp32 subtraction, as the device computes it.  NaN logits are ignored; a row
    without a non-NaN logit gives (-1, 0).  Returns (ids int32 [rows], gap float32 [rows])."""
    x = logits
    if x.dtype == np.uint16:
        x = (x.astype(np.uint32) << 16).view(np.float32)
    x = np.asarray(x, dtype=np.float32)
    ids = np.empty(x.shape[0], dtype=np.int32)
    gap = np.empty(x.shape[0], dtype=np.float32)
    for r in range(x.shape[0]):
        keep = np.flatnonzero(~np.isnan(x[r]))
        if keep.size == 0:
            ids[r], gap[r] = -1, 0.0
            continue
        vals = x[r][keep]
        j = int(np.argmax(vals))                 # first occurrence = lowest id among ties
        l1 = vals[j]
        l2 = np.sort(vals)[-2] if vals.size > 1 else np.float32(-np.inf)
        ids[r] = keep[j]
        gap[r] = np.float32(l1) - np.float32(l2)
    return ids, gap


def memory_model_bytes(num_layers, d, n_ctx, sizeof) -> int:
    """Eq. (memory): M_KV = 2 * L * d * n_ctx * sizeof(dtype)."""
    return 2 * num_layers * d * n_ctx * sizeof


def query_macs(n_cached: int, m: int, num_q_heads: int, d: int) -> int:
    """MACs of QK^T for m new rows over n cached keys ("O(m*n)"):
    Hq * d * sum_{i<m} (n + i + 1)  (the same count again for PV)."""
    return num_q_heads * d * (m * n_cached + m * (m + 1) // 2)


# ----------------------------------------------------------------------------
# fused data-plane projection (`Forward` of Alg. 1)
# ----------------------------------------------------------------------------
def round_bf16(x: np.ndarray) -> np.ndarray:
    """fp64 -> bf16 bit patterns (uint16), one round-to-nearest-even to an 8-bit
    significand (reading R-10: outputs are rounded once).  Finite normal range only."""
    x = np.asarray(x, dtype=np.float64)
    m, e = np.frexp(x)                         # x = m * 2^e, 0.5 <= |m| < 1
    q = np.round(m * 256.0)                    # 8 significant bits, half to even
    y = np.ldexp(q, e - 8).astype(np.float32)  # exact: q has <= 9 bits
    return (y.view(np.uint32) >> np.uint32(16)).astype(np.uint16)


def qkv_projection(x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """[Q | K | V] = X W^T: the q/k/v projections of the paper's model (Llama-3.1-8B,
    P:641) inside `Forward` (Alg. 1).  x [n][hidden], w [n_out][hidden]
    (nn.Linear weight), bf16 bits or floats, decoded exactly; one fp64 matmul."""
    return to_f64(x) @ to_f64(w).T


def rope(x: np.ndarray, positions, theta: float) -> np.ndarray:
    """Rotary position embedding, rotate-half form (reading R-21; the paper's model
    uses RoPE, SURVEY A-6): for x [n][H][d] and pair j < d/2 of every head,
        angle = positions[i] * theta^(-2j/d)
        x'[j]       = x[j] cos(angle) - x[j + d/2] sin(angle)
        x'[j + d/2] = x[j + d/2] cos(angle) + x[j] sin(angle)."""
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    half = d // 2
    inv = np.array([theta ** (-2.0 * j / d) for j in range(half)], dtype=np.float64)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv[None, :]
    c = np.cos(ang)[:, None, :]
    s = np.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def qkv_rope(x, w, num_q_heads: int, num_kv_heads: int, head_dim: int, pos0: int, theta: float):
    """The fused projection's result in fp64: Q, K, V of shapes [n][Hq][d], [n][Hkv][d],
    [n][Hkv][d]; RoPE on Q and K at positions pos0 .. pos0+n-1 (theta <= 0: none)."""
    y = qkv_projection(x, w)
    n = y.shape[0]
    q = y[:, : num_q_heads * head_dim].reshape(n, num_q_heads, head_dim)
    k = y[:, num_q_heads * head_dim: (num_q_heads + num_kv_heads) * head_dim].reshape(n, num_kv_heads, head_dim)
    v = y[:, (num_q_heads + num_kv_heads) * head_dim:].reshape(n, num_kv_heads, head_dim)
    if theta > 0:
        pos = np.arange(pos0, pos0 + n)
        q, k = rope(q, pos, theta), rope(k, pos, theta)
    return q, k, v
