"""Seeded synthetic input streams for the stateful-session attention path.

This module is shared by the oracle tests, the GPU parity tests, ``bench.py``
and ``__graft_entry__.smoke()``.  It holds **no attention arithmetic** — only a
counter-based random number generator, the stream recipes of DESIGN.md §4
(SURVEY.md §8(d) "Synthetic input streams") and bf16 round-to-nearest-even.

Every element is a pure function of
``(seed, stream, session, domain, layer, tensor, token, head, dim)`` so any
chunking of a session's token stream sees identical bits (
SPEC S:79 "chunked = full").  ``domain`` 0 is the session's data tokens
(C = [S; D_1..D_k], §2) indexed by global position; domain
``1 + j`` is the j-th query Q_j and ``FLASH_DOMAIN + i`` the i-th
registered Flash Query f_i (Eq. flash-eval).

The generator is implemented twice — numpy (``*_np``) and torch (``*_torch``,
any device) — with integer-only hashing and exactly-rounded float32 steps, so
both produce identical bits (checked by ``tests/test_streams.py``).  A normal
variate is the Irwin–Hall sum of four 16-bit uniforms, standardised; it has
unit variance and bounded support (|x| <= 3.46).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

TENSOR_Q, TENSOR_K, TENSOR_V = 0, 1, 2
FLASH_DOMAIN = 1 << 20
_M32 = 0xFFFFFFFF
# 1/sqrt(4 * (2^32-1)/12 ...) : Irwin-Hall(4) of U{0..65535} has variance
# 4 * (65536^2 - 1) / 12; standardise with this float32 constant.
_IH_SCALE = np.float32(1.0 / math.sqrt(4.0 * (65536.0 ** 2 - 1.0) / 12.0))
_IH_MEAN = 2 * 65535  # 4 * 65535 / 2

STREAMS = ("peaked", "flat", "market", "needle")


def _h32(x: int) -> int:
    """lowbias32 integer hash on a python int (uint32 semantics)."""
    x &= _M32
    x ^= x >> 16
    x = (x * 0x7FEB352D) & _M32
    x ^= x >> 15
    x = (x * 0x846CA68B) & _M32
    x ^= x >> 16
    return x


def _base_key(seed: int, stream: int, session: int, domain: int, layer: int, tensor: int) -> int:
    h = _h32(seed ^ 0xA5A5A5A5)
    for v in (stream, session, domain, layer, tensor):
        h = _h32(h ^ (v & _M32) ^ ((v >> 32) & _M32) * 0x9E3779B1)
    return h


def _h32_np(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64) & _M32
    x ^= x >> np.uint64(16)
    x = (x * np.uint64(0x7FEB352D)) & np.uint64(_M32)
    x ^= x >> np.uint64(15)
    x = (x * np.uint64(0x846CA68B)) & np.uint64(_M32)
    x ^= x >> np.uint64(16)
    return x


def _normal_np(base: int, idx: np.ndarray) -> np.ndarray:
    """Standard-normal-like float32 from a flat uint64 counter array."""
    u = _h32_np(idx ^ np.uint64(base))
    w = _h32_np(u ^ np.uint64(0x9E3779B9))
    s = (u & np.uint64(0xFFFF)) + (u >> np.uint64(16)) + (w & np.uint64(0xFFFF)) + (w >> np.uint64(16))
    return (s.astype(np.int64) - _IH_MEAN).astype(np.float32) * _IH_SCALE


def _normal_torch(base: int, idx):
    import torch
    m = 0xFFFFFFFF

    def h(x):
        x = x & m
        x = x ^ (x >> 16)
        x = (x * 0x7FEB352D) & m   # wraps in int64; low 32 bits exact
        x = x ^ (x >> 15)
        x = (x * 0x846CA68B) & m
        x = x ^ (x >> 16)
        return x

    u = h(idx ^ base)
    w = h(u ^ 0x9E3779B9)
    s = (u & 0xFFFF) + (u >> 16) + (w & 0xFFFF) + (w >> 16)
    return (s - _IH_MEAN).to(torch.float32) * float(_IH_SCALE)


def bf16_bits_np(x: np.ndarray) -> np.ndarray:
    """float32 -> bf16 bit pattern (uint16), round to nearest even."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))
    return (b >> np.uint64(16)).astype(np.uint16)


def bf16_bits_to_f32_np(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << np.uint32(16)).view(np.float32)


@dataclass(frozen=True)
class StreamSpec:
    """One synthetic stream.

    peaked: K,V ~ N(0,1), Q ~ N(0, alpha^2) with alpha=3 (logit std ~3).
    flat:   Q,K,V ~ N(0,1).
    market: 16-token records ("~16 tokens per sample"): data token t >= iid_prefix
            has K = E[t mod 16] + 0.5 N(0,1), E fixed per (layer, kv head); V ~ N(0,1);
            Q ~ N(0, alpha^2).  The first ``iid_prefix`` tokens (R0) are i.i.d.
    needle: every key ~ 0.1 N(0,1) except the data tokens at ``needles`` whose K is
            gamma * u_g (u_g a fixed unit vector per kv head); every query row of group g
            is gamma * u_g; V ~ N(0,1).  Q6 "exact value retrieval".
    """
    name: str = "peaked"
    seed: int = 0
    alpha: float = 3.0
    iid_prefix: int = 512
    gamma: float = 19.0
    needles: tuple = ()

    @property
    def stream_id(self) -> int:
        return STREAMS.index(self.name)


def _unit_vectors(spec: StreamSpec, layer: int, hkv: int, d: int) -> np.ndarray:
    base = _base_key(spec.seed, spec.stream_id, 0, 0xFFFF, layer, 7)
    idx = np.arange(hkv * d, dtype=np.uint64)
    u = _normal_np(base, idx).astype(np.float64).reshape(hkv, d)
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    return u.astype(np.float32)


def _role_embeddings(spec: StreamSpec, layer: int, hkv: int, d: int) -> np.ndarray:
    base = _base_key(spec.seed, spec.stream_id, 0, 0xFFFE, layer, 6)
    idx = np.arange(16 * hkv * d, dtype=np.uint64)
    return _normal_np(base, idx).reshape(16, hkv, d)


def gen_f32(spec: StreamSpec, session: int, domain: int, layer: int, tensor: int,
            tok0: int, ntok: int, heads: int, d: int) -> np.ndarray:
    """float32 values [ntok][heads][d] of one tensor (numpy)."""
    base = _base_key(spec.seed, spec.stream_id, session, domain, layer, tensor)
    idx = (np.arange(ntok, dtype=np.uint64)[:, None, None] + np.uint64(tok0)) * np.uint64(heads * d) \
        + np.arange(heads, dtype=np.uint64)[None, :, None] * np.uint64(d) \
        + np.arange(d, dtype=np.uint64)[None, None, :]
    x = _normal_np(base, idx.reshape(-1)).reshape(ntok, heads, d)
    return _shape_stream(spec, x, domain, layer, tensor, tok0, ntok, heads, d)


def _shape_stream(spec, x, domain, layer, tensor, tok0, ntok, heads, d):
    """Apply the stream recipe to standard normals (numpy or torch, same float32 ops)."""
    name = spec.name
    if name == "flat":
        return x
    if name == "peaked":
        return x * np.float32(spec.alpha) if tensor == TENSOR_Q else x
    if name == "market":
        if tensor == TENSOR_Q:
            return x * np.float32(spec.alpha)
        if tensor == TENSOR_K and domain == 0:
            emb = _role_embeddings(spec, layer, heads, d)
            t = np.arange(tok0, tok0 + ntok)
            rec = t >= spec.iid_prefix
            out = x * np.float32(0.5) + _as_like(x, emb[t % 16])
            return _where_rows(x, rec, out)
        return x
    if name == "needle":
        if tensor != TENSOR_K:
            return x  # V ~ N(0,1); Q rows are built by needle_queries()
        out = x * np.float32(0.1)
        if domain == 0 and spec.needles:
            u = _unit_vectors(spec, layer, heads, d) * np.float32(spec.gamma)
            t = np.arange(tok0, tok0 + ntok)
            hit = np.isin(t, np.asarray(spec.needles))
            needle_rows = _as_like(x, np.broadcast_to(u, (ntok, heads, d)).copy())
            out = _where_rows(x, hit, needle_rows, out)
        return out
    raise ValueError(name)


def _as_like(x, arr):
    if isinstance(x, np.ndarray):
        return arr.astype(np.float32)
    import torch
    return torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).to(x.device)


def _where_rows(x, mask_rows, a, b=None):
    if b is None:
        b = x
    if isinstance(x, np.ndarray):
        return np.where(mask_rows[:, None, None], a, b)
    import torch
    m = torch.from_numpy(np.asarray(mask_rows)).to(x.device)[:, None, None]
    return torch.where(m, a, b)


def needle_queries(spec: StreamSpec, layer: int, ntok: int, hq: int, hkv: int, d: int):
    """Needle-stream Q rows: every q head of group g is gamma * u_g (A-5 GQA map)."""
    u = _unit_vectors(spec, layer, hkv, d) * np.float32(spec.gamma)
    g = hq // hkv
    q = np.repeat(u, g, axis=0)  # [hq][d], head h -> kv head h // g
    return np.broadcast_to(q, (ntok, hq, d)).astype(np.float32).copy()


def gen_tensor_np(spec: StreamSpec, session: int, domain: int, layer: int, tensor: int,
                  tok0: int, ntok: int, heads: int, d: int, hkv: int | None = None,
                  dtype: str = "bf16") -> np.ndarray:
    """Storage-dtype values: uint16 bf16 bits, or float32 for dtype 'fp32'."""
    if spec.name == "needle" and tensor == TENSOR_Q:
        x = needle_queries(spec, layer, ntok, heads, hkv or heads, d)
    else:
        x = gen_f32(spec, session, domain, layer, tensor, tok0, ntok, heads, d)
    return bf16_bits_np(x) if dtype == "bf16" else np.ascontiguousarray(x, dtype=np.float32)


def gen_tensor_torch(spec: StreamSpec, session: int, domain: int, layer: int, tensor: int,
                     tok0: int, ntok: int, heads: int, d: int, hkv: int | None = None,
                     dtype: str = "bf16", device="cpu"):
    """Same bits as :func:`gen_tensor_np`, produced by torch on ``device``.

    Returns a torch tensor of dtype bfloat16 (bit-identical to the numpy uint16
    pattern) or float32.
    """
    import torch
    if spec.name == "needle" and tensor == TENSOR_Q:
        x = torch.from_numpy(needle_queries(spec, layer, ntok, heads, hkv or heads, d)).to(device)
    else:
        base = _base_key(spec.seed, spec.stream_id, session, domain, layer, tensor)
        idx = (torch.arange(ntok, dtype=torch.int64, device=device)[:, None, None] + tok0) * (heads * d) \
            + torch.arange(heads, dtype=torch.int64, device=device)[None, :, None] * d \
            + torch.arange(d, dtype=torch.int64, device=device)[None, None, :]
        x = _normal_torch(base, idx)
        x = _shape_stream_torch(spec, x, domain, layer, tensor, tok0, ntok, heads, d)
    if dtype == "fp32":
        return x.contiguous()
    b = x.contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return _i64_to_bf16(b)


def _i64_to_bf16(b):
    import torch
    b16 = (b & 0xFFFF)
    b16 = torch.where(b16 >= 0x8000, b16 - 0x10000, b16).to(torch.int16)
    return b16.view(torch.bfloat16)


def _shape_stream_torch(spec, x, domain, layer, tensor, tok0, ntok, heads, d):
    name = spec.name
    if name == "flat":
        return x
    if name == "peaked":
        return x * float(np.float32(spec.alpha)) if tensor == TENSOR_Q else x
    if name in ("market", "needle"):
        return _shape_stream(spec, x, domain, layer, tensor, tok0, ntok, heads, d)
    raise ValueError(name)


# ----------------------------------------------------------------------------
# fused projection inputs: hidden states X and the q/k/v weight
# ----------------------------------------------------------------------------
TENSOR_X, TENSOR_W = 3, 4


def gen_hidden(seed: int, session: int, domain: int, layer: int, tok0: int, n: int, hidden: int, device=None):
    """Hidden-state rows X [n][hidden], bf16, i.i.d. N(0,1) per (token, dim); a pure
    function of the global token index (chunking-invariant).  numpy uint16 bits when
    ``device`` is None, else a torch bfloat16 tensor on ``device`` (same bits)."""
    spec = StreamSpec("flat", seed=seed)
    if device is None:
        return gen_tensor_np(spec, session, domain, layer, TENSOR_X, tok0, n, 1, hidden).reshape(n, hidden)
    return gen_tensor_torch(spec, session, domain, layer, TENSOR_X, tok0, n, 1, hidden, device=device).reshape(n, hidden)


def gen_qkv_weight(seed: int, layer: int, n_out: int, hidden: int, device=None):
    """q/k/v projection weight W [n_out][hidden] (nn.Linear layout), bf16, N(0, 1/hidden)
    so that X W^T has unit variance (random init; no trained weights)."""
    spec = StreamSpec("flat", seed=seed)
    scale = np.float32(1.0 / math.sqrt(hidden))
    if device is None:
        x = gen_f32(spec, 0, 0xFFFD, layer, TENSOR_W, 0, n_out, 1, hidden) * scale
        return bf16_bits_np(x).reshape(n_out, hidden)
    import torch
    base = _base_key(spec.seed, spec.stream_id, 0, 0xFFFD, layer, TENSOR_W)
    out = torch.empty(n_out, hidden, dtype=torch.bfloat16, device=device)
    step = max(1, (1 << 24) // hidden)
    for r0 in range(0, n_out, step):   # bounded temporaries
        r1 = min(n_out, r0 + step)
        idx = torch.arange(r0 * hidden, r1 * hidden, dtype=torch.int64, device=device)
        x = _normal_torch(base, idx) * float(scale)
        b = x.contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        b = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
        out[r0:r1] = _i64_to_bf16(b).view(r1 - r0, hidden)
    return out
