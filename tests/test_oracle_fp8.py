"""Pins for the oracle's FP8 (E4M3) KV-cache variant (reading
R-22): the code table against the format's closed forms, the quantizer against
brute force over the table and against torch's float8_e4m3fn cast (an independent
library implementation), saturation, and the session-level identities that must
still hold when the cache holds codes.  CPU only."""
import numpy as np
import pytest
import torch

import oracle
import streams


def test_e4m3_code_table_closed_forms():
    d = oracle.e4m3_decode
    codes = np.array([0x00, 0x01, 0x07, 0x08, 0x38, 0x3F, 0x40, 0x7E, 0x80, 0x81, 0xB8, 0xFE], dtype=np.uint8)
    want = [0.0, 2.0**-9, 7 * 2.0**-9, 2.0**-6, 1.0, 1.875, 2.0, 448.0, -0.0, -(2.0**-9), -1.0, -448.0]
    got = d(codes)
    assert np.array_equal(got, np.array(want))
    assert np.signbit(got[8]) and not np.signbit(got[0])
    assert np.isnan(d(np.array([0x7F, 0xFF], dtype=np.uint8))).all()
    pos = d(np.arange(127, dtype=np.uint8))
    assert np.all(np.diff(pos) > 0)                     # monotone: codes order like values
    # spacing: 2^-9 through the subnormals and the first binade, then doubling per binade
    assert np.allclose(np.diff(pos[:16]), 2.0**-9)
    for e in range(1, 15):
        b = pos[8 * e: 8 * e + 8]
        assert np.allclose(np.diff(b), 2.0 ** (e - 7 - 3))


def test_e4m3_decode_matches_torch_for_every_code():
    codes = np.arange(256, dtype=np.uint8)
    t = torch.from_numpy(codes).view(torch.float8_e4m3fn).to(torch.float64).numpy()
    mine = oracle.e4m3_decode(codes)
    assert np.array_equal(np.isnan(t), np.isnan(mine))
    ok = ~np.isnan(t)
    assert np.array_equal(t[ok], mine[ok])


def _brute(y: np.ndarray) -> np.ndarray:
    """Nearest finite E4M3 value by exhaustive search, ties to the even code, saturating."""
    table = oracle.e4m3_decode(np.arange(127, dtype=np.uint8))
    out = np.empty(y.shape, dtype=np.uint8)
    for i, v in enumerate(y):
        a = min(abs(float(v)), 448.0)
        dist = np.abs(table - a)
        best = np.flatnonzero(dist == dist.min())
        c = int(best[0]) if len(best) == 1 else int(best[best % 2 == 0][0])
        out[i] = c | (0x80 if np.signbit(v) else 0)
    return out


def test_e4m3_encode_brute_force_including_ties():
    rng = np.random.default_rng(3)
    table = oracle.e4m3_decode(np.arange(127, dtype=np.uint8))
    mids = (table[1:] + table[:-1]) / 2                 # every tie point
    y = np.concatenate([
        rng.standard_normal(3000) * np.exp2(rng.uniform(-12, 9, 3000)),
        mids, -mids, table, -table,
        np.nextafter(mids.astype(np.float32), np.float32(np.inf)).astype(np.float64),
        np.nextafter(mids.astype(np.float32), np.float32(0)).astype(np.float64),
        [448.0, 455.0, 464.0, 465.0, 1e6, -1e30, 1e-12, -1e-12, 0.0, -0.0],
    ]).astype(np.float32)
    got = oracle.e4m3_encode(y, 1.0)
    assert np.array_equal(got, _brute(y.astype(np.float64)))


def test_e4m3_encode_matches_torch_cast_in_range():
    # torch's fp32 -> float8_e4m3fn cast is round-to-nearest-even; it overflows to NaN
    # instead of saturating, so compare below the largest rounding-to-448 value
    rng = np.random.default_rng(5)
    y = (rng.standard_normal(200000) * np.exp2(rng.uniform(-14, 8, 200000))).astype(np.float32)
    y = y[np.abs(y) < 464]
    want = torch.from_numpy(y).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    assert np.array_equal(oracle.e4m3_encode(y, 1.0), want)


def test_e4m3_encode_saturates_and_divides_in_fp32():
    big = np.array([448.0, 449.0, 500.0, 3e38, -470.0], dtype=np.float32)
    assert list(oracle.e4m3_encode(big, 1.0)) == [0x7E, 0x7E, 0x7E, 0x7E, 0xFE]
    assert oracle.e4m3_encode(np.array([np.nan], dtype=np.float32), 1.0)[0] == 0x7F
    # the quotient is formed once in fp32 (the decision is taken in the kernel's precision)
    rng = np.random.default_rng(9)
    x = streams.bf16_bits_np(rng.standard_normal(5000) * 3)
    for scale in (1 / 64, 0.0123, 3.0):
        q = (oracle.to_f64(x).astype(np.float32) / np.float32(scale)).astype(np.float32)
        assert np.array_equal(oracle.e4m3_encode(x, scale), oracle.e4m3_encode(q, 1.0))
    # a power-of-two scale commutes with the grid: encode(decode(c) * s, s) == c
    codes = np.array([c for c in range(256) if c not in (0x7F, 0xFF)], dtype=np.uint8)
    vals = (oracle.e4m3_decode(codes) * (1 / 64)).astype(np.float32)
    assert np.array_equal(oracle.e4m3_encode(vals, 1 / 64), codes)


def _fp8_store(L=1, hq=4, hkv=2, d=16, P=16, npages=64, ks=1 / 16, vs=1 / 32):
    return oracle.OracleStore(L, hq, hkv, d, P, npages, dtype="bf16", kv_format="e4m3",
                              k_scale=ks, v_scale=vs)


def _kv(rng, L, m, h, d, sd=1.0):
    return streams.bf16_bits_np(rng.standard_normal((L, m, h, d)) * sd)


def test_fp8_incremental_equals_recompute_over_dequantized_stream():
    rng = np.random.default_rng(11)
    L, hq, hkv, d = 1, 4, 2, 16
    st = _fp8_store(L, hq, hkv, d)
    segs = [20, 7, 33]
    Qs = [_kv(rng, L, m, hq, d, 3.0) for m in segs]
    Ks = [_kv(rng, L, m, hkv, d) for m in segs]
    Vs = [_kv(rng, L, m, hkv, d) for m in segs]
    sid, O0 = st.session_create(segs[0], Qs[0], Ks[0], Vs[0])
    outs = [O0]
    for i in (1, 2):
        O, _ = st.session_append(sid, Qs[i], Ks[i], Vs[i])
        outs.append(O)
    q = _kv(rng, L, 5, hq, d, 3.0)
    kq, vq = _kv(rng, L, 5, hkv, d), _kv(rng, L, 5, hkv, d)
    Oq = st.session_query(sid, q, kq, vq)
    # full recompute over the dequantized concatenation (no session state)
    kall = np.concatenate([k[0] for k in Ks] + [kq[0]])
    vall = np.concatenate([v[0] for v in Vs] + [vq[0]])
    qall = np.concatenate([x[0] for x in Qs] + [q[0]])
    kdq = oracle.e4m3_decode(oracle.e4m3_encode(kall, 1 / 16)) / 16
    vdq = oracle.e4m3_decode(oracle.e4m3_encode(vall, 1 / 32)) / 32
    ref = oracle.full_recompute(qall, kdq, vdq, hkv, oracle.default_scale(d))
    got = np.concatenate([o[0] for o in outs] + [Oq[0]])
    assert np.max(np.abs(ref - got)) <= 1e-12
    # the quantization is not a no-op: the bf16 stream gives a different answer
    ref_bf16 = oracle.full_recompute(qall, kall, vall, hkv, oracle.default_scale(d))
    assert np.max(np.abs(ref_bf16 - got)) > 1e-4


def test_fp8_digest_is_over_codes_and_query_is_state_neutral():
    rng = np.random.default_rng(12)
    st = _fp8_store()
    K, V = _kv(rng, 1, 40, 2, 16), _kv(rng, 1, 40, 2, 16)
    sid, _ = st.session_create(40, _kv(rng, 1, 40, 4, 16), K, V)
    want = oracle.session_digest([oracle.e4m3_encode(K[0], 1 / 16)], [oracle.e4m3_encode(V[0], 1 / 32)], 40)
    assert st.digest(sid) == want
    st.session_query(sid, _kv(rng, 1, 3, 4, 16), _kv(rng, 1, 3, 2, 16), _kv(rng, 1, 3, 2, 16))
    assert st.digest(sid) == want and st.info(sid)["version"] == 1


def test_fp8_closed_forms_constant_v_and_single_key():
    st = _fp8_store(ks=1 / 16, vs=1 / 64)
    rng = np.random.default_rng(13)
    n = 24
    K = _kv(rng, 1, n, 2, 16)
    V = streams.bf16_bits_np(np.full((1, n, 2, 16), 0.5))      # 0.5 * 64 = 32: on the grid
    sid, O = st.session_create(n, _kv(rng, 1, n, 4, 16, 3.0), K, V)
    assert np.array_equal(O, np.full(O.shape, 0.5))
    # a row whose key set is its own token returns that token's dequantized V
    st2 = _fp8_store(vs=1 / 64)
    v1 = _kv(rng, 1, 1, 2, 16)
    _, O1 = st2.session_create(1, _kv(rng, 1, 1, 4, 16), _kv(rng, 1, 1, 2, 16), v1)
    vdq = oracle.e4m3_decode(oracle.e4m3_encode(v1, 1 / 64)) / 64
    assert np.array_equal(O1[0, 0, 0], vdq[0, 0, 0]) and np.array_equal(O1[0, 0, 3], vdq[0, 0, 1])
