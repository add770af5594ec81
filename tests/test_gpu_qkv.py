"""GPU parity of the fused data-plane projection (kernels_qkv.cu)
against the fp64 oracle (oracle.qkv_rope, reading R-21).

Tolerance (derived): the kernel accumulates in fp32 and rounds once to
bf16, so each output is within half a bf16 ulp of the exact value plus the fp32
accumulation error: |gpu - exact| <= 2^-8 |exact| + 1e-3.  The north-star bf16 bound
(max-abs 2e-2 / mean-abs 2e-3) is checked as well.  K/V placed in pages by the fused
append must be bit-identical to the dense output of the same projection (index work).
"""
import numpy as np
import pytest

import oracle
import streams
from helpers import TOL, errors, f64, from_dev, gen_qkv, to_dev

pytestmark = pytest.mark.gpu


def _ssa():
    import paper_2605_13784_b200 as ssa
    return ssa


def _check_proj(got_bits, exact, what):
    g = f64(got_bits)
    err = np.abs(g - exact)
    bound = 2.0 ** -8 * np.abs(exact) + 1e-3
    bad = np.argwhere(err > bound)
    assert bad.size == 0, f"{what}: {len(bad)} elements over the bound, first {bad[:3].tolist()}"
    assert err.max() <= TOL["bf16"][0] and err.mean() <= TOL["bf16"][1], (what, err.max(), err.mean())
    same = np.mean(got_bits == oracle.round_bf16(exact))
    assert same >= 0.95, f"{what}: only {same:.3f} of outputs equal the correctly rounded value"


def _proj_case(cuda, st, hq, hkv, hidden, n, pos0, theta, seed=11):
    import torch
    d = 128
    X = streams.gen_hidden(seed, 0, 0, 0, pos0, n, hidden)
    W = streams.gen_qkv_weight(seed, 0, (hq + 2 * hkv) * d, hidden)
    Q = torch.full((n, hq, d), float("nan"), dtype=torch.bfloat16, device=cuda)
    K = torch.full((n, hkv, d), float("nan"), dtype=torch.bfloat16, device=cuda)
    V = torch.full((n, hkv, d), float("nan"), dtype=torch.bfloat16, device=cuda)
    st.qkv_rope(to_dev(X, cuda), to_dev(W, cuda), Q, K, V, pos0=pos0, rope_theta=theta)
    torch.cuda.synchronize()
    q, k, v = oracle.qkv_rope(X, W, hq, hkv, d, pos0, theta)
    return (from_dev(Q), from_dev(K), from_dev(V)), (q, k, v)


@pytest.mark.parametrize("hq,hkv,hidden,n,pos0,theta", [
    (8, 2, 512, 32, 0, 500000.0),        # 6 column tiles, split-K 8 (one k-block per CTA)
    (8, 2, 512, 1, 7, 500000.0),         # single token
    (8, 2, 1024, 200, 1000, 10000.0),    # ragged second token tile
    (5, 1, 256, 64, 3, 500000.0),        # odd head count: half-empty last column tile
    (6, 1, 256, 130, 5, 0.0),            # no rotary embedding: the plain GEMM
    (4, 2, 256, 300, 131000, 500000.0),  # large positions (angle reduction)
    (32, 8, 4096, 256, 32512, 500000.0),  # BJ.configs[1] append shape (split-K 2)
    (32, 8, 4096, 32, 32768, 500000.0),   # BJ.configs[1] query shape (split-K 5)
    (32, 8, 4096, 1024, 0, 500000.0),     # 192 tiles, no split
])
def test_qkv_rope_parity(cuda, hq, hkv, hidden, n, pos0, theta):
    ssa = _ssa()
    st = ssa.Store(1, hq, hkv, 128, page_size=64, num_pages=4, max_sessions=1, dtype="bf16")
    got, ref = _proj_case(cuda, st, hq, hkv, hidden, n, pos0, theta)
    for g, r, name in zip(got, ref, "QKV"):
        _check_proj(g, r, name)
    st.close()


def test_qkv_rope_negative_control_wrong_position(cuda):
    """A position off by one must fail the bound (the check is discriminating)."""
    ssa = _ssa()
    st = ssa.Store(1, 8, 2, 128, page_size=64, num_pages=4, max_sessions=1, dtype="bf16")
    got, _ = _proj_case(cuda, st, 8, 2, 512, 64, 100, 10000.0)
    _, ref = _proj_case(cuda, st, 8, 2, 512, 64, 100, 10000.0)
    q_wrong = oracle.qkv_rope(streams.gen_hidden(11, 0, 0, 0, 100, 64, 512),
                              streams.gen_qkv_weight(11, 0, 12 * 128, 512), 8, 2, 128, 101, 10000.0)[0]
    with pytest.raises(AssertionError):
        _check_proj(got[0], q_wrong, "Q (pos + 1)")
    _check_proj(got[0], ref[0], "Q")
    st.close()


def _oracle_layers(X, W, hq, hkv, pos0, theta):
    qs, ks, vs = [], [], []
    for x, w in zip(X, W):
        q, k, v = oracle.qkv_rope(x, w, hq, hkv, 128, pos0, theta)
        qs.append(oracle.round_bf16(q))
        ks.append(oracle.round_bf16(k))
        vs.append(oracle.round_bf16(v))
    return np.stack(qs), np.stack(ks), np.stack(vs)


@pytest.mark.parametrize("P", [16, 64])
def test_append_and_query_fused_parity(cuda, P):
    """Session create (plain path) -> fused appends (K/V straight into pages, no scatter)
    -> fused query; outputs vs the oracle, page table bit-exact, paged K/V bit-identical
    to the dense projection output, and the query leaves the session unchanged."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, hidden, theta = 2, 8, 2, 128, 512, 500000.0
    spec = streams.StreamSpec("peaked", seed=3)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=256, max_sessions=2, dtype="bf16")
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=256, dtype="bf16")
    st.set_option(ssa.OPT_TIMING, 1)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 100)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    sid = st.session_create(to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    rsid, _ = ref.session_create(100, Q, K, V)
    W = [streams.gen_qkv_weight(5, l, (hq + 2 * hkv) * d, hidden) for l in range(L)]
    Wd = [to_dev(w, cuda) for w in W]
    pos = 100
    for n in (200, 37, 128):
        X = [streams.gen_hidden(5, 0, 0, l, pos, n, hidden) for l in range(L)]
        ticket = st.append_begin(sid, n)
        outs = []
        for l in range(L):
            Ol = torch.empty((n, hq, d), dtype=torch.bfloat16, device=cuda)
            st.append_layer_fused(sid, ticket, l, to_dev(X[l], cuda), Wd[l], Ol, rope_theta=theta)
            outs.append(from_dev(Ol))
        st.append_commit(sid, ticket)
        Qr, Kr, Vr = _oracle_layers(X, W, hq, hkv, pos, theta)
        Oref, _ = ref.session_append(rsid, Qr, Kr, Vr)
        mx, mn = errors(np.stack(outs), Oref)
        assert mx <= TOL["bf16"][0] and mn <= TOL["bf16"][1], (n, mx, mn)
        assert st.page_table(sid) == ref.page_table(rsid)
        assert st.info(sid) == ref.info(rsid)
        for l in range(L):
            Kp, Vp = st.read_kv(sid, l, pos, n)
            Kd = torch.empty((n, hkv, d), dtype=torch.bfloat16, device=cuda)
            Vd = torch.empty_like(Kd)
            Qd = torch.empty((n, hq, d), dtype=torch.bfloat16, device=cuda)
            st.qkv_rope(to_dev(X[l], cuda), Wd[l], Qd, Kd, Vd, pos0=pos, rope_theta=theta)
            torch.cuda.synchronize()
            assert np.array_equal(Kp, from_dev(Kd)) and np.array_equal(Vp, from_dev(Vd)), (n, l)
            _check_proj(Kp, oracle.qkv_rope(X[l], W[l], hq, hkv, d, pos, theta)[1], "paged K")
        pos += n
    # fused query: 32 tokens after the cache, per layer; state unchanged
    dig, info = st.digest(sid), st.info(sid)
    n_q = 32
    for l in range(L):
        Xq = streams.gen_hidden(5, 0, 1, l, pos, n_q, hidden)
        Oq = torch.empty((n_q, hq, d), dtype=torch.bfloat16, device=cuda)
        st.session_query_fused(sid, l, to_dev(Xq, cuda), Wd[l], Oq, rope_theta=theta)
        q, k, v = oracle.qkv_rope(Xq, W[l], hq, hkv, d, pos, theta)
        Oref = ref.session_query(rsid, oracle.round_bf16(q)[None], oracle.round_bf16(k)[None],
                                 oracle.round_bf16(v)[None], layer=l)
        mx, mn = errors(from_dev(Oq)[None], Oref)
        assert mx <= TOL["bf16"][0] and mn <= TOL["bf16"][1], (l, mx, mn)
    assert st.digest(sid) == dig and st.info(sid) == info
    t = st.timing()
    assert t["qkv_rope"][1] >= 2 * L and t["scatter"][1] == 1   # only the create scattered
    st.close()


def test_fused_rejects_bad_arguments(cuda):
    import torch
    ssa = _ssa()
    st = ssa.Store(1, 8, 2, 128, page_size=64, num_pages=8, max_sessions=1, dtype="bf16")
    X = torch.zeros((4, 100), dtype=torch.bfloat16, device=cuda)      # hidden % 64 != 0
    W = torch.zeros((12 * 128, 100), dtype=torch.bfloat16, device=cuda)
    Q = torch.empty((4, 8, 128), dtype=torch.bfloat16, device=cuda)
    K = torch.empty((4, 2, 128), dtype=torch.bfloat16, device=cuda)
    with pytest.raises(ssa.SsaError):
        st.qkv_rope(X, W, Q, K, K)
    Xh = torch.zeros((4, 128), dtype=torch.bfloat16)                  # host X
    Wd = torch.zeros((12 * 128, 128), dtype=torch.bfloat16, device=cuda)
    with pytest.raises(ssa.SsaError):
        st.qkv_rope(Xh, Wd, Q, K, K)
    st.close()


def test_fused_append_e4m3_store(cuda):
    """Fused projection into an E4M3 store (R-22): the epilogue writes codes of the
    bf16-rounded K/V; they, the digest and the attention output are bit-identical to the
    unfused path (dense projection -> quantize kernel -> scatter), and O matches the e4m3
    oracle fed with the projection's bf16 values."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, hidden, theta, P = 2, 8, 2, 128, 512, 500000.0, 64
    kw = dict(page_size=P, num_pages=128, max_sessions=2, dtype="bf16", kv_format="e4m3",
              k_scale=1 / 16, v_scale=1 / 16)
    a = ssa.Store(L, hq, hkv, d, **kw)        # fused
    b = ssa.Store(L, hq, hkv, d, **kw)        # unfused reference path
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=128, kv_format="e4m3",
                             k_scale=1 / 16, v_scale=1 / 16)
    spec = streams.StreamSpec("peaked", seed=12)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 100)
    sa = a.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    sb = b.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    rs, _ = ref.session_create(100, Q, K, V, compute=False)
    W = [streams.gen_qkv_weight(6, l, (hq + 2 * hkv) * d, hidden) for l in range(L)]
    Wd = [to_dev(w, cuda) for w in W]
    pos, n = 100, 77
    X = [streams.gen_hidden(6, 0, 0, l, pos, n, hidden) for l in range(L)]
    ta, tb = a.append_begin(sa, n), b.append_begin(sb, n)
    Oa, Ob = [], []
    for l in range(L):
        o = torch.empty((n, hq, d), dtype=torch.bfloat16, device=cuda)
        a.append_layer_fused(sa, ta, l, to_dev(X[l], cuda), Wd[l], o, rope_theta=theta)
        Oa.append(o)
        Qd = torch.empty((n, hq, d), dtype=torch.bfloat16, device=cuda)
        Kd = torch.empty((n, hkv, d), dtype=torch.bfloat16, device=cuda)
        Vd = torch.empty_like(Kd)
        b.qkv_rope(to_dev(X[l], cuda), Wd[l], Qd, Kd, Vd, pos0=pos, rope_theta=theta)
        o2 = torch.empty_like(o)
        b.append_layer(sb, tb, l, Qd[None], Kd[None], Vd[None], o2[None])
        Ob.append(o2)
    a.append_commit(sa, ta)
    b.append_commit(sb, tb)
    torch.cuda.synchronize()
    for l in range(L):
        assert torch.equal(Oa[l].view(torch.int16), Ob[l].view(torch.int16)), l
        ka, va = a.read_kv(sa, l, 0, 100 + n)
        kb, vb = b.read_kv(sb, l, 0, 100 + n)
        assert np.array_equal(ka, kb) and np.array_equal(va, vb), l
    assert a.digest(sa) == b.digest(sb)
    Qr, Kr, Vr = _oracle_layers(X, W, hq, hkv, pos, theta)
    Oref, _ = ref.session_append(rs, Qr, Kr, Vr)
    mx, mn = errors(np.stack([from_dev(o) for o in Oa]), Oref)
    assert mx <= TOL["bf16"][0] and mn <= TOL["bf16"][1], (mx, mn)
    assert a.digest(sa) == ref.digest(rs)
    a.close()
    b.close()
