"""GPU parity of the CUDA path against the fp64 oracle.

Every test drives libssa through the C ABI (Python binding) and compares with
the oracle on the same seeded inputs (streams.py): KV append and page indexing
bit-exact; attention within the north-star tolerances (bf16 max-abs 2e-2 /
mean-abs 2e-3; fp32 1e-5).  Negative controls (fault injection) must FAIL.
"""
import numpy as np
import pytest

import oracle
import streams
from helpers import TOL, abs_bits, attention_bound, errors, f64, from_dev, gen_qkv, to_dev, within, within_bound

pytestmark = pytest.mark.gpu


def _ssa():
    import paper_2605_13784_b200 as ssa
    return ssa


def _rows_ref(ref, sid, layer, Q, K, V, tokens=None, heads=None):
    """Oracle rows of a new segment against the session's current cache (one layer)."""
    s = ref.sessions[sid]
    return oracle.segment_rows(s.k[layer][:s.n_tokens], s.v[layer][:s.n_tokens], Q, K, V, ref.hkv, ref.scale,
                               tokens, heads)[0]


def _bound(ref, sid, Q, K, V, O_ref, heads=None):
    """Derived per-element bound (helpers.attention_bound) of new-segment rows [L][m][H][d]
    against the session's current cache: the oracle's attention of the same rows with |V|."""
    s = ref.sessions[sid]
    A = np.stack([oracle.segment_rows(s.k[l][:s.n_tokens], abs_bits(s.v[l][:s.n_tokens]), Q[l], K[l],
                                      abs_bits(V[l]), ref.hkv, ref.scale, None, heads)[0]
                  for l in range(Q.shape[0])])
    return attention_bound(A, O_ref, s.n_tokens + Q.shape[1])


# --------------------------------------------------------------------------- config 1 (toy fp32)
@pytest.mark.parametrize("page_size", [16, 64])
def test_config1_toy_fp32(cuda, page_size):
    """BJ.configs[0]: 1 layer, 4 heads d=64 fp32; S=128, 8 appends of 64, |q|=16 query after each."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d = 1, 4, 4, 64
    spec = streams.StreamSpec("peaked", seed=1)
    st = ssa.Store(L, hq, hkv, d, page_size=page_size, num_pages=64, dtype="fp32")
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=page_size, num_pages=64, dtype="fp32")
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 128, "fp32")
    O = torch.empty(Q.shape, dtype=torch.float32, device=cuda)
    sid = st.session_create(to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    rsid, Oref = ref.session_create(128, Q, K, V)
    worst = errors(from_dev(O), Oref)
    tok = 128
    for i in range(8):
        Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, tok, 64, "fp32")
        O = torch.empty(Q.shape, dtype=torch.float32, device=cuda)
        st.session_append(sid, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
        Oref, _ = ref.session_append(rsid, Q, K, V)
        worst = max(worst, errors(from_dev(O), Oref))
        tok += 64
        Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1 + i, 0, 16, "fp32")
        Oq = torch.empty(Qq.shape, dtype=torch.float32, device=cuda)
        st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
        worst = max(worst, errors(from_dev(Oq), ref.session_query(rsid, Qq, Kq, Vq)))
        assert st.page_table(sid) == ref.page_table(rsid)
    assert worst[0] <= TOL["fp32"][0], worst
    assert st.digest(sid) == ref.digest(rsid)
    assert st.info(sid) == ref.info(rsid)


def test_ragged_appends_r0_padding_fp32(cuda):
    """Odd sizes: R0 of 100 tokens padded to a page boundary (hole masked), partial pages."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 4, 2, 32, 16
    spec = streams.StreamSpec("market", seed=7, iid_prefix=100)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=128, dtype="fp32")
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=128, dtype="fp32")
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 100, "fp32")
    O = torch.empty(Q.shape, device=cuda)
    sid = st.session_create(to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    rsid, Oref = ref.session_create(100, Q, K, V)
    worst = errors(from_dev(O), Oref)
    tok = 100
    for m in (37, 91, 1, 5, 64, 129):
        Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, tok, m, "fp32")
        O = torch.empty(Q.shape, device=cuda)
        st.session_append(sid, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
        Oref, _ = ref.session_append(rsid, Q, K, V)
        worst = max(worst, errors(from_dev(O), Oref))
        tok += m
        assert st.page_table(sid) == ref.page_table(rsid)
    Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, 3, "fp32")
    Oq = torch.empty(Qq.shape, device=cuda)
    st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
    worst = max(worst, errors(from_dev(Oq), ref.session_query(rsid, Qq, Kq, Vq)))
    assert worst[0] <= TOL["fp32"][0], worst
    for l in range(L):
        Kb, Vb = st.read_kv(sid, l, 0, tok)
        assert np.array_equal(Kb, ref.sessions[rsid].k[l]) and np.array_equal(Vb, ref.sessions[rsid].v[l])
    assert st.digest(sid) == ref.digest(rsid)


# --------------------------------------------------------------------------- Llama-shaped bf16
LL = dict(L=2, hq=32, hkv=8, d=128, P=64)


def _llama_session(cuda, spec, n0=512, appends=(256, 256), num_pages=256, backend=0):
    import torch
    ssa = _ssa()
    st = ssa.Store(LL["L"], LL["hq"], LL["hkv"], LL["d"], page_size=LL["P"], num_pages=num_pages, dtype="bf16")
    if backend:
        st.set_option(ssa.OPT_ATTN_BACKEND, backend)
    ref = oracle.OracleStore(LL["L"], LL["hq"], LL["hkv"], LL["d"], page_size=LL["P"], num_pages=num_pages)
    Q, K, V = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 0, 0, n0)
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    rsid, _ = ref.session_create(n0, Q, K, V, compute=False)
    tok = n0
    outs = []
    for m in appends:
        Q, K, V = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 0, tok, m)
        O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
        Ref_rows = np.stack([_rows_ref(ref, rsid, l, Q[l], K[l], V[l], heads=[0, 9, 31]) for l in range(LL["L"])])
        bound = _bound(ref, rsid, Q, K, V, Ref_rows, heads=[0, 9, 31])
        st.session_append(sid, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
        ref.session_append(rsid, Q, K, V, compute=False)
        outs.append((from_dev(O)[:, :, [0, 9, 31]], Ref_rows, bound))
        tok += m
    return st, ref, sid, rsid, tok, outs


@pytest.mark.parametrize("stream_name", ["peaked", "market", "flat"])
@pytest.mark.parametrize("backend", [2, 1])
def test_llama_append_and_query_bf16(cuda, stream_name, backend):
    """backend 2 = tcgen05 kernel, 1 = SIMT kernel; both against the oracle."""
    import torch
    spec = streams.StreamSpec(stream_name, seed=2)
    st, ref, sid, rsid, tok, outs = _llama_session(cuda, spec, backend=backend)
    assert (st.stats()["tc_launches"] > 0) == (backend == 2)
    for got, want, bound in outs:
        ok, e = within(got, want, "bf16")
        assert ok, ("append", e)
        if backend == 2:   # the tcgen05 kernel's derived per-element bound (bf16 P, bf16 O)
            ok, r = within_bound(got, want, bound)
            assert ok, ("append bound", r)
    Qq, Kq, Vq = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 1, 0, 32)
    Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
    want = ref.session_query(rsid, Qq, Kq, Vq)
    ok, e = within(from_dev(Oq), want, "bf16")
    assert ok, ("query", e)
    if backend == 2:
        ok, r = within_bound(from_dev(Oq), want, _bound(ref, rsid, Qq, Kq, Vq, want))
        assert ok, ("query bound", r)
    assert st.page_table(sid) == ref.page_table(rsid)
    assert st.digest(sid) == ref.digest(rsid)


@pytest.mark.parametrize("backend", [0, 2])
@pytest.mark.parametrize("nq", [1, 4, 32, 33, 100])
def test_query_lengths_bf16(cuda, nq, backend):
    """|q| = 1 .. 100 (several q tiles, ragged tail); auto (0) and forced tcgen05 (2)."""
    import torch
    spec = streams.StreamSpec("peaked", seed=3)
    st, ref, sid, rsid, tok, _ = _llama_session(cuda, spec, n0=700, appends=(300,), backend=backend)
    Qq, Kq, Vq = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 1, 0, nq)
    Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
    ok, e = within(from_dev(Oq), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
    assert ok, e


def test_needle_probes_at_boundaries(cuda):
    """Needles at slot 0, P-1, P, split boundaries and n-1 must be retrieved (O = v_j)."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 1, 32, 8, 128, 64
    n = 2048
    for pos in (0, 63, 64, 127, 128, 1000, n - 1):
        spec = streams.StreamSpec("needle", seed=4, needles=(pos,))
        st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
        ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=64)
        Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
        sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
        rsid, _ = ref.session_create(n, Q, K, V, compute=False)
        Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, 32)
        Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
        st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
        want = ref.session_query(rsid, Qq, Kq, Vq)
        ok, e = within(from_dev(Oq), want, "bf16")
        assert ok, (pos, e)
        # the oracle itself returns v_needle (weight ~1): the probe is live
        vn = f64(V[0, pos])
        assert np.abs(want[0] - np.repeat(vn, hq // hkv, axis=0)[None]).max() < 1e-6
        st.close()


@pytest.mark.parametrize("backend", [1, 2])
@pytest.mark.parametrize("fault", [1, 2])
def test_negative_controls_fail(cuda, fault, backend):
    """A kernel that drops the last key tile / misses its own key must fail the tolerance."""
    import torch
    ssa = _ssa()
    spec = streams.StreamSpec("peaked", seed=5)
    st, ref, sid, rsid, tok, _ = _llama_session(cuda, spec, n0=512, appends=(128,), backend=backend)
    st.set_option(ssa.OPT_FAULT_INJECT, fault)
    Qq, Kq, Vq = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 1, 0, 32)
    Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
    ok, e = within(from_dev(Oq), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
    assert not ok, ("negative control passed", fault, e)


# --------------------------------------------------------------------------- flash queries / batch
def test_flash_query_batch(cuda):
    import torch
    spec = streams.StreamSpec("market", seed=6)
    st, ref, sid, rsid, tok, _ = _llama_session(cuda, spec, n0=640, appends=(256,))
    dg = st.digest(sid)
    lens = [32, 7, 32, 19, 1, 32, 50]
    qs = [gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], streams.FLASH_DOMAIN + i, 0, m)
          for i, m in enumerate(lens)]
    for layer in (0, 1):
        Q = np.concatenate([q[0][layer:layer + 1] for q in qs], axis=1)
        K = np.concatenate([q[1][layer:layer + 1] for q in qs], axis=1)
        V = np.concatenate([q[2][layer:layer + 1] for q in qs], axis=1)
        O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
        st.flash_query_batch(sid, lens, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O, layer=layer)
        want = ref.flash_query_batch(rsid, [(q[0][layer], q[1][layer], q[2][layer]) for q in qs], layer)
        ok, e = within(from_dev(O)[0], np.concatenate(want), "bf16")
        assert ok, e
    assert st.digest(sid) == dg     # state neutrality


@pytest.mark.parametrize("per_layer", [False, True])
def test_batch_run_snapshot(cuda, per_layer):
    """One launch: appends + queries of several sessions + stateless prompts (R-7); per_layer:
    the same batch as one single-layer launch per layer (cluster-merge plans over mixed
    SHARED / SPLIT pair-items), the appends committed by the last layer's call."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    spec = streams.StreamSpec("market", seed=8)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=512)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=512)
    sids = []
    for s, n in enumerate([300, 1024, 777]):
        Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n, session=s)
        sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
        rsid, _ = ref.session_create(n, Q, K, V, compute=False)
        assert sid == rsid
        sids.append((sid, n))
    # items: append s0, query s0 (same batch -> sees old state), query s1, append s2, stateless
    plan = [("append", 0, 64), ("query", 0, 32), ("query", 1, 32), ("append", 2, 100), ("stateless", -1, 200)]
    Qs, Ks, Vs, items, ref_items, row = [], [], [], [], [], 0
    for i, (kind, s, m) in enumerate(plan):
        if kind == "append":
            Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, sids[s][1], m, session=s)
        else:
            Q, K, V = gen_qkv(spec, L, hq, hkv, d, 50 + i, 0, m, session=max(s, 0))
        Qs.append(Q); Ks.append(K); Vs.append(V)
        items.append(({"append": ssa.WORK_APPEND, "query": ssa.WORK_QUERY, "stateless": ssa.WORK_STATELESS}[kind],
                      s, m, row))
        ref_items.append(dict(kind=kind, session=s, Q=Q, K=K, V=V))
        row += m
    Q, K, V = (np.concatenate(x, axis=1) for x in (Qs, Ks, Vs))
    O = torch.full(Q.shape, float("nan"), dtype=torch.bfloat16, device=cuda)
    Qd, Kd, Vd = to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda)
    if per_layer:
        for l in range(L):
            st.batch_run(items, Qd[l:l + 1], Kd[l:l + 1], Vd[l:l + 1], O[l:l + 1], layer=l)
            assert st.last_plan()["cm_C"] >= 1
    else:
        st.batch_run(items, Qd, Kd, Vd, O)
    want = np.concatenate(ref.batch_run(ref_items), axis=1)
    ok, e = within(from_dev(O), want, "bf16")
    assert ok, e
    for sid, _ in sids:
        assert st.info(sid) == ref.info(sid)
        assert st.page_table(sid) == ref.page_table(sid)
        assert st.digest(sid) == ref.digest(sid)


def test_per_layer_append_equals_all_layer(cuda):
    """Per-layer tickets (single-layer launches, cluster-merge plans) vs one all-layer append:
    identical pages and digest (bit-exact), both within tolerance and within the derived
    per-element bound of the oracle (the split structures differ, so the fp32 sums do too)."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 3, 8, 2, 128, 64
    spec = streams.StreamSpec("peaked", seed=9)
    a = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
    b = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=64)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 200)
    sa = a.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    sb = b.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    rs, _ = ref.session_create(200, Q, K, V, compute=False)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 200, 90)
    Oref = np.stack([_rows_ref(ref, rs, l, Q[l], K[l], V[l]) for l in range(L)])
    bound = _bound(ref, rs, Q, K, V, Oref)
    ref.session_append(rs, Q, K, V, compute=False)
    Oa = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    a.session_append(sa, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), Oa)
    t = b.append_begin(sb, 90)
    Ob = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    for l in range(L):
        b.append_layer(sb, t, l, to_dev(Q[l:l + 1], cuda), to_dev(K[l:l + 1], cuda), to_dev(V[l:l + 1], cuda), Ob[l:l + 1])
    with pytest.raises(ssa.SsaError):
        b.append_layer(sb, t, 0, to_dev(Q[:1], cuda), to_dev(K[:1], cuda), to_dev(V[:1], cuda), Ob[:1])
    b.append_commit(sb, t)
    for O in (Oa, Ob):
        ok, e = within(from_dev(O), Oref, "bf16")
        assert ok, e
        ok, r = within_bound(from_dev(O), Oref, bound)
        assert ok, r
    assert a.digest(sa) == b.digest(sb) and a.info(sa) == b.info(sb)


# --------------------------------------------------------------------------- store contract
def test_host_pointers_equal_device_pointers(cuda):
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 8, 2, 128, 64
    spec = streams.StreamSpec("peaked", seed=10)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 300)
    a = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
    b = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
    Od = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    sa = a.session_create(to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), Od)
    Oh = np.zeros(Q.shape, dtype=np.uint16)
    sb = b.session_create(Q, K, V, Oh)        # pageable host numpy buffers
    torch.cuda.synchronize()
    assert np.array_equal(from_dev(Od), Oh)
    Qp = torch.from_numpy(Q.view(np.int16)).pin_memory()
    Op = torch.zeros(Q.shape, dtype=torch.int16).pin_memory()
    Q2, K2, V2 = gen_qkv(spec, L, hq, hkv, d, 1, 0, 32)
    O2d = torch.empty(Q2.shape, dtype=torch.bfloat16, device=cuda)
    a.session_query(sa, to_dev(Q2, cuda), to_dev(K2, cuda), to_dev(V2, cuda), O2d)
    O2h = torch.zeros(Q2.shape, dtype=torch.int16).pin_memory()
    b.session_query(sb, torch.from_numpy(Q2.view(np.int16)).pin_memory(), torch.from_numpy(K2.view(np.int16)).pin_memory(),
                    torch.from_numpy(V2.view(np.int16)).pin_memory(), O2h)
    torch.cuda.synchronize()
    assert np.array_equal(from_dev(O2d), O2h.numpy().view(np.uint16))
    assert b.stats()["h2d_bytes"] > 0
    del Qp, Op


def test_pipelined_host_query_all_layers(cuda):
    """All-layer query with host buffers runs in layer chunks whose copies overlap the
    kernels (copy streams + events); O is complete once the CALL's stream is synchronized.
    Pinned and pageable buffers; results vs the oracle; state unchanged."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 8, 8, 2, 128, 64
    spec = streams.StreamSpec("peaked", seed=12)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=256)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=256, dtype="bf16")
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 700)
    sid = st.session_create(to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda),
                            torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda))
    rsid, _ = ref.session_create(700, Q, K, V)
    before = (st.digest(sid), st.info(sid))
    s = torch.cuda.Stream(device=cuda)
    for i, pinned in enumerate((True, False, True)):
        Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1 + i, 0, 32)
        if pinned:
            hq_, hk_, hv_ = (torch.from_numpy(x.view(np.int16)).pin_memory() for x in (Qq, Kq, Vq))
            Oh = torch.full(Qq.shape, -1, dtype=torch.int16).pin_memory()
        else:
            hq_, hk_, hv_ = (np.ascontiguousarray(x) for x in (Qq, Kq, Vq))
            Oh = np.full(Qq.shape, 0xFFFF, dtype=np.uint16)
        st.session_query(sid, hq_, hk_, hv_, Oh, stream=s)
        s.synchronize()
        got = Oh.numpy().view(np.uint16) if pinned else Oh
        mx, mn = errors(got, ref.session_query(rsid, Qq, Kq, Vq))
        assert mx <= TOL["bf16"][0] and mn <= TOL["bf16"][1], (i, mx, mn)
    assert (st.digest(sid), st.info(sid)) == before
    st.close()


def test_errors_leave_no_state_change(cuda):
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 1, 4, 4, 64, 16
    spec = streams.StreamSpec("flat", seed=11)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=6, max_sessions=2, dtype="fp32")
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 64, "fp32")
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    before = (st.info(sid), st.page_table(sid), st.occupancy(), st.digest(sid))
    Q2, K2, V2 = gen_qkv(spec, L, hq, hkv, d, 0, 64, 40, "fp32")
    with pytest.raises(ssa.SsaError) as e:
        st.session_append(sid, None, to_dev(K2, cuda), to_dev(V2, cuda))
    assert e.value.name == "SSA_ERR_POOL_EXHAUSTED"
    with pytest.raises(ssa.SsaError) as e:
        st.session_append(77, None, to_dev(K2, cuda), to_dev(V2, cuda))
    assert e.value.name == "SSA_ERR_UNKNOWN_SESSION"
    with pytest.raises(ssa.SsaError) as e:
        st.session_query(sid, to_dev(Q2, cuda), to_dev(K2, cuda), to_dev(V2, cuda), None)
    assert e.value.name == "SSA_ERR_INVALID_ARG"
    assert (st.info(sid), st.page_table(sid), st.occupancy(), st.digest(sid)) == before
    s2 = st.session_create(None, to_dev(K[:, :16], cuda), to_dev(V[:, :16], cuda))
    with pytest.raises(ssa.SsaError) as e:
        st.session_create(None, to_dev(K[:, :16], cuda), to_dev(V[:, :16], cuda))
    assert e.value.name in ("SSA_ERR_SESSION_LIMIT", "SSA_ERR_POOL_EXHAUSTED")
    st.session_destroy(s2)


def test_query_cost_invariance(cuda):
    """Rows computed per query = |q| * Hq * L at every context size."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    spec = streams.StreamSpec("market", seed=12)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=512)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 512)
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    tok = 512
    Qq, Kq, Vq = (to_dev(x, cuda) for x in gen_qkv(spec, L, hq, hkv, d, 1, 0, 30))
    Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    for step in range(5):
        Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, tok, 1000)
        st.load_kv(sid, to_dev(K, cuda), to_dev(V, cuda))
        tok += 1000
        d0 = st.info(sid)
        st.stats(reset=True)
        st.session_query(sid, Qq, Kq, Vq, Oq)
        s = st.stats()
        assert s["query_rows"] == 30 * hq * L and s["tokens_appended"] == 0 and s["pages_reserved"] == 0
        assert st.info(sid) == d0


def test_streams_torch_matches_numpy_on_gpu(cuda):
    import torch
    for name in streams.STREAMS:
        spec = streams.StreamSpec(name, seed=13, needles=(3, 70))
        a = streams.gen_tensor_np(spec, 2, 0, 1, streams.TENSOR_K, 50, 40, 8, 128, hkv=8)
        b = streams.gen_tensor_torch(spec, 2, 0, 1, streams.TENSOR_K, 50, 40, 8, 128, hkv=8, device=cuda)
        assert np.array_equal(a, from_dev(b))


def test_flash_query_batch_64x32(cuda):
    """BJ.configs[3] shape at small context: 64 registered 32-token questions in one launch
    (pairs share the cached K/V tiles, private own-token tails)."""
    import torch
    spec = streams.StreamSpec("market", seed=14)
    st, ref, sid, rsid, tok, _ = _llama_session(cuda, spec, n0=1000, appends=(200,), num_pages=128)
    k, m = 64, 32
    layer = 1
    qs = [gen_qkv(spec, 1, LL["hq"], LL["hkv"], LL["d"], streams.FLASH_DOMAIN + i, 0, m, layers=[layer])
          for i in range(k)]
    Q = np.concatenate([q[0] for q in qs], axis=1)
    K = np.concatenate([q[1] for q in qs], axis=1)
    V = np.concatenate([q[2] for q in qs], axis=1)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    st.stats(reset=True)
    st.flash_query_batch(sid, [m] * k, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O, layer=layer)
    assert st.stats()["tc_launches"] == 1
    got = from_dev(O)[0]
    for i in (0, 1, 17, 62, 63):
        want = ref.flash_query_batch(rsid, [(qs[i][0][0], qs[i][1][0], qs[i][2][0])], layer)[0]
        ok, e = within(got[i * m:(i + 1) * m], want, "bf16")
        assert ok, (i, e)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("nq", [1, 32])
def test_sharded_partials_merge(cuda, world, nq):
    """A9 on one GPU: `world` stores hold contiguous shards (R-12); rank partials + merge == unsharded."""
    import torch
    from paper_2605_13784_b200.sharding import shard_range
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    n = 3001
    spec = streams.StreamSpec("market", seed=15)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=64)
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, nq)
    rows = L * nq
    chunk = rows * hq * (d + 1)
    parts = torch.empty((world, chunk), dtype=torch.float32, device=cuda)
    stores = []
    for r in range(world):
        lo, hi = shard_range(n, r, world)
        st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
        sid = st.session_create(None, to_dev(K[:, lo:hi], cuda), to_dev(V[:, lo:hi], cuda))
        st.sharded_partial(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), parts[r],
                           include_tail=(r == world - 1))
        stores.append(st)
    O = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    stores[0].merge_rank_partials(world, rows, parts, O)
    ok, e = within(from_dev(O), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
    assert ok, e


def test_sharded_query_nccl_world1(cuda):
    """The NCCL path end to end (world = 1 on a single GPU): partial -> ncclAllGather -> merge."""
    import torch
    ssa = _ssa()
    spec = streams.StreamSpec("peaked", seed=16)
    st, ref, sid, rsid, tok, _ = _llama_session(cuda, spec, n0=900, appends=(100,))
    st.comm_init(0, 1, ssa.Store.comm_unique_id())
    Qq, Kq, Vq = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 1, 0, 32)
    O = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    st.sharded_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), O)
    ok, e = within(from_dev(O), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
    assert ok, e
    st.comm_destroy()


# --------------------------------------------------------------------------- cluster merge (CM)
def _needle_positions(n):
    # slot 0, page edges, key-tile edges, unit / cluster boundaries of the single-layer plans, n-1
    return (0, 63, 64, 127, 128, n // 2 - 1, n // 2, n // 4, 3 * n // 4, n - 1)


@pytest.mark.parametrize("stream_name", ["market", "needle"])
@pytest.mark.parametrize("nq", [1, 32])
def test_cluster_merge_per_layer_query(cuda, nq, stream_name):
    """Single-layer query calls (the per-layer form of Alg. 2 L295 a model issues) under every
    cluster-merge plan: split-KV ranges merged through DSMEM inside the cluster and, when a
    group spans several clusters, by the last arriving CTA (R-11).  C = 0 planner's choice,
    -1 LPT plan regrouped (C = 1).  Needles sit at page, tile and split boundaries; every call
    runs twice (the merge tickets must be back at zero)."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    n = 12000
    kw = dict(needles=_needle_positions(n)) if stream_name == "needle" else {}
    spec = streams.StreamSpec(stream_name, seed=61, **kw)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=n // P + 8)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=n // P + 8)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, nq)
    want = ref.session_query(rsid, Qq, Kq, Vq)
    bound = _bound(ref, rsid, Qq, Kq, Vq, want)
    Qd, Kd, Vd = to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda)
    for C, merge in ((0, 1), (-1, 1), (1, 1), (1, 0), (2, 1), (2, 0), (4, 1), (4, 0), (6, 1), (8, 1), (0, 2), (0, 4)):   # 2: merge kernel, 4: group barrier
        st.set_option(ssa.OPT_CLUSTER, C)
        st.set_option(ssa.OPT_CM_MERGE, merge)   # separate merge kernel / last-arriving CTA
        splits = []
        for rep in range(2):
            O = torch.full(Qd.shape, float("nan"), dtype=torch.bfloat16, device=cuda)
            for l in range(L):
                st.session_query(sid, Qd[l:l + 1], Kd[l:l + 1], Vd[l:l + 1], O[l:l + 1], layer=l)
                plan = st.last_plan()
                assert plan["cm_C"] == (C if C > 0 else plan["cm_C"]) and plan["cm_C"] >= 1, (C, plan)
                splits.append(plan["max_split"])
            ok, e = within(from_dev(O), want, "bf16")
            assert ok, (C, rep, e)
            ok, r = within_bound(from_dev(O), want, bound)
            assert ok, (C, rep, "bound", r)
        if C in (1, 2) or merge >= 2:
            assert max(splits) > 1, (C, splits)     # the cross-cluster (last-arriver) merge ran
        if merge >= 2:
            assert plan["gbar"] == 1, plan          # group-barrier plan (merged in the kernel / by gm_merge)
    assert st.stats()["cm_launches"] >= 2 * L * 12


@pytest.mark.parametrize("C", [1, 4, 8, "gbar", "gbar_barrier"])
def test_cluster_merge_empty_ranges(cuda, C):
    """A short cache (2 key tiles per head) under a forced cluster size (or the group-barrier
    merge): most CTAs of the plan get empty key ranges (lse = -inf, skipped by the merge)."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 1, 32, 8, 128, 16
    spec = streams.StreamSpec("peaked", seed=62)
    for n in (1, 150, 300):
        st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
        if C == "gbar":
            st.set_option(ssa.OPT_CM_MERGE, 2)   # group plan, merge kernel (the default)
        elif C == "gbar_barrier":
            st.set_option(ssa.OPT_CM_MERGE, 4)   # group plan, in-kernel group barrier
        else:
            st.set_option(ssa.OPT_CLUSTER, C)
        ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=64)
        Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
        sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
        rsid, _ = ref.session_create(n, Q, K, V, compute=False)
        for nq in (1, 7, 32):
            Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, nq)
            O = torch.full((1, nq, hq, d), float("nan"), dtype=torch.bfloat16, device=cuda)
            st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), O, layer=0)
            ok, e = within(from_dev(O), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
            assert ok, (n, nq, e)
        st.close()


@pytest.mark.parametrize("C", [0, 1, 2, 4, 8, "gbar", "gbar_barrier"])
def test_cluster_merge_per_layer_append(cuda, C):
    """Per-layer data-plane steps (Alg. 1: append_begin / append_layer per layer / commit)
    under the cluster-merge plans: SHARED CTA pairs (two q tiles over the same keys), the key
    range split over the cluster; a ragged append and a second one on top."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    spec = streams.StreamSpec("market", seed=63)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=256)
    if C == "gbar":
        st.set_option(ssa.OPT_CM_MERGE, 3)   # group plan on the data plane too (merge kernel)
    elif C == "gbar_barrier":
        st.set_option(ssa.OPT_CM_MERGE, 5)   # group plan on the data plane, in-kernel group barrier
    else:
        st.set_option(ssa.OPT_CLUSTER, C)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=256)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 3000)
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    rsid, _ = ref.session_create(3000, Q, K, V, compute=False)
    tok = 3000
    for m in (256, 100):
        Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, tok, m)
        Qd, Kd, Vd = to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda)
        O = torch.full(Qd.shape, float("nan"), dtype=torch.bfloat16, device=cuda)
        t = st.append_begin(sid, m)
        for l in range(L):
            st.append_layer(sid, t, l, Qd[l:l + 1], Kd[l:l + 1], Vd[l:l + 1], O[l:l + 1])
        st.append_commit(sid, t)
        if C in ("gbar", "gbar_barrier"):
            assert st.last_plan()["gbar"] == 1, st.last_plan()
        Oref, _ = ref.session_append(rsid, Q, K, V)
        ok, e = within(from_dev(O), Oref, "bf16")
        assert ok, (m, e)
        tok += m
    assert st.page_table(sid) == ref.page_table(rsid)
    assert st.digest(sid) == ref.digest(rsid)


def test_per_layer_append_cuda_graph(cuda):
    """ssa_append_layer captured into a CUDA graph (scatter + attention per layer, cached work
    lists): replayed inside a ticket of the same session state it reproduces the eager step
    bit for bit, including the pages."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    spec = streams.StreamSpec("market", seed=64)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=128)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 2000)
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    Qa, Ka, Va = (to_dev(x, cuda) for x in gen_qkv(spec, L, hq, hkv, d, 0, 2000, 256))
    want = torch.empty(Qa.shape, dtype=torch.bfloat16, device=cuda)
    t = st.append_begin(sid, 256)
    for l in range(L):
        st.append_layer(sid, t, l, Qa[l:l + 1], Ka[l:l + 1], Va[l:l + 1], want[l:l + 1])
    st.append_commit(sid, t)
    torch.cuda.synchronize()
    want_digest = st.digest(sid)
    want_pages = st.page_table(sid)
    uploads = st.stats()["plan_uploads"]
    for rep in range(2):
        st.session_truncate(sid, 2000)
        t = st.append_begin(sid, 256)
        O = torch.zeros_like(want)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            s = torch.cuda.current_stream()
            for l in range(L):
                st.append_layer(sid, t, l, Qa[l:l + 1], Ka[l:l + 1], Va[l:l + 1], O[l:l + 1], stream=s)
        st.append_commit(sid, t)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(O.view(torch.int16), want.view(torch.int16))
        assert st.page_table(sid) == want_pages and st.digest(sid) == want_digest
    assert st.stats()["plan_uploads"] == uploads     # captured calls reused the cached work lists
    st.close()


def test_cross_stream_ordering_page_reuse(cuda):
    """A query on stream A, then (no host sync) truncation and a new session on stream B that
    reuses the released pages: the store orders B's writes after A's reads."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 8, 32, 8, 128, 64
    spec = streams.StreamSpec("market", seed=65)
    n = 16384
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=n // P + 8)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=n // P + 8)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
    sid = st.session_create(None, to_dev(K[:, :512], cuda), to_dev(V[:, :512], cuda))   # R0 = 512 tokens
    st.load_kv(sid, to_dev(K[:, 512:], cuda), to_dev(V[:, 512:], cuda))
    rsid, _ = ref.session_create(512, Q[:, :512], K[:, :512], V[:, :512], compute=False)
    ref.session_append(rsid, Q[:, 512:], K[:, 512:], V[:, 512:], compute=False)
    Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, 32)
    want = ref.session_query(rsid, Qq, Kq, Vq)
    Qd, Kd, Vd = to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda)
    K2 = torch.full((L, n - 1000, hkv, d), 7.0, dtype=torch.bfloat16, device=cuda)
    torch.cuda.synchronize()
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    O = torch.empty(Qd.shape, dtype=torch.bfloat16, device=cuda)
    for _ in range(3):
        st.session_query(sid, Qd, Kd, Vd, O, stream=sa)
    st.session_truncate(sid, 1000)
    sid2 = st.session_create(None, K2, K2, stream=sb)
    torch.cuda.synchronize()
    ok, e = within(from_dev(O), want, "bf16")
    assert ok, e
    st.close()


def test_batch_mixed_and_needles(cuda):
    """A varlen batch (an append, a query and a stateless prompt) in one cluster-merge launch, also on the needle
    stream (boundary keys must be retrieved exactly)."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 1, 32, 8, 128, 64
    for stream_name in ("market", "needle"):
        spec = streams.StreamSpec(stream_name, seed=22)
        st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=256, dtype="bf16")
        ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=256)
        sids, rsids = [], []
        for s, n in enumerate((1000, 2500)):
            Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n, session=s)
            sids.append(st.session_create(None, to_dev(K, cuda), to_dev(V, cuda)))
            rsids.append(ref.session_create(n, Q, K, V, compute=False)[0])
        parts, items, ritems, row = [], [], [], 0
        for s, (kind, m, dom, tok0) in enumerate(((ssa.WORK_APPEND, 256, 0, 1000), (ssa.WORK_QUERY, 32, 1, 0))):
            Q, K, V = gen_qkv(spec, L, hq, hkv, d, dom, tok0, m, session=s)
            parts.append((Q, K, V))
            items.append((kind, sids[s], m, row))
            ritems.append({"kind": "append" if kind == ssa.WORK_APPEND else "query", "session": rsids[s],
                           "Q": Q, "K": K, "V": V})
            row += m
        Q, K, V = gen_qkv(spec, L, hq, hkv, d, 9, 0, 300, session=7)
        parts.append((Q, K, V))
        items.append((ssa.WORK_STATELESS, -1, 300, row))
        ritems.append({"kind": "stateless", "session": -1, "Q": Q, "K": K, "V": V})
        Qa, Ka, Va = (np.concatenate([p[i] for p in parts], axis=1) for i in range(3))
        O = torch.empty(Qa.shape, dtype=torch.bfloat16, device=cuda)
        st.stats(reset=True)
        st.batch_run(items, to_dev(Qa, cuda), to_dev(Ka, cuda), to_dev(Va, cuda), O)
        assert st.stats()["cm_launches"] == 1
        got = from_dev(O)
        want = ref.batch_run(ritems)
        for (kind, sid, m, row), w in zip(items, want):
            ok, e = within(got[:, row:row + m], w, "bf16")
            assert ok, (stream_name, kind, e)


@pytest.mark.parametrize("page_size", [16, 64])
def test_retention_eviction_parity(cuda, page_size):
    """Region-1 FIFO eviction (Alg. 1) through the retention guard and explicit
    evict_oldest: attention over the retained keys, page tables (evicted pages leave, hole at
    the head of the first R1 page) and digests (original positions) match the oracle."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d = 2, 32, 8, 128
    spec = streams.StreamSpec("peaked", seed=31)
    st = ssa.Store(L, hq, hkv, d, page_size=page_size, num_pages=8192 // page_size, dtype="bf16")
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=page_size, num_pages=8192 // page_size)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 100)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    sid = st.session_create(to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    rsid, _ = ref.session_create(100, Q, K, V)
    st.set_retention(sid, 700)
    ref.set_retention(rsid, 700)
    tok = 100
    for m in (300, 256, 200, 37, 129):
        Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, tok, m)
        O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
        st.session_append(sid, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
        Oref, _ = ref.session_append(rsid, Q, K, V)
        ok, e = within(from_dev(O), Oref, "bf16")
        assert ok, (m, e)
        assert st.page_table(sid) == ref.page_table(rsid), m
        assert st.info(sid) == ref.info(rsid), m
        tok += m
    assert st.info(sid)["n_evicted"] > 0
    st.evict_oldest(sid, 51)
    ref.evict_oldest(rsid, 51)
    assert st.page_table(sid) == ref.page_table(rsid)
    assert st.digest(sid) == ref.digest(rsid)
    Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, 33)
    Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
    ok, e = within(from_dev(Oq), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
    assert ok, ("query", e)
    n_keep = ref.info(rsid)["n_tokens"]
    Kb, Vb = st.read_kv(sid, 1, 0, n_keep)
    assert np.array_equal(Kb, ref.sessions[rsid].k[1][:n_keep]) and np.array_equal(Vb, ref.sessions[rsid].v[1][:n_keep])
    assert st.occupancy() == ref.occupancy()
    # an append larger than the evictable Region 1 fails without state change
    digest = st.digest(sid)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, tok, 800)
    with pytest.raises(ssa.SsaError):
        st.session_append(sid, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda))
    assert st.digest(sid) == digest and st.page_table(sid) == ref.page_table(rsid)


def test_alias_prefix_parity(cuda):
    """Metadata-only prefix aliasing: whole pages shared by reference, the page
    holding token m-1 copied; independent appends on donor and alias, deferred free."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    spec = streams.StreamSpec("market", seed=32)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=256, dtype="bf16")
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=256)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 100)
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    rsid, _ = ref.session_create(100, Q, K, V, compute=False)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 100, 900)
    st.session_append(sid, None, to_dev(K, cuda), to_dev(V, cuda))
    ref.session_append(rsid, Q, K, V, compute=False)
    tids = {}
    for m in (1000, 640, 57):
        tids[m] = (st.alias_prefix(sid, m), ref.alias_prefix(rsid, m))
        g, r = tids[m]
        assert st.page_table(g) == ref.page_table(r), m
        assert st.digest(g) == ref.digest(r), m
        assert st.info(g) == ref.info(r), m
        assert st.occupancy() == ref.occupancy(), m
    # independent continuations: target 1000 and the donor
    g, r = tids[1000]
    for who, (gs, rs), dom in (("alias", (g, r), 5), ("donor", (sid, rsid), 6)):
        Q, K, V = gen_qkv(spec, L, hq, hkv, d, dom, 0, 77)
        O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
        st.session_append(gs, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
        Oref, _ = ref.session_append(rs, Q, K, V)
        ok, e = within(from_dev(O), Oref, "bf16")
        assert ok, (who, e)
        assert st.page_table(gs) == ref.page_table(rs)
    assert st.digest(tids[640][0]) == ref.digest(tids[640][1])   # untouched by the others' appends
    # deferred free: destroying the donor keeps the shared pages alive for the aliases
    st.session_destroy(sid)
    ref.session_destroy(rsid)
    assert st.occupancy() == ref.occupancy()
    g, r = tids[640]
    Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, 32)
    Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    st.session_query(g, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
    ok, e = within(from_dev(Oq), ref.session_query(r, Qq, Kq, Vq), "bf16")
    assert ok, e
    # a new session reuses freed pages only; the aliases still read their own data
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 300, session=9)
    n2 = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    r2, _ = ref.session_create(300, Q, K, V, compute=False)
    assert st.page_table(n2) == ref.page_table(r2)
    assert st.digest(g) == ref.digest(r)


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
@pytest.mark.parametrize("rows,vocab,stride", [(1, 128256, 128256), (7, 128256, 128256), (64, 128256, 128264),
                                               (5, 1, 1), (3, 33, 35), (9, 4097, 4097), (4, 1001, 1003)])
def test_greedy_sample_parity(cuda, dtype, rows, vocab, stride):
    """On-device greedy sampling: argmax ids bit-exact (ties toward the lowest id,
    including ties planted across the kernel's split boundaries), logit gap bit-exact (one fp32
    subtraction on both sides), NaN ignored, strided / unaligned rows."""
    import torch
    ssa = _ssa()
    st = ssa.Store(1, 4, 4, 64, page_size=16, num_pages=4, dtype="fp32")
    rng = np.random.default_rng(rows * 1000 + vocab)
    x = rng.standard_normal((rows, stride)).astype(np.float32) * 4
    for r in range(rows):
        top = float(x[r, :vocab].max()) + 1.0
        for j in rng.choice(vocab, size=min(vocab, 1 + r % 3), replace=False):   # planted ties
            x[r, j] = top
        if vocab > 8 and r % 2:
            x[r, rng.integers(0, vocab)] = np.nan
    if vocab > 4096:
        x[0, [4095, 4096]] = x[0, :vocab].max() + 2.0                              # tie across a split edge
    if dtype == "bf16":
        xb = oracle_bits = (x.view(np.uint32) >> 16).astype(np.uint16)              # truncate to bf16 bits
        dev = torch.from_numpy(xb.view(np.int16)).view(torch.bfloat16).to(cuda)
        want_ids, want_gap = oracle.greedy_sample(oracle_bits[:, :vocab])
    else:
        dev = torch.from_numpy(x).to(cuda)
        want_ids, want_gap = oracle.greedy_sample(x[:, :vocab])
    logits = dev[:, :vocab]
    ids = torch.empty(rows, dtype=torch.int32, device=cuda)
    gap = torch.empty(rows, dtype=torch.float32, device=cuda)
    draft = torch.from_numpy(want_ids.copy()).to(cuda)
    if rows > 2:
        draft[rows // 2] += 1                                                        # first mismatch
    n_acc = torch.zeros(1, dtype=torch.int32, device=cuda)
    for _ in range(2):                                                               # counters reset between calls
        st.greedy_sample(logits, ids, gap, draft=draft, out_n_accept=n_acc)
        got_ids, got_gap = ids.cpu().numpy(), gap.cpu().numpy()
        assert np.array_equal(got_ids, want_ids)
        assert np.array_equal(got_gap.view(np.uint32), want_gap.view(np.uint32))
        assert int(n_acc.item()) == (rows // 2 if rows > 2 else rows)
    st.close()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("nq", [1, 32])
def test_sharded_peer_push_virtual_ranks(cuda, world, nq):
    """A9 over peer memory, `world` virtual ranks on one GPU: each rank's combine epilogue stores
    its partial into every rank's gathered buffer and releases an epoch flag; every rank's merge
    acquires the flags and merges, then acks.  Two rounds on one stream exercise the epoch
    protocol and the alternating buffer halves."""
    import torch
    from paper_2605_13784_b200.sharding import chunk_floats, shard_range
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    n = 3001
    spec = streams.StreamSpec("market", seed=41)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=64)
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    ch = chunk_floats(nq, L, hq, d)
    bufs = [torch.zeros(2 * world * ch, dtype=torch.float32, device=cuda) for _ in range(world)]
    flags = [torch.zeros(2 * world, dtype=torch.int32, device=cuda) for _ in range(world)]
    stores, sids = [], []
    for r in range(world):
        lo, hi = shard_range(n, r, world)
        st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
        sids.append(st.session_create(None, to_dev(K[:, lo:hi], cuda), to_dev(V[:, lo:hi], cuda)))
        st.comm_attach_peers(r, world, [b.data_ptr() for b in bufs], [f.data_ptr() for f in flags],
                             2 * world * ch * 4)
        stores.append(st)
    for rnd in range(2):
        Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1 + rnd, 0, nq)
        want = ref.session_query(rsid, Qq, Kq, Vq)
        for r in range(world):
            stores[r].sharded_push(sids[r], to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda))
        for r in range(world):
            O = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
            stores[r].sharded_merge(O)
            ok, e = within(from_dev(O), want, "bf16")
            assert ok, (rnd, r, e)
        torch.cuda.synchronize()
        assert all(int(f[q].item()) == rnd + 1 for f in flags for q in range(2 * world))   # ready + ack
    with pytest.raises(ssa.SsaError, match="STATE"):   # a merge needs a pushed epoch
        stores[0].sharded_merge(torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_peer_push_pipelined_rounds(cuda, world):
    """The peer-memory exchange under back-to-back per-layer rounds with no cross-rank
    synchronisation: `world` virtual ranks on one GPU, each on its own stream, run 64 rounds of
    push + merge (single-layer sharded queries, cycling layers and query inputs) before the one
    host sync at the end.  Without the per-half acks a fast rank would overwrite a half a slow
    rank's merge is still reading.  Every round of every rank must equal the oracle."""
    import torch
    from paper_2605_13784_b200.sharding import chunk_floats, shard_range
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    n, nq, rounds = 3001, 32, 64
    spec = streams.StreamSpec("market", seed=43)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=64)
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    inputs = [gen_qkv(spec, L, hq, hkv, d, 1 + i, 0, nq) for i in range(4)]
    wants = [ref.session_query(rsid, *x) for x in inputs]
    dev_in = [tuple(to_dev(a, cuda) for a in x) for x in inputs]
    ch = chunk_floats(nq, 1, hq, d)
    bufs = [torch.zeros(2 * world * ch, dtype=torch.float32, device=cuda) for _ in range(world)]
    flags = [torch.zeros(2 * world, dtype=torch.int32, device=cuda) for _ in range(world)]
    stores, sids, streams_ = [], [], []
    for r in range(world):
        lo, hi = shard_range(n, r, world)
        st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
        sids.append(st.session_create(None, to_dev(K[:, lo:hi], cuda), to_dev(V[:, lo:hi], cuda)))
        st.comm_attach_peers(r, world, [b.data_ptr() for b in bufs], [f.data_ptr() for f in flags],
                             2 * world * ch * 4)
        stores.append(st)
        streams_.append(torch.cuda.Stream())
    torch.cuda.synchronize()
    outs = [[torch.empty((1, nq, hq, d), dtype=torch.bfloat16, device=cuda) for _ in range(rounds)]
            for _ in range(world)]
    for rnd in range(rounds):
        i, l = rnd % 4, rnd % L
        Qd, Kd, Vd = dev_in[i]
        # rank order rotates so no rank is always first
        for r in [(rnd + j) % world for j in range(world)]:
            s = streams_[r]
            stores[r].sharded_push(sids[r], Qd[l:l + 1], Kd[l:l + 1], Vd[l:l + 1], layer=l, stream=s)
            stores[r].sharded_merge(outs[r][rnd], layer=l, stream=s)
    torch.cuda.synchronize()
    for rnd in range(rounds):
        i, l = rnd % 4, rnd % L
        for r in range(world):
            ok, e = within(from_dev(outs[r][rnd]), wants[i][l:l + 1], "bf16")
            assert ok, (rnd, r, e)
            assert torch.equal(outs[r][rnd].view(torch.int16), outs[0][rnd].view(torch.int16))
    for st in stores:
        st.close()


def test_sharded_symmetric_memory_world1(cuda):
    """The torch-symmetric-memory attach path (world 1 on one GPU): push + merge == oracle."""
    import os
    import tempfile
    import torch
    import torch.distributed as dist
    from paper_2605_13784_b200.sharding import attach_symmetric, chunk_floats
    try:
        import torch.distributed._symmetric_memory  # noqa: F401
    except Exception as exc:   # pragma: no cover
        pytest.skip(f"no symmetric memory: {exc}")
    ssa = _ssa()
    spec = streams.StreamSpec("peaked", seed=42)
    st, ref, sid, rsid, tok, _ = _llama_session(cuda, spec, n0=900, appends=(100,))
    init_here = not dist.is_initialized()
    if init_here:
        f = tempfile.NamedTemporaryFile(delete=False)
        dist.init_process_group("nccl", init_method=f"file://{f.name}", rank=0, world_size=1,
                                device_id=torch.device(cuda))
    try:
        try:
            keep = attach_symmetric(st, chunk_floats(32, LL["L"], LL["hq"], LL["d"]))
        except Exception as exc:
            pytest.skip(f"symmetric memory unavailable here: {type(exc).__name__}: {exc}")
        Qq, Kq, Vq = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 1, 0, 32)
        O = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
        st.sharded_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), O)
        ok, e = within(from_dev(O), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
        assert ok, e
        del keep
    finally:
        if init_here:
            dist.destroy_process_group()


def test_sharded_peer_push_two_processes(cuda):
    """A9 over peer memory across two processes on one GPU: the gathered buffers and flags are
    CUDA-IPC mapped into both processes (torch.multiprocessing), so the pushes, the system-scope
    flag release and the acquiring merge cross a process boundary as they do across GPUs."""
    import torch
    import torch.multiprocessing as mp
    import p2p_worker
    from paper_2605_13784_b200.sharding import chunk_floats
    L, hq, hkv, d, P, n, world = 2, 32, 8, 128, 64, 3001, 2
    spec = streams.StreamSpec("market", seed=44)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
    qs = [gen_qkv(spec, L, hq, hkv, d, 1 + r, 0, 32) for r in range(3)]
    ch = chunk_floats(32, L, hq, d)
    bufs = [torch.zeros(2 * world * ch, dtype=torch.float32, device=cuda) for _ in range(world)]
    flags = [torch.zeros(2 * world, dtype=torch.int32, device=cuda) for _ in range(world)]
    ctx = mp.get_context("spawn")
    out_q = ctx.Queue()
    procs = [ctx.Process(target=p2p_worker.run,
                         args=(r, world, bufs, flags, K, V, [q[0] for q in qs], [q[1] for q in qs],
                               [q[2] for q in qs], out_q, n, (L, hq, hkv, d, P)))
             for r in range(world)]
    for p in procs:
        p.start()
    results = dict(out_q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=64)
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    for i, (Qq, Kq, Vq) in enumerate(qs):
        want = ref.session_query(rsid, Qq, Kq, Vq)
        for r in range(world):
            ok, e = within(results[r][i], want, "bf16")
            assert ok, (r, i, e)
    assert all(int(f[q].item()) == 3 for f in flags for q in range(2 * world))   # ready + ack


@pytest.mark.parametrize("kv", [None, "e4m3"])
def test_query_plane_cuda_graph_capture(cuda, kv):
    """Query-plane calls captured into a CUDA graph (work lists in the store's graph arena)
    replay bit-identically to direct calls, repeatedly; per-layer and all-layer forms.  An
    append cannot be captured (it changes the store at call time)."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d = LL["L"], LL["hq"], LL["hkv"], LL["d"]
    kw = dict(kv_format="e4m3", k_scale=1 / 16, v_scale=1 / 32) if kv else {}
    st = ssa.Store(L, hq, hkv, d, page_size=64, num_pages=128, dtype="bf16", **kw)
    spec = streams.StreamSpec("market", seed=42)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 3000)
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    Qq, Kq, Vq = (to_dev(x, cuda) for x in gen_qkv(spec, L, hq, hkv, d, 1, 0, 32))
    want = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    for l in range(L):                     # direct calls (also the warm-up: scratch sized)
        st.session_query(sid, Qq[l:l + 1], Kq[l:l + 1], Vq[l:l + 1], want[l:l + 1], layer=l)
    want_all = torch.empty_like(want)
    st.session_query(sid, Qq, Kq, Vq, want_all)
    Qbig, Kbig, Vbig = (to_dev(x, cuda) for x in gen_qkv(spec, L, hq, hkv, d, 2, 0, 2048))
    Obig = torch.empty(Qbig.shape, dtype=torch.bfloat16, device=cuda)
    torch.cuda.synchronize()
    O = torch.zeros_like(want)
    O_all = torch.zeros_like(want)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        s = torch.cuda.current_stream()
        for l in range(L):
            st.session_query(sid, Qq[l:l + 1], Kq[l:l + 1], Vq[l:l + 1], O[l:l + 1], layer=l, stream=s)
        st.session_query(sid, Qq, Kq, Vq, O_all, stream=s)
    for _ in range(2):
        O.zero_()
        O_all.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(O.view(torch.int16), want.view(torch.int16))
        assert torch.equal(O_all.view(torch.int16), want_all.view(torch.int16))
    Qa, Ka, Va = (to_dev(x, cuda) for x in gen_qkv(spec, L, hq, hkv, d, 0, 3000, 64))
    occ = st.occupancy()
    with pytest.raises(ssa.SsaError):
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2):
            st.session_append(sid, Qa, Ka, Va, torch.empty_like(Qa), stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert st.info(sid)["n_tokens"] == 3000 and st.occupancy() == occ
    # call shapes never run eagerly take arena space (cached shapes do not); the arena is
    # exhausted by enough of them and recycled on request
    exhausted = False
    for nq in range(1, 2049):
        args = (Qbig[0:1, :nq], Kbig[0:1, :nq], Vbig[0:1, :nq], Obig[0:1, :nq])
        try:
            g3 = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g3):
                st.session_query(sid, *args, layer=0, stream=torch.cuda.current_stream())
        except ssa.SsaError as exc:
            torch.cuda.synchronize()
            if "arena" in str(exc):
                exhausted = True
                break
            assert "warm up" in str(exc), exc
            st.session_query(sid, *args, layer=0)   # sizes scratch for this shape, then capture again
            torch.cuda.synchronize()
    assert exhausted
    torch.cuda.synchronize()
    st.set_option(ssa.OPT_GRAPH_ARENA_RESET, 1)
    g4 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g4):
        st.session_query(sid, Qq, Kq, Vq, O_all, stream=torch.cuda.current_stream())
    O_all.zero_()
    g4.replay()
    torch.cuda.synchronize()
    assert torch.equal(O_all.view(torch.int16), want_all.view(torch.int16))
    st.close()


def test_borrowed_pool_from_torch(cuda):
    """ssa_store_config.pool_ptr: the KV pool lives in a torch allocation.  The
    store writes its pages there (the K half of the buffer holds the session's keys at their
    page slots), parity as with a store-owned pool; an undersized or host buffer is rejected."""
    import torch
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    nb = ssa.Store.pool_bytes(L, hq, hkv, d, P, 64)
    buf = torch.zeros(nb, dtype=torch.uint8, device=cuda)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64, pool=buf)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=64)
    spec = streams.StreamSpec("market", seed=66)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 1000)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    sid = st.session_create(to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    rsid, Oref = ref.session_create(1000, Q, K, V)
    ok, e = within(from_dev(O), Oref, "bf16")
    assert ok, e
    torch.cuda.synchronize()
    # token 0 of layer 0, kv head 0 sits at page_table[0], slot 0: [L][pages][Hkv][P][d] bf16
    pg = st.page_table(sid)[0]
    k_pool = buf[: nb // 2].view(torch.int16).view(L, 64, hkv, P, d)
    assert np.array_equal(k_pool[0, pg, 0, 0].cpu().numpy().view(np.uint16), K[0, 0, 0])
    Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, 32)
    Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
    ok, e = within(from_dev(Oq), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
    assert ok, e
    assert st.digest(sid) == ref.digest(rsid)
    st.close()
    with pytest.raises(ssa.SsaError, match="INVALID_ARG"):
        ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64, pool=torch.zeros(nb // 2, dtype=torch.uint8, device=cuda))
    with pytest.raises(ssa.SsaError, match="INVALID_ARG"):
        ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64, pool=torch.zeros(nb, dtype=torch.uint8))


def test_two_devices_in_one_process():
    """Two stores on two devices of one process (per-device kernel attributes, per-device
    plans): each runs its own session, and a sharded query over NCCL (world 2, one process,
    ncclCommInitRank per device) equals the oracle.  Needs 2 GPUs."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    ssa = _ssa()
    L, hq, hkv, d, P = 2, 32, 8, 128, 64
    spec = streams.StreamSpec("market", seed=45)
    n = 2000
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=64)
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, 32)
    want = ref.session_query(rsid, Qq, Kq, Vq)
    for dev in (0, 1):
        cd = torch.device("cuda", dev)
        st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64, device=dev)
        sid = st.session_create(None, to_dev(K, cd), to_dev(V, cd))
        O = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cd)
        st.session_query(sid, to_dev(Qq, cd), to_dev(Kq, cd), to_dev(Vq, cd), O)
        ok, e = within(from_dev(O), want, "bf16")
        assert ok, (dev, e)
        for l in range(L):   # single-layer calls: cluster-merge launches on this device
            Ol = torch.empty((1, 32, hq, d), dtype=torch.bfloat16, device=cd)
            st.session_query(sid, to_dev(Qq[l:l + 1], cd), to_dev(Kq[l:l + 1], cd), to_dev(Vq[l:l + 1], cd), Ol,
                             layer=l)
            ok, e = within(from_dev(Ol), want[l:l + 1], "bf16")
            assert ok, (dev, l, e)
        st.close()
