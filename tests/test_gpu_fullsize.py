"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

The oracle cannot recompute every output at 32k/128k context in seconds, so these
tests compare SAMPLED rows (chosen layers, tokens at tile edges, heads across KV
groups) element by element with the fp64 oracle (oracle.segment_rows, Eq.
query-attention P:150-155), plus properties that hold at any size: the page table
follows the lowest-free-id rule (R-9), appended K/V read back bit-exactly, and the
query leaves the session untouched (R-3).  Inputs come from streams.py only (the
GPU side generates them with gen_tensor_torch, the oracle side with gen_tensor_np;
the two are bit-identical, tests/test_gpu_parity.py::test_streams_torch_matches_numpy_on_gpu).
"""
import numpy as np
import pytest

import bench
import oracle
import streams
from helpers import from_dev, within

pytestmark = pytest.mark.gpu

CFG = bench.CFG
L, HQ, HKV, D, P = CFG["L"], CFG["hq"], CFG["hkv"], CFG["d"], CFG["P"]


def _np(spec, session, domain, layer, tensor, tok0, n, heads):
    return streams.gen_tensor_np(spec, session, domain, layer, tensor, tok0, n, heads, D, hkv=HKV)


def _cache(spec, layer, n, session=0):
    return (_np(spec, session, 0, layer, streams.TENSOR_K, 0, n, HKV),
            _np(spec, session, 0, layer, streams.TENSOR_V, 0, n, HKV))


def _check_rows(got_layer, spec, layer, kc, vc, domain, tok0, m, tokens, heads, session=0):
    """got_layer: GPU O of one layer [m][Hq][d] (bf16 bits)."""
    q = _np(spec, session, domain, layer, streams.TENSOR_Q, tok0, m, HQ)
    k = _np(spec, session, domain, layer, streams.TENSOR_K, tok0, m, HKV)
    v = _np(spec, session, domain, layer, streams.TENSOR_V, tok0, m, HKV)
    want, _ = oracle.segment_rows(kc, vc, q, k, v, HKV, oracle.default_scale(D), tokens, heads)
    got = got_layer[np.ix_(tokens, heads)]
    return within(got, want, "bf16")


def test_bench_config_full_size_sampled(cuda):
    """BJ.configs[1] exactly as bench.py runs it: one market session at n=32,512 over 32
    layers -> 256-token append (one call, all layers) -> 32-token query at n=32,768."""
    import torch
    import paper_2605_13784_b200 as ssa
    dev = cuda
    n0, m_app, q_len = CFG["n_ctx"] - CFG["m_append"], CFG["m_append"], CFG["q_len"]
    st = ssa.Store(L, HQ, HKV, D, page_size=P, num_pages=CFG["n_ctx"] // P + 16, max_sessions=4, dtype="bf16")
    spec = streams.StreamSpec("market", seed=2)
    sid = bench.build_session(st, torch, dev, spec, n0)
    Qa, Ka, Va = bench.gen_new(torch, dev, spec, 0, n0, m_app)
    Oa = torch.empty_like(Qa)
    Qq, Kq, Vq = bench.gen_new(torch, dev, spec, 1, 0, q_len)
    Oq = torch.empty_like(Qq)
    st.stats(reset=True)
    st.session_append(sid, Qa, Ka, Va, Oa)
    digest = st.digest(sid)
    st.session_query(sid, Qq, Kq, Vq, Oq)
    torch.cuda.synchronize()
    assert st.stats()["tc_launches"] >= 2            # both planes on the tcgen05 kernel
    assert st.digest(sid) == digest                  # query is state-neutral (R-3)
    assert st.page_table(sid) == list(range(CFG["n_ctx"] // P))   # lowest free id first (R-9)
    Oa_h, Oq_h = from_dev(Oa), from_dev(Oq)
    heads = [0, 5, 13, 31]
    for layer in (0, 31):
        kc, vc = _cache(spec, layer, n0)
        ok, e = _check_rows(Oa_h[layer], spec, layer, kc, vc, 0, n0, m_app, [0, 1, 31, 32, 127, 128, 200, 255],
                            heads)
        assert ok, ("append", layer, e)
        # the appended keys, read back from the pages, are the inputs bit for bit
        kb, vb = st.read_kv(sid, layer, n0, m_app)
        assert np.array_equal(kb, _np(spec, 0, 0, layer, streams.TENSOR_K, n0, m_app, HKV))
        assert np.array_equal(vb, _np(spec, 0, 0, layer, streams.TENSOR_V, n0, m_app, HKV))
        kc2 = np.concatenate([kc, kb]); vc2 = np.concatenate([vc, vb])
        ok, e = _check_rows(Oq_h[layer], spec, layer, kc2, vc2, 1, 0, q_len, list(range(q_len)), heads)
        assert ok, ("query", layer, e)
    st.close()


@pytest.mark.parametrize("q_len", [1, 32])
def test_split128k_full_size_sampled(cuda, q_len):
    """BJ.configs[4] at N=1 as bench.py's split_kv_128k leg: n=131,072 over 32 layers, one
    query call; every row is a many-way split-KV merge (A6)."""
    import torch
    import paper_2605_13784_b200 as ssa
    n = 131072
    st = ssa.Store(L, HQ, HKV, D, page_size=P, num_pages=n // P + 8, max_sessions=2, dtype="bf16")
    spec = streams.StreamSpec("market", seed=5)
    sid = bench.build_session_n(st, torch, cuda, spec, n)
    q, k, v = bench.gen_new(torch, cuda, spec, 1, 0, q_len)
    o = torch.empty_like(q)
    st.session_query(sid, q, k, v, o)
    torch.cuda.synchronize()
    layer = 31
    kc, vc = _cache(spec, layer, n)
    toks = list(range(q_len)) if q_len <= 4 else [0, 15, 31]
    ok, e = _check_rows(from_dev(o)[layer], spec, layer, kc, vc, 1, 0, q_len, toks, [0, 3, 17, 30])
    assert ok, e
    st.close()


def test_multitenant_full_size_sampled(cuda):
    """BJ.configs[2] as bench.py's multi_tenant leg: 48 sessions n=4096+256s, one batch_run
    over 32 layers with 24 appends x256, 24 queries x32 and 4 stateless x1024 prompts
    (snapshot semantics, R-7).  Samples an append, a query and a stateless item."""
    import torch
    import paper_2605_13784_b200 as ssa
    ns = [4096 + 256 * s for s in range(48)]
    num_pages = sum(-(-(n + 256) // P) for n in ns) + 64
    st = ssa.Store(L, HQ, HKV, D, page_size=P, num_pages=num_pages, max_sessions=64, dtype="bf16")
    spec = streams.StreamSpec("market", seed=3)
    sids = [bench.build_session_n(st, torch, cuda, spec, n, session=s) for s, n in enumerate(ns)]
    items, Qs, Ks, Vs, row, where = [], [], [], [], 0, {}
    for s, n in enumerate(ns):
        if s % 2 == 0:
            q, k, v = bench.gen_new(torch, cuda, spec, 0, n, 256, session=s)
            items.append((ssa.WORK_APPEND, sids[s], 256, row))
            where[s] = (row, 256)
            row += 256
        else:
            q, k, v = bench.gen_new(torch, cuda, spec, 1, 0, 32, session=s)
            items.append((ssa.WORK_QUERY, sids[s], 32, row))
            where[s] = (row, 32)
            row += 32
        Qs.append(q); Ks.append(k); Vs.append(v)
    for j in range(4):
        q, k, v = bench.gen_new(torch, cuda, spec, 100 + j, 0, 1024, session=60 + j)
        items.append((ssa.WORK_STATELESS, -1, 1024, row))
        where[100 + j] = (row, 1024)
        row += 1024
        Qs.append(q); Ks.append(k); Vs.append(v)
    Q, K, V = (torch.cat(x, dim=1).contiguous() for x in (Qs, Ks, Vs))
    O = torch.empty_like(Q)
    st.stats(reset=True)
    st.batch_run(items, Q, K, V, O)
    torch.cuda.synchronize()
    assert st.stats()["tc_launches"] == 1
    Oh = from_dev(O)
    layer = 7
    heads = [0, 9, 31]
    # a query item (odd s) and an append item (even s), each against its own session's cache
    for s, domain, tok0, toks in ((47, 1, 0, [0, 31]), (46, 0, ns[46], [0, 128, 255]), (1, 1, 0, [7])):
        r0, m = where[s]
        kc, vc = _cache(spec, layer, ns[s], session=s)
        ok, e = _check_rows(Oh[layer, r0:r0 + m], spec, layer, kc, vc, domain, tok0, m, toks, heads, session=s)
        assert ok, (s, e)
        info = st.info(sids[s])
        assert info["n_tokens"] == ns[s] + (256 if s % 2 == 0 else 0)
    # a stateless prompt: causal prefill over its own tokens only (R-16)
    r0, m = where[101]
    empty = np.zeros((0, HKV, D), dtype=np.uint16)
    ok, e = _check_rows(Oh[layer, r0:r0 + m], spec, layer, empty, empty, 101, 0, m, [0, 127, 128, 1023], heads,
                        session=61)
    assert ok, ("stateless", e)
    st.close()


@pytest.mark.parametrize("q_len", [1, 32])
def test_per_layer_query_full_size_sampled(cuda, q_len):
    """bench.py's per_layer leg: the 32-token (and 1-token) query at n=32,768 issued as 32
    single-layer calls (Alg. 2 L295 layer by layer) captured in one CUDA graph and replayed
    twice -- the launch configuration the bench times: group-barrier merge, 136 CTAs, 17
    key ranges per KV head merged in the kernel (R-11).  Sampled rows of layers 0, 13, 31
    against the fp64 oracle; the replay reproduces the eager call bit for bit."""
    import torch
    import paper_2605_13784_b200 as ssa
    n = CFG["n_ctx"]
    st = ssa.Store(L, HQ, HKV, D, page_size=P, num_pages=n // P + 16, max_sessions=2, dtype="bf16")
    spec = streams.StreamSpec("market", seed=2)
    sid = bench.build_session(st, torch, cuda, spec, n)
    q, k, v = bench.gen_new(torch, cuda, spec, 1, 0, q_len)
    o_eager = torch.empty_like(q)
    s = torch.cuda.Stream(device=cuda)

    def per_layer(o):
        for l in range(L):
            st.session_query(sid, q[l:l + 1], k[l:l + 1], v[l:l + 1], o[l:l + 1], layer=l, stream=s)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        per_layer(o_eager)
    s.synchronize()
    plan = st.last_plan()
    assert plan["gbar"] == 1 and plan["max_split"] > 1, plan
    o = torch.full_like(q, float("nan"))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        per_layer(o)
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(o.view(torch.int16), o_eager.view(torch.int16))
    oh = from_dev(o)
    toks = list(range(q_len)) if q_len <= 4 else [0, 1, 15, 31]
    for layer in (0, 13, 31):
        kc, vc = _cache(spec, layer, n)
        ok, e = _check_rows(oh[layer], spec, layer, kc, vc, 1, 0, q_len, toks, [0, 3, 4, 17, 30, 31])
        assert ok, (layer, e)
    st.close()


def test_fp8_bench_config_full_size_sampled(cuda):
    """bench.py's fp8_kv leg: BJ.configs[1] on an E4M3 KV store (k_scale = v_scale = 1/32,
    reading R-22): n=32,512 bulk-loaded -> 256-token append (all layers, one call) ->
    32-token query at n=32,768.  Sampled rows of layers 0 and 31 against the fp64 oracle
    over the dequantized stream (codes computed by the oracle's own e4m3_encode); the
    appended codes read back from the pages equal the oracle's codes bit for bit."""
    import torch
    import paper_2605_13784_b200 as ssa
    ks = vs = 1.0 / 32
    n0, m_app, q_len = CFG["n_ctx"] - CFG["m_append"], CFG["m_append"], CFG["q_len"]
    st = ssa.Store(L, HQ, HKV, D, page_size=P, num_pages=CFG["n_ctx"] // P + 16, max_sessions=4, dtype="bf16",
                   kv_format="e4m3", k_scale=ks, v_scale=vs)
    spec = streams.StreamSpec("market", seed=2)
    sid = bench.build_session(st, torch, cuda, spec, n0)
    Qa, Ka, Va = bench.gen_new(torch, cuda, spec, 0, n0, m_app)
    Oa = torch.empty_like(Qa)
    Qq, Kq, Vq = bench.gen_new(torch, cuda, spec, 1, 0, q_len)
    Oq = torch.empty_like(Qq)
    st.session_append(sid, Qa, Ka, Va, Oa)
    st.session_query(sid, Qq, Kq, Vq, Oq)
    torch.cuda.synchronize()
    Oa_h, Oq_h = from_dev(Oa), from_dev(Oq)

    def deq(bits, scale):
        return oracle.e4m3_decode(oracle.e4m3_encode(bits, scale)) * scale

    heads = [0, 5, 13, 31]
    for layer in (0, 31):
        kc_b, vc_b = _cache(spec, layer, n0)
        kc, vc = deq(kc_b, ks), deq(vc_b, vs)
        qa = _np(spec, 0, 0, layer, streams.TENSOR_Q, n0, m_app, HQ)
        ka = _np(spec, 0, 0, layer, streams.TENSOR_K, n0, m_app, HKV)
        va = _np(spec, 0, 0, layer, streams.TENSOR_V, n0, m_app, HKV)
        toks = [0, 1, 31, 32, 127, 128, 200, 255]
        want, _ = oracle.segment_rows(kc, vc, qa, deq(ka, ks), deq(va, vs), HKV, oracle.default_scale(D), toks,
                                      heads)
        ok, e = within(Oa_h[layer][np.ix_(toks, heads)], want, "bf16")
        assert ok, ("append", layer, e)
        kb, vb = st.read_kv(sid, layer, n0, m_app)   # E4M3 codes
        assert np.array_equal(kb, oracle.e4m3_encode(ka, ks))
        assert np.array_equal(vb, oracle.e4m3_encode(va, vs))
        kc2 = np.concatenate([kc, deq(ka, ks)])
        vc2 = np.concatenate([vc, deq(va, vs)])
        qq = _np(spec, 0, 1, layer, streams.TENSOR_Q, 0, q_len, HQ)
        kq = _np(spec, 0, 1, layer, streams.TENSOR_K, 0, q_len, HKV)
        vq = _np(spec, 0, 1, layer, streams.TENSOR_V, 0, q_len, HKV)
        want, _ = oracle.segment_rows(kc2, vc2, qq, deq(kq, ks), deq(vq, vs), HKV, oracle.default_scale(D),
                                      list(range(q_len)), heads)
        ok, e = within(Oq_h[layer][:, heads], want, "bf16")
        assert ok, ("query", layer, e)
    st.close()
