"""GPU parity of the FP8 (E4M3) KV-cache variant (reading R-22)
against the fp64 oracle with ``kv_format="e4m3"``.

The stored codes (pages, read back through the C ABI) and digests must equal the
oracle's quantizer bit for bit; attention over the dequantized cache must meet the
bf16 tolerances (max-abs 2e-2, mean-abs 2e-3) -- the oracle attends over
code * scale, so the quantization error itself is not in the comparison.
"""
import numpy as np
import pytest

import oracle
import streams
from helpers import f64, from_dev, gen_qkv, to_dev, within

pytestmark = pytest.mark.gpu

LL = dict(L=2, hq=32, hkv=8, d=128)
KS, VS = 1 / 16, 1 / 32


def _ssa():
    import paper_2605_13784_b200 as ssa
    return ssa


def _pair(L, P, num_pages, ks=KS, vs=VS):
    ssa = _ssa()
    st = ssa.Store(L, LL["hq"], LL["hkv"], LL["d"], page_size=P, num_pages=num_pages, dtype="bf16",
                   kv_format="e4m3", k_scale=ks, v_scale=vs)
    ref = oracle.OracleStore(L, LL["hq"], LL["hkv"], LL["d"], page_size=P, num_pages=num_pages,
                             kv_format="e4m3", k_scale=ks, v_scale=vs)
    return st, ref


def _session(cuda, spec, P=64, n0=512, appends=(256,), L=2, num_pages=512, ks=KS, vs=VS):
    import torch
    st, ref = _pair(L, P, num_pages, ks, vs)
    Q, K, V = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 0, 0, n0)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    sid = st.session_create(to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    rsid, want = ref.session_create(n0, Q, K, V)
    outs = [(from_dev(O), want)]
    tok = n0
    for m in appends:
        Q, K, V = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 0, tok, m)
        O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
        st.session_append(sid, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
        want, _ = ref.session_append(rsid, Q, K, V)
        outs.append((from_dev(O), want))
        tok += m
    return st, ref, sid, rsid, tok, outs


def test_fp8_codes_bit_exact_incl_ties_and_saturation(cuda):
    """Quantization on the GPU (fp32 quotient, RNE, satfinite) == the oracle's, every element."""
    L, P, n = 2, 16, 300
    st, ref = _pair(L, P, 64, ks=0.0123, vs=1 / 64)
    rng = np.random.default_rng(21)
    table = oracle.e4m3_decode(np.arange(127, dtype=np.uint8))
    mids = (table[1:] + table[:-1]) / 2
    K = rng.standard_normal((L, n, LL["hkv"], LL["d"])) * np.exp2(rng.uniform(-8, 4, (L, n, LL["hkv"], LL["d"])))
    V = rng.standard_normal((L, n, LL["hkv"], LL["d"])) * 2
    flatV = V.reshape(-1)
    flatV[: 2 * len(mids)] = np.concatenate([mids, -mids]) / 64      # exact ties after x / (1/64)
    flatV[2 * len(mids): 2 * len(mids) + 6] = [500.0 / 64, 448.0 / 64, 464.0 / 64, -470.0 / 64, 1e-9, -1e-9]
    K, V = streams.bf16_bits_np(K), streams.bf16_bits_np(V)
    Q = streams.bf16_bits_np(rng.standard_normal((L, n, LL["hq"], LL["d"])) * 3)
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    for l in range(L):
        gk, gv = st.read_kv(sid, l, 0, n)
        assert np.array_equal(gk, oracle.e4m3_encode(K[l], 0.0123))
        assert np.array_equal(gv, oracle.e4m3_encode(V[l], 1 / 64))
    assert st.page_table(sid) == ref.page_table(rsid)
    assert st.digest(sid) == ref.digest(rsid)
    assert st.pool_bytes(L, LL["hq"], LL["hkv"], LL["d"], P, 64, kv_format="e4m3") == 2 * L * 64 * LL["hkv"] * P * LL["d"]
    st.close()


@pytest.mark.parametrize("P", [16, 64, 128])
@pytest.mark.parametrize("stream_name", ["peaked", "market"])
def test_fp8_create_append_query_parity(cuda, P, stream_name):
    import torch
    spec = streams.StreamSpec(stream_name, seed=31)
    st, ref, sid, rsid, tok, outs = _session(cuda, spec, P=P, n0=700, appends=(256, 37))
    assert st.stats()["tc_launches"] > 0
    for got, want in outs:
        ok, e = within(got, want, "bf16")
        assert ok, ("data plane", e)
    for nq in (1, 4, 32, 33, 100):
        Qq, Kq, Vq = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 1, 0, nq)
        Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
        st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
        ok, e = within(from_dev(Oq), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
        assert ok, ("query", nq, e)
    assert st.page_table(sid) == ref.page_table(rsid)
    assert st.digest(sid) == ref.digest(rsid)
    st.close()


def test_fp8_differs_from_bf16_cache(cuda):
    """The E4M3 path really reads codes: its output matches the e4m3 oracle and not the bf16 one
    better than the tolerance would allow by chance (the two oracles differ by > 2e-2 here)."""
    import torch
    spec = streams.StreamSpec("peaked", seed=32)
    st, ref, sid, rsid, tok, _ = _session(cuda, spec, n0=1024, appends=(), L=1, ks=1 / 2, vs=1 / 2)
    ref16 = oracle.OracleStore(1, LL["hq"], LL["hkv"], LL["d"], page_size=64, num_pages=512)
    Q, K, V = gen_qkv(spec, 1, LL["hq"], LL["hkv"], LL["d"], 0, 0, 1024)
    r16, _ = ref16.session_create(1024, Q, K, V, compute=False)
    Qq, Kq, Vq = gen_qkv(spec, 1, LL["hq"], LL["hkv"], LL["d"], 1, 0, 32)
    Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
    w8 = ref.session_query(rsid, Qq, Kq, Vq)
    w16 = ref16.session_query(r16, Qq, Kq, Vq)
    assert np.abs(w8 - w16).max() > 2e-2
    ok, e = within(from_dev(Oq), w8, "bf16")
    assert ok, e
    ok16, _ = within(from_dev(Oq), w16, "bf16")
    assert not ok16
    st.close()


def test_fp8_needles_at_boundaries(cuda):
    import torch
    n = 2048
    for pos in (0, 63, 64, 127, 128, 1000, n - 1):
        spec = streams.StreamSpec("needle", seed=33, needles=(pos,))
        st, ref = _pair(1, 64, 64, ks=1 / 16, vs=1 / 32)    # needle keys 19 * 16 = 304 < 448
        Q, K, V = gen_qkv(spec, 1, LL["hq"], LL["hkv"], LL["d"], 0, 0, n)
        sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
        rsid, _ = ref.session_create(n, Q, K, V, compute=False)
        Qq, Kq, Vq = gen_qkv(spec, 1, LL["hq"], LL["hkv"], LL["d"], 1, 0, 32)
        Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
        st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
        want = ref.session_query(rsid, Qq, Kq, Vq)
        ok, e = within(from_dev(Oq), want, "bf16")
        assert ok, (pos, e)
        vn = oracle.e4m3_decode(oracle.e4m3_encode(V[0, pos], 1 / 32)) / 32   # the needle's dequantized v
        assert np.abs(want[0] - np.repeat(vn, LL["hq"] // LL["hkv"], axis=0)[None]).max() < 1e-6
        st.close()


def test_fp8_flash_batch_and_varlen_batch(cuda):
    import torch
    ssa = _ssa()
    spec = streams.StreamSpec("market", seed=34)
    st, ref, sid, rsid, tok, _ = _session(cuda, spec, n0=640, appends=(256,))
    dg = st.digest(sid)
    lens = [32, 7, 32, 19, 1, 32, 50]
    qs = [gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], streams.FLASH_DOMAIN + i, 0, m)
          for i, m in enumerate(lens)]
    layer = 1
    Q = np.concatenate([q[0][layer:layer + 1] for q in qs], axis=1)
    K = np.concatenate([q[1][layer:layer + 1] for q in qs], axis=1)
    V = np.concatenate([q[2][layer:layer + 1] for q in qs], axis=1)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    st.flash_query_batch(sid, lens, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O, layer=layer)
    want = ref.flash_query_batch(rsid, [(q[0][layer], q[1][layer], q[2][layer]) for q in qs], layer)
    ok, e = within(from_dev(O)[0], np.concatenate(want), "bf16")
    assert ok, e
    assert st.digest(sid) == dg
    # varlen batch: append + query of the same session (snapshot, R-7), a second session, a stateless prompt
    Q2, K2, V2 = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 0, 0, 300, session=1)
    sid2 = st.session_create(None, to_dev(K2, cuda), to_dev(V2, cuda))
    rsid2, _ = ref.session_create(300, Q2, K2, V2, compute=False)
    plan = [("append", sid, rsid, 64), ("query", sid, rsid, 32), ("query", sid2, rsid2, 20), ("stateless", -1, -1, 150)]
    Qs, Ks, Vs, items, ref_items, row = [], [], [], [], [], 0
    for i, (kind, s, rs, m) in enumerate(plan):
        if kind == "append":
            q, k, v = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 0, tok, m)
        else:
            q, k, v = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 60 + i, 0, m)
        Qs.append(q); Ks.append(k); Vs.append(v)
        items.append(({"append": ssa.WORK_APPEND, "query": ssa.WORK_QUERY, "stateless": ssa.WORK_STATELESS}[kind],
                      s, m, row))
        ref_items.append(dict(kind=kind, session=rs, Q=q, K=k, V=v))
        row += m
    Q, K, V = (np.concatenate(x, axis=1) for x in (Qs, Ks, Vs))
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    st.batch_run(items, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    want = np.concatenate(ref.batch_run(ref_items), axis=1)
    ok, e = within(from_dev(O), want, "bf16")
    assert ok, e
    for s, rs in ((sid, rsid), (sid2, rsid2)):
        assert st.info(s) == ref.info(rs)
        assert st.page_table(s) == ref.page_table(rs)
        assert st.digest(s) == ref.digest(rs)
    st.close()


@pytest.mark.parametrize("fault", [1, 2])
def test_fp8_negative_controls_fail(cuda, fault):
    import torch
    ssa = _ssa()
    spec = streams.StreamSpec("peaked", seed=35)
    st, ref, sid, rsid, tok, _ = _session(cuda, spec, n0=512, appends=(128,))
    st.set_option(ssa.OPT_FAULT_INJECT, fault)
    Qq, Kq, Vq = gen_qkv(spec, LL["L"], LL["hq"], LL["hkv"], LL["d"], 1, 0, 32)
    Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
    ok, e = within(from_dev(Oq), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
    assert not ok, e
    st.close()


def test_fp8_long_session_split_kv_sampled(cuda):
    """16k cached tokens (split-KV query plane, many tiles per unit); sampled heads."""
    import torch
    spec = streams.StreamSpec("market", seed=36)
    L, n = 1, 16384
    st, ref = _pair(L, 64, 300)
    Q, K, V = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 0, 0, n)
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    for nq in (1, 32):
        Qq, Kq, Vq = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 1, 0, nq)
        Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
        st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
        heads = [0, 5, 13, 31]
        want = ref.session_query(rsid, Qq, Kq, Vq, heads=heads)
        ok, e = within(from_dev(Oq)[:, :, heads], want, "bf16")
        assert ok, (nq, e)
    st.close()


def test_fp8_unsupported_paths_fail_loudly(cuda):
    ssa = _ssa()
    st, _ = _pair(1, 64, 64)
    st.set_option(ssa.OPT_ATTN_BACKEND, 1)      # SIMT kernels have no E4M3 path
    spec = streams.StreamSpec("peaked", seed=37)
    Q, K, V = gen_qkv(spec, 1, LL["hq"], LL["hkv"], LL["d"], 0, 0, 64)
    import torch
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(ssa.SsaError) as ei:
        st.session_create(to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    assert ei.value.name == "SSA_ERR_UNSUPPORTED"
    st.close()
    with pytest.raises(ssa.SsaError):
        ssa.Store(1, 32, 8, 64, kv_format="e4m3", k_scale=1.0, v_scale=1.0)      # head_dim 64
    with pytest.raises(ssa.SsaError):
        ssa.Store(1, 32, 8, 128, kv_format="e4m3", k_scale=0.0, v_scale=1.0)     # scale must be > 0


def test_fp8_retention_alias_and_read_back(cuda):
    """Store paths that move pages on an E4M3 pool (1-byte elements): retention eviction,
    prefix aliasing with the one-page copy, destroy / reuse -- codes, page tables and digests
    bit-exact, attention within tolerance."""
    import torch
    spec = streams.StreamSpec("peaked", seed=38)
    L, P = 2, 64
    st, ref = _pair(L, P, 128)
    Q, K, V = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 0, 0, 100)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    sid = st.session_create(to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    rsid, _ = ref.session_create(100, Q, K, V)
    st.set_retention(sid, 700)
    ref.set_retention(rsid, 700)
    tok = 100
    for m in (300, 256, 200, 37):
        Q, K, V = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 0, tok, m)
        O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
        st.session_append(sid, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
        Oref, _ = ref.session_append(rsid, Q, K, V)
        ok, e = within(from_dev(O), Oref, "bf16")
        assert ok, (m, e)
        assert st.page_table(sid) == ref.page_table(rsid) and st.info(sid) == ref.info(rsid)
        tok += m
    assert st.info(sid)["n_evicted"] > 0
    n_keep = ref.info(rsid)["n_tokens"]
    Kb, Vb = st.read_kv(sid, 1, 0, n_keep)
    assert np.array_equal(Kb, ref.sessions[rsid].k[1][:n_keep]) and np.array_equal(Vb, ref.sessions[rsid].v[1][:n_keep])
    # aliasing on a fresh donor (no eviction): shared pages + copied partial page
    Q, K, V = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 0, 0, 500, session=1)
    d0 = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    r0, _ = ref.session_create(500, Q, K, V, compute=False)
    g, r = st.alias_prefix(d0, 333), ref.alias_prefix(r0, 333)
    assert st.page_table(g) == ref.page_table(r) and st.digest(g) == ref.digest(r)
    Q, K, V = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 7, 0, 45, session=1)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    st.session_append(g, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    Oref, _ = ref.session_append(r, Q, K, V)
    ok, e = within(from_dev(O), Oref, "bf16")
    assert ok, e
    st.session_destroy(d0)
    ref.session_destroy(r0)
    assert st.digest(g) == ref.digest(r) and st.occupancy() == ref.occupancy()
    st.close()


def test_fp8_per_layer_and_host_buffers(cuda):
    """Per-layer tickets == one all-layer append; pageable host buffers (the pipelined
    all-layer path) == device buffers, on an E4M3 store."""
    import torch
    spec = streams.StreamSpec("market", seed=39)
    L = 3
    a, ref = _pair(L, 64, 64)
    b, _ = _pair(L, 64, 64)
    Q, K, V = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 0, 0, 200)
    sa = a.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    sb = b.session_create(None, K, V)                   # host inputs
    rs, _ = ref.session_create(200, Q, K, V, compute=False)
    Q, K, V = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 0, 200, 90)
    Oref, _ = ref.session_append(rs, Q, K, V)
    Oa = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    a.session_append(sa, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), Oa)
    t = b.append_begin(sb, 90)
    Ob = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    for l in range(L):
        b.append_layer(sb, t, l, to_dev(Q[l:l + 1], cuda), to_dev(K[l:l + 1], cuda), to_dev(V[l:l + 1], cuda),
                       Ob[l:l + 1])
    b.append_commit(sb, t)
    for O in (Oa, Ob):     # per-layer launches use cluster-merge plans: not bit-identical to all-layer
        ok, e = within(from_dev(O), Oref, "bf16")
        assert ok, e
    assert a.digest(sa) == b.digest(sb)
    Qq, Kq, Vq = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 1, 0, 32)
    Od = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    a.session_query(sa, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Od)
    Oh = np.zeros(Qq.shape, dtype=np.uint16)
    b.session_query(sb, Qq, Kq, Vq, Oh)
    torch.cuda.synchronize()
    assert np.array_equal(from_dev(Od), Oh)
    a.close()
    b.close()


@pytest.mark.parametrize("world", [2, 3])
def test_fp8_sharded_partials_merge(cuda, world):
    """A9 on E4M3 shards: rank partials + log-sum-exp merge == the unsharded e4m3 oracle."""
    import torch
    from paper_2605_13784_b200.sharding import shard_range
    spec = streams.StreamSpec("market", seed=40)
    L, n, nq = 2, 3001, 32
    Q, K, V = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 0, 0, n)
    _, ref = _pair(L, 64, 64)
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    Qq, Kq, Vq = gen_qkv(spec, L, LL["hq"], LL["hkv"], LL["d"], 1, 0, nq)
    rows = L * nq
    parts = torch.empty((world, rows * LL["hq"] * (LL["d"] + 1)), dtype=torch.float32, device=cuda)
    stores = []
    for r in range(world):
        lo, hi = shard_range(n, r, world)
        st, _ = _pair(L, 64, 64)
        sid = st.session_create(None, to_dev(K[:, lo:hi], cuda), to_dev(V[:, lo:hi], cuda))
        st.sharded_partial(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), parts[r],
                           include_tail=(r == world - 1))
        stores.append(st)
    O = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
    stores[0].merge_rank_partials(world, rows, parts, O)
    ok, e = within(from_dev(O), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
    assert ok, e
    for st in stores:
        st.close()


@pytest.mark.parametrize("opt", ["cluster_1", "cluster_2", "cluster_8", "no_cluster_plan", "max_splits_16",
                                 "group_plan", "group_barrier"])
def test_fp8_kernel_options(cuda, opt):
    """E4M3 store under the kernel options: forced cluster sizes of the single-layer
    cluster-merge plan, the LPT plan, a high split cap -- append, all-layer and per-layer
    query parity."""
    import torch
    ssa = _ssa()
    spec = streams.StreamSpec("market", seed=41)
    st, ref = _pair(2, 64, 256)
    if opt.startswith("cluster_"):
        st.set_option(ssa.OPT_CLUSTER, int(opt.split("_")[1]))
    elif opt == "no_cluster_plan":
        st.set_option(ssa.OPT_CLUSTER, -1)
    elif opt == "group_plan":
        st.set_option(ssa.OPT_CM_MERGE, 3)   # group plan for single-layer calls of both planes, merge kernel
    elif opt == "group_barrier":
        st.set_option(ssa.OPT_CM_MERGE, 5)   # group plan for both planes, in-kernel group barrier
    else:
        st.set_option(ssa.OPT_MAX_SPLITS, 16)
    Q, K, V = gen_qkv(spec, 2, LL["hq"], LL["hkv"], LL["d"], 0, 0, 3000)
    sid = st.session_create(None, to_dev(K, cuda), to_dev(V, cuda))
    rsid, _ = ref.session_create(3000, Q, K, V, compute=False)
    Q, K, V = gen_qkv(spec, 2, LL["hq"], LL["hkv"], LL["d"], 0, 3000, 200)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=cuda)
    st.session_append(sid, to_dev(Q, cuda), to_dev(K, cuda), to_dev(V, cuda), O)
    Oref, _ = ref.session_append(rsid, Q, K, V)
    ok, e = within(from_dev(O), Oref, "bf16")
    assert ok, ("append", e)
    for nq in (1, 32):
        Qq, Kq, Vq = gen_qkv(spec, 2, LL["hq"], LL["hkv"], LL["d"], 1, 0, nq)
        Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=cuda)
        st.session_query(sid, to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda), Oq)
        want = ref.session_query(rsid, Qq, Kq, Vq)
        ok, e = within(from_dev(Oq), want, "bf16")
        assert ok, ("query", nq, e)
        Qd, Kd, Vd = to_dev(Qq, cuda), to_dev(Kq, cuda), to_dev(Vq, cuda)
        Ol = torch.full(Qd.shape, float("nan"), dtype=torch.bfloat16, device=cuda)
        for l in range(2):
            st.session_query(sid, Qd[l:l + 1], Kd[l:l + 1], Vd[l:l + 1], Ol[l:l + 1], layer=l)
        if opt in ("group_plan", "group_barrier"):
            assert st.last_plan()["gbar"] == 1, st.last_plan()
        ok, e = within(from_dev(Ol), want, "bf16")
        assert ok, ("per-layer query", nq, e)
    st.close()
