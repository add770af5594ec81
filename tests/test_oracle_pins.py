"""Pins for the fp64 oracle — CPU only.

Each test checks the oracle against something other than itself: an
independent 50-digit mpmath brute force, closed forms, mathematical
invariants, or values printed in the paper/spec (tests/golden/).  Together
they make a dropped term, a wrong sign, an off-by-one in the causal key set,
a wrong GQA index or a transposed operand fail at least one test.
"""
import json
import math
import os
import random

import numpy as np
import pytest

import oracle
import streams

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- brute force
def _mp_attention(q, k, v, nvis, scale):
    """Independent 50-digit implementation of Eq. (attention)."""
    import mpmath as mp
    mp.mp.dps = 50
    out, lses = [], []
    for r in range(len(q)):
        n = int(nvis[r])
        s = [mp.mpf(scale) * mp.fsum(mp.mpf(float(q[r][e])) * mp.mpf(float(k[j][e])) for e in range(len(q[r])))
             for j in range(n)]
        w = [mp.e ** x for x in s]  # no max-subtraction: exact arithmetic at 50 digits
        z = mp.fsum(w)
        out.append([float(mp.fsum(w[j] * mp.mpf(float(v[j][e])) for j in range(n)) / z) for e in range(len(v[0]))])
        lses.append(float(mp.log(z)))
    return np.array(out), np.array(lses)


@pytest.mark.parametrize("seed", range(6))
def test_brute_force_mpmath(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 9))
    d = int(rng.integers(1, 5))
    dv = int(rng.integers(1, 5))
    nr = int(rng.integers(1, 5))
    q = rng.normal(size=(nr, d)) * 2
    k = rng.normal(size=(n, d))
    v = rng.normal(size=(n, dv))
    nvis = rng.integers(1, n + 1, size=nr)
    scale = 1.0 / math.sqrt(d)
    o, lse = oracle.attention_rows(q, k, v, nvis, scale)
    o2, lse2 = _mp_attention(q, k, v, nvis, scale)
    assert np.max(np.abs(o - o2)) <= 1e-13
    assert np.max(np.abs(lse - lse2)) <= 1e-13


def test_two_key_golden():
    line = [l for l in open(os.path.join(GOLDEN, "two_key_softmax.txt")) if not l.startswith("#")][0]
    x = [float(t) for t in line.split()]
    q, k0, k1, v0, v1, o_exp, lse_exp = [x[0]], [x[1]], [x[2]], x[3:5], x[5:7], x[7:9], x[9]
    o, lse = oracle.attention_rows(np.array([q]), np.array([k0, k1]), np.array([v0, v1]), [2], 1.0)
    assert np.allclose(o[0], o_exp, rtol=0, atol=1e-14)
    assert abs(lse[0] - lse_exp) <= 1e-14


# ---------------------------------------------------------------- closed forms
def test_single_key_returns_v():
    rng = np.random.default_rng(1)
    q, k, v = rng.normal(size=(1, 8)), rng.normal(size=(5, 8)), rng.normal(size=(5, 3))
    o, lse = oracle.attention_rows(q, k, v, [1], 0.3)
    assert np.array_equal(o[0], v[0])
    assert lse[0] == pytest.approx(0.3 * float(q[0] @ k[0]), abs=1e-15)


def test_constant_v():
    rng = np.random.default_rng(2)
    q, k = rng.normal(size=(4, 6)) * 3, rng.normal(size=(20, 6))
    v = np.tile(np.array([[1.5, -2.25, 0.125]]), (20, 1))
    o, _ = oracle.attention_rows(q, k, v, [3, 7, 20, 11], 0.5)
    assert np.max(np.abs(o - v[:4])) <= 1e-14


def test_uniform_weights_give_prefix_mean():
    rng = np.random.default_rng(3)
    k, v = rng.normal(size=(10, 4)), rng.normal(size=(10, 2))
    q = np.zeros((10, 4))
    o, lse = oracle.attention_rows(q, k, v, np.arange(1, 11), 1.0)
    for i in range(10):
        assert np.allclose(o[i], v[:i + 1].mean(axis=0), atol=1e-14)
        assert lse[i] == pytest.approx(math.log(i + 1), abs=1e-14)


def test_dominant_logit_selects_value():
    rng = np.random.default_rng(4)
    d = 16
    u = rng.normal(size=d)
    u /= np.linalg.norm(u)
    k = rng.normal(size=(50, d)) * 0.01
    k[17] = 12 * u
    v = rng.normal(size=(50, 5))
    o, _ = oracle.attention_rows((12 * u)[None], k, v, [50], 1.0)  # logit gap ~144
    assert np.max(np.abs(o[0] - v[17])) <= 1e-40 + 1e-14
    o, _ = oracle.attention_rows((12 * u)[None], k, v, [17], 1.0)  # needle not visible
    assert np.max(np.abs(o[0] - v[17])) > 0.1


def test_softmax_sign_and_scale():
    # larger logit must get larger weight; scale multiplies the logits
    q, k, v = np.array([[1.0]]), np.array([[0.0], [2.0]]), np.array([[0.0], [1.0]])
    o1, _ = oracle.attention_rows(q, k, v, [2], 1.0)
    o2, _ = oracle.attention_rows(q, k, v, [2], 0.5)
    assert o1[0, 0] == pytest.approx(math.exp(2) / (1 + math.exp(2)), abs=1e-15)
    assert o2[0, 0] == pytest.approx(math.exp(1) / (1 + math.exp(1)), abs=1e-15)


def test_default_scale_is_inverse_sqrt_dk():
    assert oracle.default_scale(128) == 1.0 / math.sqrt(128)


# ---------------------------------------------------------------- invariants
def test_key_shift_invariance():
    rng = np.random.default_rng(5)
    q, k, v = rng.normal(size=(3, 8)), rng.normal(size=(12, 8)), rng.normal(size=(12, 4))
    w = rng.normal(size=8)
    o1, _ = oracle.attention_rows(q, k, v, [12, 12, 12], 0.4)
    o2, _ = oracle.attention_rows(q, k + w, v, [12, 12, 12], 0.4)
    assert np.max(np.abs(o1 - o2)) <= 1e-13


def test_cached_permutation_invariance():
    rng = np.random.default_rng(6)
    q, k, v = rng.normal(size=(3, 8)) * 2, rng.normal(size=(30, 8)), rng.normal(size=(30, 4))
    perm = rng.permutation(30)
    o1, l1 = oracle.attention_rows(q, k, v, [30] * 3, 0.35)
    o2, l2 = oracle.attention_rows(q, k[perm], v[perm], [30] * 3, 0.35)
    assert np.max(np.abs(o1 - o2)) <= 1e-13 and np.max(np.abs(l1 - l2)) <= 1e-13


@pytest.mark.parametrize("G", [1, 2, 3, 7])
def test_split_merge_identity(G):
    rng = np.random.default_rng(G)
    n, d = 40, 8
    q, k, v = rng.normal(size=(5, d)) * 3, rng.normal(size=(n, d)), rng.normal(size=(n, 6))
    full_o, full_l = oracle.attention_rows(q, k, v, [n] * 5, 0.3)
    cuts = sorted(rng.choice(np.arange(1, n), size=G - 1, replace=False)) if G > 1 else []
    bounds = [0] + list(cuts) + [n]
    parts_o, parts_l = [], []
    for a, b in zip(bounds[:-1], bounds[1:]):
        o, l = oracle.attention_rows(q, k[a:b], v[a:b], [b - a] * 5, 0.3)
        parts_o.append(o)
        parts_l.append(l)
    # an empty shard (lse = -inf) must be skipped (reading R-11)
    parts_o.append(np.zeros_like(parts_o[0]))
    parts_l.append(np.full(5, -np.inf))
    mo, ml = oracle.merge_partials(np.stack(parts_o), np.stack(parts_l))
    assert np.max(np.abs(mo - full_o)) <= 1e-12
    assert np.max(np.abs(ml - full_l)) <= 1e-12


def test_merge_is_not_plain_average():
    # negative control: unequal lse weights must matter
    o = np.stack([np.ones((1, 2)), np.zeros((1, 2))])
    m, _ = oracle.merge_partials(o, np.array([[0.0], [math.log(3.0)]]))
    assert np.allclose(m, 0.25)


def _shape():
    return dict(L=2, hq=4, hkv=2, d=8)


def _inputs(spec, L, H, d, domain, tok0, n, hkv, dtype="fp32"):
    out = []
    for t in (streams.TENSOR_Q, streams.TENSOR_K, streams.TENSOR_V):
        heads = H if t == streams.TENSOR_Q else hkv
        out.append(np.stack([streams.gen_tensor_np(spec, 0, domain, l, t, tok0, n, heads, d, hkv=hkv, dtype=dtype)
                             for l in range(L)]))
    return out


@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_incremental_equals_full_recompute(dtype):
    """Eq. query-attention: appends + query == from-scratch causal attention."""
    s = _shape()
    spec = streams.StreamSpec("peaked", seed=11)
    st = oracle.OracleStore(s["L"], s["hq"], s["hkv"], s["d"], page_size=4, num_pages=64, dtype=dtype)
    chunks = [7, 5, 1, 9]
    tok = 0
    outs = []
    for i, m in enumerate(chunks):
        Q, K, V = _inputs(spec, s["L"], s["hq"], s["d"], 0, tok, m, s["hkv"], dtype)
        if i == 0:
            sid, O = st.session_create(m, Q, K, V)
        else:
            O, _ = st.session_append(sid, Q, K, V)
        outs.append(O)
        tok += m
    Qq, Kq, Vq = _inputs(spec, s["L"], s["hq"], s["d"], 1, 0, 3, s["hkv"], dtype)
    Oq = st.session_query(sid, Qq, Kq, Vq)
    Qd, Kd, Vd = _inputs(spec, s["L"], s["hq"], s["d"], 0, 0, tok, s["hkv"], dtype)
    for l in range(s["L"]):
        qa = np.concatenate([Qd[l], Qq[l]])
        ka = np.concatenate([Kd[l], Kq[l]])
        va = np.concatenate([Vd[l], Vq[l]])
        full = oracle.full_recompute(qa, ka, va, s["hkv"], oracle.default_scale(s["d"]))
        inc = np.concatenate([o[l] for o in outs] + [Oq[l]])
        assert np.max(np.abs(full - inc)) <= 1e-12


def test_chunking_invariance_bit_identical():
    """Any chunking of the same stream gives identical rows (fixed sum order) and digests."""
    s = _shape()
    spec = streams.StreamSpec("market", seed=5, iid_prefix=6)
    total = 29
    rng = random.Random(7)
    ref_rows, ref_digest = None, None
    for trial in range(6):
        cuts = sorted(rng.sample(range(1, total), rng.randint(1, 6)))
        bounds = [0] + cuts + [total]
        st = oracle.OracleStore(s["L"], s["hq"], s["hkv"], s["d"], page_size=4, num_pages=64, dtype="bf16")
        rows = []
        for i, (a, b) in enumerate(zip(bounds[:-1], bounds[1:])):
            Q, K, V = _inputs(spec, s["L"], s["hq"], s["d"], 0, a, b - a, s["hkv"], "bf16")
            if i == 0:
                sid, O = st.session_create(b - a, Q, K, V)
            else:
                O, _ = st.session_append(sid, Q, K, V)
            rows.append(O)
        rows = np.concatenate(rows, axis=1)
        dg = st.digest(sid)
        if ref_rows is None:
            ref_rows, ref_digest = rows, dg
        else:
            assert np.array_equal(rows, ref_rows)
            assert dg == ref_digest


def test_gqa_head_mapping():
    """Reading R-5: q head h uses kv head h // (Hq/Hkv) — pinned with needles."""
    d, n = 16, 12
    u = np.eye(d)
    K = np.zeros((n, 2, d))
    V = np.zeros((n, 2, d))
    K[3, 0] = 20 * u[0]          # kv head 0 needle at token 3
    K[8, 1] = 20 * u[1]          # kv head 1 needle at token 8
    V[3, 0, 0] = 1.0
    V[8, 1, 1] = 1.0
    Q = np.zeros((1, 4, d))
    Q[0, 0:2] = 20 * u[0]
    Q[0, 2:4] = 20 * u[1]
    o, _ = oracle.segment_rows(K[:n - 1], V[:n - 1], Q, K[n - 1:], V[n - 1:], 2, 1.0)
    assert np.allclose(o[0, 0:2, 0], 1.0) and np.allclose(o[0, 2:4, 1], 1.0)
    assert np.allclose(o[0, 0:2, 1], 0.0) and np.allclose(o[0, 2:4, 0], 0.0)


def test_causality_within_segment():
    """Reading R-2: row t sees new tokens 0..t inclusive, never t+1."""
    d = 8
    u = np.eye(d)[0] * 20
    kc = np.zeros((0, 1, d))
    Kn = np.zeros((4, 1, d))
    Vn = np.arange(4, dtype=float).reshape(4, 1, 1) * np.ones((1, 1, d))
    Kn[2, 0] = u   # needle at new token 2
    Qn = np.tile(u, (4, 1, 1))
    o, _ = oracle.segment_rows(kc, kc, Qn, Kn, Vn, 1, 1.0)
    assert o[0, 0, 0] == 0.0                       # row 0 sees only itself
    assert o[1, 0, 0] == pytest.approx(0.5)        # row 1: uniform over {0,1}
    assert o[2, 0, 0] == pytest.approx(2.0, abs=1e-12) and o[3, 0, 0] == pytest.approx(2.0, abs=1e-12)


def test_query_macs_counts_visible_pairs():
    for n, m in [(0, 1), (5, 3), (100, 32)]:
        pairs = sum(n + t + 1 for t in range(m))
        assert oracle.query_macs(n, m, 4, 8) == 4 * 8 * pairs


# ---------------------------------------------------------------- golden
def test_fnv_golden_vectors():
    for line in open(os.path.join(GOLDEN, "fnv1a64.txt")):
        if line.startswith("#") or not line.strip():
            continue
        s, h = line.split()
        assert oracle.fnv1a64(s.strip('"').encode()) == int(h, 16)


def test_paper_numbers():
    g = json.load(open(os.path.join(GOLDEN, "paper_numbers.json")))
    m = g["memory_model_paper_instance"]
    assert oracle.memory_model_bytes(m["L"], m["d"], m["n_ctx"], m["sizeof"]) == m["bytes"]
    assert oracle.derive_seed([]) == g["derive_seed_empty"]["value"]
    # GQA correction (reading R-13): 2*L*Hkv*d_head*n*sizeof for Llama-3-8B shapes
    assert oracle.memory_model_bytes(32, 8 * 128, 32768, 2) == 4294967296


# ---------------------------------------------------------------- store model
def test_page_allocator_lowest_free_first_and_r0_padding():
    st = oracle.OracleStore(1, 1, 1, 4, page_size=4, num_pages=16, dtype="fp32")
    z = lambda n: [np.zeros((1, n, 1, 4), np.float32)] * 3  # noqa: E731
    a, _ = st.session_create(5, *z(5), compute=False)          # 5 tokens -> pages 0,1 (slots 0..4)
    b, _ = st.session_create(3, *z(3), compute=False)          # page 2
    assert st.page_table(a) == [0, 1] and st.page_table(b) == [2]
    st.session_append(a, *z(3), compute=False)                 # R0 padded: slots 8..10 -> new page 3
    assert st.page_table(a) == [0, 1, 3]
    st.session_append(b, *z(2), compute=False)                 # b: 3 prefix -> pad 4, slots 4,5 -> page 4
    assert st.page_table(b) == [2, 4]
    st.session_destroy(a)                                       # frees 0,1,3
    c, _ = st.session_create(9, *z(9), compute=False)          # takes 0,1,3 (lowest first)
    assert st.page_table(c) == [0, 1, 3]
    assert st.occupancy() == (5, 16)


def test_pool_exhausted_leaves_no_state_change():
    st = oracle.OracleStore(1, 1, 1, 4, page_size=4, num_pages=3, dtype="fp32")
    z = lambda n: [np.zeros((1, n, 1, 4), np.float32)] * 3  # noqa: E731
    a, _ = st.session_create(8, *z(8), compute=False)
    before = (st.page_table(a), st.info(a), st.occupancy())
    with pytest.raises(oracle.OracleError) as e:
        st.session_append(a, *z(5), compute=False)
    assert e.value.code == "POOL_EXHAUSTED"
    assert (st.page_table(a), st.info(a), st.occupancy()) == before


def test_state_neutrality_query_and_flash():
    s = _shape()
    spec = streams.StreamSpec("peaked", seed=3)
    st = oracle.OracleStore(s["L"], s["hq"], s["hkv"], s["d"], page_size=4, num_pages=64, dtype="bf16")
    Q, K, V = _inputs(spec, s["L"], s["hq"], s["d"], 0, 0, 13, s["hkv"], "bf16")
    sid, _ = st.session_create(13, Q, K, V)
    d0, i0 = st.digest(sid), st.info(sid)
    for kq in (0, 1, 5, 25):   # SPEC S:691 k in {0,1,5,25}
        qs = []
        for i in range(kq):
            Qf, Kf, Vf = _inputs(spec, 1, s["hq"], s["d"], streams.FLASH_DOMAIN + i, 0, 3, s["hkv"], "bf16")
            qs.append((Qf[0], Kf[0], Vf[0]))
        st.flash_query_batch(sid, qs, 0)
        assert st.digest(sid) == d0
    Qq, Kq, Vq = _inputs(spec, s["L"], s["hq"], s["d"], 1, 0, 4, s["hkv"], "bf16")
    st.session_query(sid, Qq, Kq, Vq)
    assert st.digest(sid) == d0 and st.info(sid) == i0


def test_flash_query_equals_individual_query():
    """Reading R-4: each f_i sees the cache and only its own tokens."""
    s = _shape()
    spec = streams.StreamSpec("peaked", seed=9)
    st = oracle.OracleStore(s["L"], s["hq"], s["hkv"], s["d"], page_size=4, num_pages=64, dtype="bf16")
    Q, K, V = _inputs(spec, s["L"], s["hq"], s["d"], 0, 0, 10, s["hkv"], "bf16")
    sid, _ = st.session_create(10, Q, K, V)
    qs = []
    for i in range(3):
        Qf, Kf, Vf = _inputs(spec, 1, s["hq"], s["d"], streams.FLASH_DOMAIN + i, 0, 2 + i, s["hkv"], "bf16")
        qs.append((Qf[0], Kf[0], Vf[0]))
    outs = st.flash_query_batch(sid, qs, 1)
    for (q, k, v), o in zip(qs, outs):
        ref = st.session_query(sid, q[None], k[None], v[None], layer=1)[0]
        assert np.array_equal(o, ref)


def test_truncate_then_reappend_restores_digest():
    """seq_remove(p) then re-decoding the identical tokens restores the digest."""
    s = _shape()
    spec = streams.StreamSpec("flat", seed=2)
    st = oracle.OracleStore(s["L"], s["hq"], s["hkv"], s["d"], page_size=4, num_pages=64, dtype="bf16")
    Q, K, V = _inputs(spec, s["L"], s["hq"], s["d"], 0, 0, 10, s["hkv"], "bf16")
    sid, _ = st.session_create(6, Q[:, :6], K[:, :6], V[:, :6])
    st.session_append(sid, Q[:, 6:], K[:, 6:], V[:, 6:])
    d0, pt0 = st.digest(sid), st.page_table(sid)
    g = json.load(open(os.path.join(GOLDEN, "paper_numbers.json")))["seq_remove_example"]
    assert st.info(sid)["n_tokens"] == g["n_tokens"]
    st.truncate(sid, g["from_pos"])
    assert st.info(sid)["n_tokens"] == g["n_tokens"] - g["removed"]
    assert st.digest(sid) != d0
    st.session_append(sid, Q[:, 7:], K[:, 7:], V[:, 7:])
    assert st.digest(sid) == d0 and st.page_table(sid) == pt0


def test_batch_snapshot_semantics():
    """Reading R-7: a query batched with an append of the same session sees version t."""
    s = _shape()
    spec = streams.StreamSpec("peaked", seed=4)
    mk = lambda: oracle.OracleStore(s["L"], s["hq"], s["hkv"], s["d"], page_size=4, num_pages=64, dtype="bf16")  # noqa
    Q, K, V = _inputs(spec, s["L"], s["hq"], s["d"], 0, 0, 14, s["hkv"], "bf16")
    Qq, Kq, Vq = _inputs(spec, s["L"], s["hq"], s["d"], 1, 0, 3, s["hkv"], "bf16")
    a = mk()
    sid, _ = a.session_create(9, Q[:, :9], K[:, :9], V[:, :9])
    outs = a.batch_run([dict(kind="append", session=sid, Q=Q[:, 9:], K=K[:, 9:], V=V[:, 9:]),
                        dict(kind="query", session=sid, Q=Qq, K=Kq, V=Vq),
                        dict(kind="stateless", session=-1, Q=Q[:, :5], K=K[:, :5], V=V[:, :5])])
    b = mk()
    sid2, _ = b.session_create(9, Q[:, :9], K[:, :9], V[:, :9])
    ref_q = b.session_query(sid2, Qq, Kq, Vq)
    ref_a, _ = b.session_append(sid2, Q[:, 9:], K[:, 9:], V[:, 9:])
    assert np.array_equal(outs[0], ref_a) and np.array_equal(outs[1], ref_q)
    for l in range(s["L"]):
        ref = oracle.full_recompute(Q[l, :5], K[l, :5], V[l, :5], 2, oracle.default_scale(8))
        assert np.max(np.abs(outs[2][l] - ref)) <= 1e-12
    assert a.digest(sid) == b.digest(sid2) and a.page_table(sid) == b.page_table(sid2)


# --------------------------------------------------------------------------- greedy sampling
def test_greedy_sample_spec_examples():
    """SPEC greedy_sample examples (Eq. logit-gap)."""
    ids, gap = oracle.greedy_sample(np.array([[0.5, 0.5, 0.1]], dtype=np.float32))
    assert ids[0] == 0 and gap[0] == 0.0                         # tie toward the lowest id, gap 0
    ids, gap = oracle.greedy_sample(np.array([[0.3, 3.1, -1.0, 0.9]], dtype=np.float32))
    assert ids[0] == 1 and gap[0] == np.float32(3.1) - np.float32(0.9)   # "top 3.1, second 0.9 -> 2.2"
    assert abs(float(gap[0]) - 2.2) < 1e-6
    hot = np.zeros((1, 97), dtype=np.float32)
    hot[0, 41] = 1.75
    ids, gap = oracle.greedy_sample(hot)
    assert ids[0] == 41 and gap[0] == 1.75                       # one-hot: (k, hot - 0)


def test_greedy_sample_brute_force_and_invariance():
    rng = np.random.default_rng(5)
    x = rng.integers(-3, 4, size=(40, 23)).astype(np.float32)    # many ties
    ids, gap = oracle.greedy_sample(x)
    for r in range(x.shape[0]):
        row = [float(v) for v in x[r]]
        best = max(row)
        assert ids[r] == row.index(best)                         # first index of the max
        rest = sorted(row)[:-1]
        assert gap[r] == best - rest[-1]
    ids2, _ = oracle.greedy_sample(x + np.float32(1000.0))       # argmax invariance (SPEC)
    assert np.array_equal(ids, ids2)
    y = x.copy()
    y[:, 0] = np.nan                                             # NaNs are ignored
    ids3, _ = oracle.greedy_sample(y)
    for r in range(y.shape[0]):
        vals = [float(v) if j else -np.inf for j, v in enumerate(x[r])]
        assert ids3[r] == vals.index(max(vals))
    ids4, gap4 = oracle.greedy_sample(np.full((1, 5), np.nan, dtype=np.float32))
    assert ids4[0] == -1 and gap4[0] == 0.0
