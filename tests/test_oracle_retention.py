"""Pins of the oracle's Region-1 retention (Alg. 1, FIFO evict_oldest) and
metadata-only prefix aliasing (SPEC kv-store evict_oldest / alias_prefix).

Each check is against something other than the oracle's own arithmetic: the
from-scratch causal attention of P:42 (oracle.full_recompute, an independent
function) over the tokens that should remain, the SPEC's worked examples, the
page model's closed forms (reading R-9) and reference-count invariants.
"""
import numpy as np
import pytest

import oracle
import streams

L, HQ, HKV, D, P = 2, 4, 2, 16, 16


def _inp(spec, domain, tok0, n, session=0):
    out = []
    for t in (streams.TENSOR_Q, streams.TENSOR_K, streams.TENSOR_V):
        h = HQ if t == streams.TENSOR_Q else HKV
        out.append(np.stack([streams.gen_tensor_np(spec, session, domain, l, t, tok0, n, h, D, hkv=HKV,
                                                   dtype="fp32") for l in range(L)]))
    return out


def _store(num_pages=64):
    return oracle.OracleStore(L, HQ, HKV, D, page_size=P, num_pages=num_pages, dtype="fp32")


def _grow(st, spec, n_prefix, chunks, session=0):
    Q, K, V = _inp(spec, 0, 0, n_prefix, session)
    sid, _ = st.session_create(n_prefix, Q, K, V, compute=False)
    tok = n_prefix
    for m in chunks:
        Q, K, V = _inp(spec, 0, tok, m, session)
        st.session_append(sid, Q, K, V, compute=False)
        tok += m
    return sid, tok


def test_spec_example_capacity_100_used_95_incoming_10():
    """SPEC kv-store evict_oldest: capacity 100, used 95, incoming 10 -> the 10 oldest
    SLIDING tokens are evicted before the append (Alg. 1 guard); FROZEN untouched."""
    st = _store()
    spec = streams.StreamSpec("flat", seed=1)
    sid, tok = _grow(st, spec, 20, [75])
    st.set_retention(sid, 100)
    Q, K, V = _inp(spec, 0, tok, 10)
    st.session_append(sid, Q, K, V, compute=False)
    s = st.sessions[sid]
    assert s.n_tokens == 95 and s.n_evicted == 10
    assert s.pos == list(range(20)) + list(range(30, 105))    # positions never re-based (R-8)
    # appends within the window do not evict
    st2 = _store()
    sid2, tok2 = _grow(st2, spec, 20, [70])
    st2.set_retention(sid2, 100)
    st2.session_append(sid2, *_inp(spec, 0, tok2, 10), compute=False)
    assert st2.sessions[sid2].n_evicted == 0 and st2.sessions[sid2].n_tokens == 100


def test_evict_zero_is_noop_and_frozen_is_never_evicted():
    st = _store()
    spec = streams.StreamSpec("flat", seed=2)
    sid, _ = _grow(st, spec, 30, [40])
    v0, d0, pt0 = st.info(sid)["version"], st.digest(sid), st.page_table(sid)
    assert st.evict_oldest(sid, 0) == v0 and st.digest(sid) == d0
    with pytest.raises(oracle.OracleError):
        st.evict_oldest(sid, 41)            # only 40 Region-1 tokens: R0 is frozen
    assert st.digest(sid) == d0 and st.page_table(sid) == pt0 and st.info(sid)["version"] == v0
    st.evict_oldest(sid, 40)                # all of Region 1
    s = st.sessions[sid]
    assert s.n_tokens == 30 and s.pos == list(range(30)) and s.r1_skip == 0
    assert len(s.pages) == -(-30 // P)      # only Region 0's pages remain (R-9)


def test_retention_rejects_oversized_batch_without_state_change():
    """SPEC: 'cell-pool exhausted after eviction (batch larger than retention window)'."""
    st = _store()
    spec = streams.StreamSpec("flat", seed=3)
    sid, tok = _grow(st, spec, 10, [20])
    st.set_retention(sid, 30)
    before = (st.digest(sid), st.page_table(sid), st.info(sid), st.occupancy())
    with pytest.raises(oracle.OracleError):
        st.session_append(sid, *_inp(spec, 0, tok, 25), compute=False)   # 25 > 20 evictable
    assert (st.digest(sid), st.page_table(sid), st.info(sid), st.occupancy()) == before


@pytest.mark.parametrize("evict_steps", [[5], [16], [17, 3], [31, 1, 16]])
def test_attention_after_eviction_equals_recompute_over_retained(evict_steps):
    """After eviction the keys are R0 + the newest R1 tokens; a query equals from-scratch
    attention over exactly those keys (followed by the query's own, causal)."""
    st = _store()
    spec = streams.StreamSpec("peaked", seed=4)
    sid, tok = _grow(st, spec, 13, [40, 9])
    for n in evict_steps:
        st.evict_oldest(sid, n)
    ev = sum(evict_steps)
    Qq, Kq, Vq = _inp(spec, 1, 0, 5)
    got = st.session_query(sid, Qq, Kq, Vq)
    _, Kd, Vd = _inp(spec, 0, 0, tok)
    keep = list(range(13)) + list(range(13 + ev, tok))
    for l in range(L):
        ka = np.concatenate([Kd[l][keep], Kq[l]])
        va = np.concatenate([Vd[l][keep], Vq[l]])
        qa = np.concatenate([np.zeros((len(keep), HQ, D), np.float32), Qq[l]])
        want = oracle.full_recompute(qa, ka, va, HKV, oracle.default_scale(D), rows=range(len(keep), len(keep) + 5))
        assert np.max(np.abs(got[l] - want)) <= 1e-12
    # page model: whole pages of evicted slots leave the table; the rest is the hole
    s = st.sessions[sid]
    r0_slots = -(-13 // P) * P
    assert len(s.pages) == -(-(r0_slots + s.r1_skip + (s.n_tokens - 13)) // P)
    assert 0 <= s.r1_skip < P


def test_evicted_pages_are_reused_lowest_id_first():
    st = _store(num_pages=16)
    spec = streams.StreamSpec("flat", seed=5)
    sid, tok = _grow(st, spec, 16, [48])          # R0 page 0, R1 pages 1,2,3
    assert st.page_table(sid) == [0, 1, 2, 3]
    st.evict_oldest(sid, 20)                      # page 1 fully evicted, 4 slots of page 2
    assert st.page_table(sid) == [0, 2, 3] and st.sessions[sid].r1_skip == 4
    sid2, _ = _grow(st, spec, 10, [], session=1)  # next reservation takes page 1 again
    assert st.page_table(sid2) == [1]


def test_alias_then_independent_appends_equal_recompute():
    """SPEC alias_prefix: donor 1000 tokens, alias 1000, decode 1 token on the target ->
    equals recomputing all 1001 tokens; the donor is undisturbed by the target."""
    st = _store(num_pages=256)
    spec = streams.StreamSpec("peaked", seed=6)
    sid, tok = _grow(st, spec, 100, [900])
    d_digest = st.digest(sid)
    used0 = st.occupancy()[0]
    tid = st.alias_prefix(sid, 1000)
    # 1000 = R0 100 (padded to 112) + 900 -> 1012 slots: 63 whole pages shared, 1 copied
    assert st.occupancy()[0] == used0 + 1
    assert st.page_table(tid)[:63] == st.page_table(sid)[:63]
    assert st.page_table(tid)[63] != st.page_table(sid)[63]
    assert st.digest(tid) == d_digest
    Q1, K1, V1 = _inp(spec, 0, 1000, 1)
    O1, _ = st.session_append(tid, Q1, K1, V1)
    Qa, Ka, Va = _inp(spec, 0, 0, 1001)
    for l in range(L):
        want = oracle.full_recompute(Qa[l], Ka[l], Va[l], HKV, oracle.default_scale(D), rows=[1000])
        assert np.max(np.abs(O1[l] - want)) <= 1e-12
    assert st.digest(sid) == d_digest                     # donor undisturbed
    Qd, Kd, Vd = _inp(spec, 3, 1000, 7)                   # a different continuation on the donor
    Od, _ = st.session_append(sid, Qd, Kd, Vd)
    for l in range(L):
        ka = np.concatenate([Ka[l][:1000], Kd[l]])
        va = np.concatenate([Va[l][:1000], Vd[l]])
        qa = np.concatenate([Qa[l][:1000], Qd[l]])
        want = oracle.full_recompute(qa, ka, va, HKV, oracle.default_scale(D), rows=range(1000, 1007))
        assert np.max(np.abs(Od[l] - want)) <= 1e-12


def test_alias_cost_is_constant_and_pages_free_on_last_release():
    """Eq. T_restore: aliasing copies at most one page whatever m is; a shared
    page returns to the pool only when its last referer releases it (SPEC design decision)."""
    st = _store(num_pages=1024)
    spec = streams.StreamSpec("flat", seed=7)
    sid, _ = _grow(st, spec, 64, [9936])               # 10,000 tokens, R0 page-aligned
    for m, copies in ((10, 1), (64, 0), (10000, 0), (9999, 1)):
        used = st.occupancy()[0]
        tid = st.alias_prefix(sid, m)
        assert st.occupancy()[0] - used == copies
        st.session_destroy(tid)
        assert st.occupancy()[0] == used
    tid = st.alias_prefix(sid, 640)                    # 40 shared pages
    used = st.occupancy()[0]
    st.session_destroy(sid)                            # donor gone: shared pages stay
    assert st.occupancy()[0] == used - (len(range(0, 10000, P)) - 40) == 40
    assert st.sessions[tid].n_tokens == 640
    st.session_destroy(tid)
    assert st.occupancy()[0] == 0
    with pytest.raises(oracle.OracleError):
        st.alias_prefix(12345, 1)


def test_alias_len_zero_and_invalid_requests():
    st = _store()
    spec = streams.StreamSpec("flat", seed=8)
    sid, _ = _grow(st, spec, 20, [30])
    tid = st.alias_prefix(sid, 0)                      # SPEC: len 0 -> empty target, no pages
    assert st.info(tid)["n_tokens"] == 0 and st.page_table(tid) == []
    with pytest.raises(oracle.OracleError):
        st.alias_prefix(sid, 51)
    st.evict_oldest(sid, 5)
    with pytest.raises(oracle.OracleError):
        st.alias_prefix(sid, 30)                       # reaches into an evicted Region 1
    t2 = st.alias_prefix(sid, 20)                      # Region 0 only is still contiguous
    assert st.sessions[t2].pos == list(range(20))
