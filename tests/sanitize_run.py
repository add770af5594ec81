"""Small, fast pass over every kernel of libssa for compute-sanitizer:
SIMT fp32 (toy config), tcgen05 bf16 append / query / flash / batch, E4M3 store, scatter /
gather / digest, retention + alias page copy, split-KV partials + merge, the peer-memory
exchange over two rounds, single-layer cluster-merge launches (DSMEM reduce, merge kernel,
in-kernel last-arriver merge, clusters of 1-8) and per-layer appends, greedy sampling,
fused projection.  Exits non-zero on a parity failure against the fp64 oracle.
    compute-sanitizer --tool memcheck python tests/sanitize_run.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
import streams  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402
from helpers import from_dev, gen_qkv, to_dev, within  # noqa: E402

dev = torch.device("cuda:0")
bad = []


def check(name, got, want, dt):
    ok, e = within(got, want, dt)
    print(f"{name}: max/mean err {e[0]:.2e}/{e[1]:.2e} {'ok' if ok else 'FAIL'}", flush=True)
    if not ok:
        bad.append(name)


# toy fp32 (SIMT kernels, combine)
spec = streams.StreamSpec("peaked", seed=1)
st = ssa.Store(1, 4, 4, 64, page_size=16, num_pages=64, dtype="fp32")
ref = oracle.OracleStore(1, 4, 4, 64, page_size=16, num_pages=64, dtype="fp32")
Q, K, V = gen_qkv(spec, 1, 4, 4, 64, 0, 0, 128, dtype="fp32")
O = torch.empty(Q.shape, dtype=torch.float32, device=dev)
sid = st.session_create(to_dev(Q, dev), to_dev(K, dev), to_dev(V, dev), O)
rsid, want = ref.session_create(128, Q, K, V)
check("fp32 create", from_dev(O), want, "fp32")
Qq, Kq, Vq = gen_qkv(spec, 1, 4, 4, 64, 1, 0, 16, dtype="fp32")
Oq = torch.empty(Qq.shape, dtype=torch.float32, device=dev)
st.session_query(sid, to_dev(Qq, dev), to_dev(Kq, dev), to_dev(Vq, dev), Oq)
check("fp32 query", from_dev(Oq), ref.session_query(rsid, Qq, Kq, Vq), "fp32")
st.close()

# bf16 tcgen05 + E4M3 store: create, append, query (1 and 33 tokens), flash, batch, read-back
for kv in (None, "e4m3"):
    kw = dict(kv_format="e4m3", k_scale=1 / 16, v_scale=1 / 32) if kv else {}
    L, hq, hkv, d = 2, 8, 2, 128
    st = ssa.Store(L, hq, hkv, d, page_size=64, num_pages=64, dtype="bf16", **kw)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=64, num_pages=64, **kw)
    spec = streams.StreamSpec("market", seed=2)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, 300)
    sid = st.session_create(None, to_dev(K, dev), to_dev(V, dev))
    rsid, _ = ref.session_create(300, Q, K, V, compute=False)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 300, 130)
    O = torch.empty(Q.shape, dtype=torch.bfloat16, device=dev)
    st.session_append(sid, to_dev(Q, dev), to_dev(K, dev), to_dev(V, dev), O)
    want, _ = ref.session_append(rsid, Q, K, V)
    check(f"{kv or 'bf16'} append", from_dev(O), want, "bf16")
    for nq in (1, 33):
        Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, nq)
        Oq = torch.empty(Qq.shape, dtype=torch.bfloat16, device=dev)
        st.session_query(sid, to_dev(Qq, dev), to_dev(Kq, dev), to_dev(Vq, dev), Oq)
        check(f"{kv or 'bf16'} query {nq}", from_dev(Oq), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
    lens = [32, 5, 17]
    qs = [gen_qkv(spec, L, hq, hkv, d, streams.FLASH_DOMAIN + i, 0, m) for i, m in enumerate(lens)]
    Qf = np.concatenate([q[0][:1] for q in qs], axis=1)
    Kf = np.concatenate([q[1][:1] for q in qs], axis=1)
    Vf = np.concatenate([q[2][:1] for q in qs], axis=1)
    Of = torch.empty(Qf.shape, dtype=torch.bfloat16, device=dev)
    st.flash_query_batch(sid, lens, to_dev(Qf, dev), to_dev(Kf, dev), to_dev(Vf, dev), Of, layer=0)
    wantf = ref.flash_query_batch(rsid, [(q[0][0], q[1][0], q[2][0]) for q in qs], 0)
    check(f"{kv or 'bf16'} flash", from_dev(Of)[0], np.concatenate(wantf), "bf16")
    items = [(ssa.WORK_QUERY, sid, 20, 0), (ssa.WORK_STATELESS, -1, 150, 20)]
    qa = gen_qkv(spec, L, hq, hkv, d, 7, 0, 20)
    qb = gen_qkv(spec, L, hq, hkv, d, 8, 0, 150)
    Qb, Kb, Vb = (np.concatenate([a, b], axis=1) for a, b in zip(qa, qb))
    Ob = torch.empty(Qb.shape, dtype=torch.bfloat16, device=dev)
    st.batch_run(items, to_dev(Qb, dev), to_dev(Kb, dev), to_dev(Vb, dev), Ob)
    wantb = ref.batch_run([dict(kind="query", session=rsid, Q=qa[0], K=qa[1], V=qa[2]),
                           dict(kind="stateless", session=-1, Q=qb[0], K=qb[1], V=qb[2])])
    check(f"{kv or 'bf16'} batch", from_dev(Ob), np.concatenate(wantb, axis=1), "bf16")
    g = st.alias_prefix(sid, 333)
    st.set_retention(sid, 400)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 430, 64)
    st.session_append(sid, None, to_dev(K, dev), to_dev(V, dev))
    kr, vr = st.read_kv(g, 1, 0, 333)
    ok = st.digest(g) == ref.digest(ref.alias_prefix(rsid, 333))
    print(f"{kv or 'bf16'} alias digest {'ok' if ok else 'FAIL'}", flush=True)
    if not ok:
        bad.append("alias")
    st.close()

# split-KV partials + rank merge (virtual ranks)
from paper_2605_13784_b200.sharding import shard_range  # noqa: E402
L, hq, hkv, d, n = 1, 8, 2, 128, 700
Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
ref = oracle.OracleStore(L, hq, hkv, d, page_size=64, num_pages=64)
rsid, _ = ref.session_create(n, Q, K, V, compute=False)
Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, 32)
parts = torch.empty((2, 32 * hq * (d + 1)), dtype=torch.float32, device=dev)
stores = []
for r in range(2):
    lo, hi = shard_range(n, r, 2)
    s2 = ssa.Store(L, hq, hkv, d, page_size=64, num_pages=64)
    sid2 = s2.session_create(None, to_dev(K[:, lo:hi], dev), to_dev(V[:, lo:hi], dev))
    s2.sharded_partial(sid2, to_dev(Qq, dev), to_dev(Kq, dev), to_dev(Vq, dev), parts[r], include_tail=(r == 1))
    stores.append(s2)
Om = torch.empty(Qq.shape, dtype=torch.bfloat16, device=dev)
stores[0].merge_rank_partials(2, 32, parts, Om)
check("rank merge", from_dev(Om), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
for s2 in stores:
    s2.close()

# peer-memory exchange, two virtual ranks on one stream, two rounds (halves + acks)
from paper_2605_13784_b200.sharding import chunk_floats  # noqa: E402
ch = chunk_floats(32, L, hq, d)
bufs = [torch.zeros(2 * 2 * ch, dtype=torch.float32, device=dev) for _ in range(2)]
flags = [torch.zeros(4, dtype=torch.int32, device=dev) for _ in range(2)]
stores, sids = [], []
for r in range(2):
    lo, hi = shard_range(n, r, 2)
    s2 = ssa.Store(L, hq, hkv, d, page_size=64, num_pages=64)
    sids.append(s2.session_create(None, to_dev(K[:, lo:hi], dev), to_dev(V[:, lo:hi], dev)))
    s2.comm_attach_peers(r, 2, [b.data_ptr() for b in bufs], [f.data_ptr() for f in flags], 2 * 2 * ch * 4)
    stores.append(s2)
for rnd in range(3):
    for r in range(2):
        stores[r].sharded_push(sids[r], to_dev(Qq, dev), to_dev(Kq, dev), to_dev(Vq, dev))
    for r in range(2):
        Om = torch.empty(Qq.shape, dtype=torch.bfloat16, device=dev)
        stores[r].sharded_merge(Om)
        check(f"peer exchange round {rnd} rank {r}", from_dev(Om), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
for s2 in stores:
    s2.close()

# single-layer cluster-merge launches: C = 1..8 (DSMEM reduce), merge kernel / in-kernel merge
for kv in (None, "e4m3"):
    kw = dict(kv_format="e4m3", k_scale=1 / 16, v_scale=1 / 32) if kv else {}
    L, hq, hkv, d, n = 2, 32, 8, 128, 3000
    st = ssa.Store(L, hq, hkv, d, page_size=64, num_pages=64, **kw)
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=64, num_pages=64, **kw)
    Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
    sid = st.session_create(None, to_dev(K, dev), to_dev(V, dev))
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    for nq in (1, 32):
        Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1, 0, nq)
        want = ref.session_query(rsid, Qq, Kq, Vq)
        for C, merge in ((1, 1), (2, 1), (2, 0), (4, 1), (8, 1), (0, 2), (0, 4)):
            st.set_option(ssa.OPT_CLUSTER, C)
            st.set_option(ssa.OPT_CM_MERGE, merge)
            Ol = torch.empty(Qq.shape, dtype=torch.bfloat16, device=dev)
            for l in range(L):
                st.session_query(sid, to_dev(Qq[l:l + 1], dev), to_dev(Kq[l:l + 1], dev), to_dev(Vq[l:l + 1], dev),
                                 Ol[l:l + 1], layer=l)
            check(f"{kv or 'bf16'} per-layer query {nq} C={C} merge={merge} plan={st.last_plan()}", from_dev(Ol), want,
                  "bf16")
    tok = n
    for C, merge in ((4, 1), (0, 3), (0, 5)):   # cluster plan / group plan (merge kernel, group barrier)
        st.set_option(ssa.OPT_CLUSTER, C)
        st.set_option(ssa.OPT_CM_MERGE, merge)
        Qa, Ka, Va = gen_qkv(spec, L, hq, hkv, d, 0, tok, 200)
        Oa = torch.empty(Qa.shape, dtype=torch.bfloat16, device=dev)
        t = st.append_begin(sid, 200)
        for l in range(L):
            st.append_layer(sid, t, l, to_dev(Qa[l:l + 1], dev), to_dev(Ka[l:l + 1], dev), to_dev(Va[l:l + 1], dev),
                            Oa[l:l + 1])
        st.append_commit(sid, t)
        wa, _ = ref.session_append(rsid, Qa, Ka, Va)
        check(f"{kv or 'bf16'} per-layer append C={C} merge={merge} plan={st.last_plan()}", from_dev(Oa), wa, "bf16")
        tok += 200
    st.close()

# greedy sampling + fused projection
st = ssa.Store(1, 8, 2, 128, page_size=64, num_pages=16)
logits = torch.randn(3, 1000, device=dev)
ids = torch.empty(3, dtype=torch.int32, device=dev)
gap = torch.empty(3, dtype=torch.float32, device=dev)
st.greedy_sample(logits, ids, gap)
ok = torch.equal(ids.long().cpu(), logits.argmax(dim=1).cpu())
print(f"greedy {'ok' if ok else 'FAIL'}", flush=True)
if not ok:
    bad.append("greedy")
X = streams.gen_hidden(3, 0, 0, 0, 5, 40, 256)
W = streams.gen_qkv_weight(3, 0, 12 * 128, 256)
Qp = torch.empty((40, 8, 128), dtype=torch.bfloat16, device=dev)
Kp = torch.empty((40, 2, 128), dtype=torch.bfloat16, device=dev)
Vp = torch.empty_like(Kp)
st.qkv_rope(to_dev(X, dev), to_dev(W, dev), Qp, Kp, Vp, pos0=5)
torch.cuda.synchronize()
q, k, v = oracle.qkv_rope(X, W, 8, 2, 128, 5, 500000.0)
check("qkv_rope Q", from_dev(Qp), q, "bf16")
st.close()
print("SANITIZE_RUN", "FAIL " + ",".join(bad) if bad else "OK", flush=True)
sys.exit(1 if bad else 0)
