"""Per-layer calls on the 32k bench session: device time of 32 single-layer 32-token
(and 1-token) queries and of one per-layer 256-token append step, replayed from a CUDA
graph, under each cluster-merge setting (SSA_OPT_CLUSTER) and with / without PDL; plus
the plan of a single-layer call (units, groups, CTAs, cluster size, clusters per group)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402
import streams  # noqa: E402

C = bench.CFG
L = C["L"]
dev = torch.device("cuda", 0)
st = ssa.Store(L, C["hq"], C["hkv"], C["d"], page_size=C["P"], num_pages=C["n_ctx"] // C["P"] + 16, max_sessions=2)
spec = streams.StreamSpec("market", seed=2)
n0 = C["n_ctx"] - C["m_append"]
sid = bench.build_session(st, torch, dev, spec, n0)
Qa, Ka, Va = bench.gen_new(torch, dev, spec, 0, n0, C["m_append"])
print("LAYER max active clusters", {c: ssa.lib.ssa_debug_tc_clusters(c, 0) for c in (1, 2, 3, 4, 5, 6, 7, 8, 16)})
Oa = torch.empty_like(Qa)


def timed(fn, reps=20):
    s = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    b.synchronize()
    return a.elapsed_time(b) / reps


def graph_of(fn):
    fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


for q_len in (32, 1):
    st.session_truncate(sid, n0)
    st.session_append(sid, Qa, Ka, Va, Oa)   # n = 32,768
    q, k, v = bench.gen_new(torch, dev, spec, 1, 0, q_len)
    o = torch.empty_like(q)

    def per_layer():
        s = torch.cuda.current_stream()
        for l in range(L):
            st.session_query(sid, q[l:l + 1], k[l:l + 1], v[l:l + 1], o[l:l + 1], layer=l, stream=s)
    for cl, pdl, mk in [tuple(int(x) for x in c.split(",")) for c in os.environ.get(
            "LAYER_CFGS", "0,1,1 4,1,1 0,1,2 0,0,2").split()]:
        if True:
            st.set_option(ssa.OPT_CLUSTER, cl)
            st.set_option(ssa.OPT_PDL, pdl)
            st.set_option(ssa.OPT_CM_MERGE, mk)
            g = graph_of(per_layer)
            ms = timed(g.replay)
            print(f"LAYER q={q_len} cluster={cl} pdl={pdl} merge_kernel={mk} graph {ms * 1e3 / L:.1f} us/layer "
                  f"plan {st.last_plan()}", flush=True)
    st.set_option(ssa.OPT_CM_MERGE, 0)
    st.set_option(ssa.OPT_PDL, 1)
    ms = timed(lambda: st.session_query(sid, q, k, v, o))
    print(f"LAYER q={q_len} all-layer call {ms * 1e3 / L:.1f} us/layer plan {st.last_plan()}", flush=True)

st.set_option(ssa.OPT_PDL, 1)
for cl, mk in (((0, 1), (4, 1), (0, 2)) if os.environ.get("LAYER_APPEND", "1") != "0" else ()):
    st.set_option(ssa.OPT_CLUSTER, cl)
    st.set_option(ssa.OPT_CM_MERGE, mk)
    st.session_truncate(sid, n0)
    reps = 10
    tot = 0.0
    for r in range(reps + 2):
        t = st.append_begin(sid, C["m_append"])
        g = torch.cuda.CUDAGraph()
        if r == 0:   # eager warm-up (caches the work lists)
            for l in range(L):
                st.append_layer(sid, t, l, Qa[l:l + 1], Ka[l:l + 1], Va[l:l + 1], Oa[l:l + 1])
        else:
            with torch.cuda.graph(g):
                s = torch.cuda.current_stream()
                for l in range(L):
                    st.append_layer(sid, t, l, Qa[l:l + 1], Ka[l:l + 1], Va[l:l + 1], Oa[l:l + 1], stream=s)
        st.append_commit(sid, t)
        if r > 0:
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            g.replay()
            b.record()
            b.synchronize()
            if r >= 2:
                tot += a.elapsed_time(b)
        st.session_truncate(sid, n0)
    ms = tot / reps
    fl = bench.append_flops_per_layer(n0, C["m_append"], C["hq"], C["d"])
    print(f"LAYER append cluster={cl} merge={mk} graph {ms * 1e3 / L:.1f} us/layer = {fl / (ms / L * 1e-3) / 1e12:.0f} TFLOP/s "
          f"plan {st.last_plan()}", flush=True)
