"""A/B of the per-layer 256-token append (32 append_layer calls in one CUDA graph) under
merge settings, alternating configurations over several rounds on the 32k bench session."""
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
Oa = torch.empty_like(Qa)
cfgs = [tuple(int(x) for x in c.split(",")) for c in os.environ.get("AB_CFGS", "0,2 4,1 0,1 3,1").split()]
res = {c: [] for c in cfgs}
fl = bench.append_flops_per_layer(n0, C["m_append"], C["hq"], C["d"])
for rnd in range(4):
    for cl, mk in cfgs:
        st.set_option(ssa.OPT_CLUSTER, cl)
        st.set_option(ssa.OPT_CM_MERGE, mk)
        ts = []
        for r in range(5):
            t = st.append_begin(sid, C["m_append"])
            if r == 0:
                for l in range(L):
                    st.append_layer(sid, t, l, Qa[l:l + 1], Ka[l:l + 1], Va[l:l + 1], Oa[l:l + 1])
            else:
                g = torch.cuda.CUDAGraph()
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
                ts.append(a.elapsed_time(b) / L * 1e3)
            st.session_truncate(sid, n0)
        res[(cl, mk)].append(min(ts))
for c, v in res.items():
    us = sorted(v)[len(v) // 2]
    print(f"AB append cluster={c[0]} merge={c[1]} median {us:.1f} us/layer ({fl / (us * 1e-6) / 1e12:.0f} TFLOP/s) all {['%.1f' % x for x in v]} plan {st.last_plan() if False else ''}")
