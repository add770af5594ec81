"""Per-layer query calls on the 32k session: kernel times (SSA_OPT_TIMING) and the plan
(units / split groups) of a single-layer call vs the all-layer call."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402
import streams  # noqa: E402

C = bench.CFG
dev = torch.device("cuda", 0)
st = ssa.Store(C["L"], C["hq"], C["hkv"], C["d"], page_size=C["P"], num_pages=C["n_ctx"] // C["P"] + 16, max_sessions=2)
spec = streams.StreamSpec("market", seed=2)
sid = bench.build_session(st, torch, dev, spec, C["n_ctx"])
q, k, v = bench.gen_new(torch, dev, spec, 1, 0, C["q_len"])
o = torch.empty_like(q)
for mode in ("all", "per_layer"):
    for _ in range(2):
        if mode == "all":
            st.session_query(sid, q, k, v, o)
        else:
            for l in range(C["L"]):
                st.session_query(sid, q[l:l + 1], k[l:l + 1], v[l:l + 1], o[l:l + 1], layer=l)
    torch.cuda.synchronize()
    st.set_option(ssa.OPT_TIMING, 1)
    st.timing(reset=True)
    if mode == "all":
        st.session_query(sid, q, k, v, o)
    else:
        for l in range(C["L"]):
            st.session_query(sid, q[l:l + 1], k[l:l + 1], v[l:l + 1], o[l:l + 1], layer=l)
    tm = st.timing(reset=True)
    st.set_option(ssa.OPT_TIMING, 0)
    print("LAYER", mode, {a: (round(b[0] * 1e3, 1), b[1]) for a, b in tm.items() if b[1]}, st.last_plan() if hasattr(st, "last_plan") else "")
for ms in (2, 4, 6, 8, 12, 16):
    st.set_option(ssa.OPT_MAX_SPLITS, ms)
    for l in range(C["L"]):
        st.session_query(sid, q[l:l + 1], k[l:l + 1], v[l:l + 1], o[l:l + 1], layer=l)
    torch.cuda.synchronize()
    st.set_option(ssa.OPT_TIMING, 1)
    st.timing(reset=True)
    for l in range(C["L"]):
        st.session_query(sid, q[l:l + 1], k[l:l + 1], v[l:l + 1], o[l:l + 1], layer=l)
    tm = st.timing(reset=True)
    st.set_option(ssa.OPT_TIMING, 0)
    print("LAYER max_splits", ms, {a: (round(b[0] * 1e3 / 32, 1), b[1]) for a, b in tm.items() if b[1]})
st.set_option(ssa.OPT_MAX_SPLITS, 0)
for fm in (1,):
    st.set_option(ssa.OPT_FUSED_MERGE, fm)
    for ms in (0, 8, 16):
        st.set_option(ssa.OPT_MAX_SPLITS, ms)
        for l in range(C["L"]):
            st.session_query(sid, q[l:l + 1], k[l:l + 1], v[l:l + 1], o[l:l + 1], layer=l)
        torch.cuda.synchronize()
        st.set_option(ssa.OPT_TIMING, 1)
        st.timing(reset=True)
        for l in range(C["L"]):
            st.session_query(sid, q[l:l + 1], k[l:l + 1], v[l:l + 1], o[l:l + 1], layer=l)
        tm = st.timing(reset=True)
        st.set_option(ssa.OPT_TIMING, 0)
        print("LAYER fused_merge max_splits", ms, {a: (round(b[0] * 1e3 / 32, 1), b[1]) for a, b in tm.items() if b[1]})
# 1-token per-layer query
q1, k1, v1 = bench.gen_new(torch, dev, spec, 1, 0, 1)
o1 = torch.empty_like(q1)
st.set_option(ssa.OPT_FUSED_MERGE, 0)
st.set_option(ssa.OPT_MAX_SPLITS, 0)
for l in range(C["L"]):
    st.session_query(sid, q1[l:l + 1], k1[l:l + 1], v1[l:l + 1], o1[l:l + 1], layer=l)
torch.cuda.synchronize()
st.set_option(ssa.OPT_TIMING, 1)
st.timing(reset=True)
for l in range(C["L"]):
    st.session_query(sid, q1[l:l + 1], k1[l:l + 1], v1[l:l + 1], o1[l:l + 1], layer=l)
tm = st.timing(reset=True)
print("LAYER q1 per-layer", {a: (round(b[0] * 1e3 / 32, 1), b[1]) for a, b in tm.items() if b[1]})
