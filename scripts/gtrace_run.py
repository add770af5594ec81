"""Launch-phase trace (a -DSSA_GTRACE build of libssa): per CTA %globaltimer of entry /
setup / Q landed / first K / first S / last PV / end for each of the 32 single-layer
query launches of one CUDA-graph replay; prints per-launch phase percentiles (relative
to the launch's first CTA entry) and the gap between consecutive launches."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import streams  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402

C = bench.CFG
L = C["L"]
dev = torch.device("cuda:0")
st = ssa.Store(L, C["hq"], C["hkv"], C["d"], page_size=C["P"], num_pages=C["n_ctx"] // C["P"] + 16, max_sessions=2)
spec = streams.StreamSpec("market", seed=2)
sid = bench.build_session(st, torch, dev, spec, C["n_ctx"])
buf = np.zeros(32 * 256 * 16, dtype=np.uint64)
names = ["entry", "setup", "q", "k0", "s0", "o_fin", "end", None, "staged", "csync1", "reduced", "ticket", "merged",
         "csync2", "o_fin1", "st1"]
for qlen in (32, 1):
    q, k, v = bench.gen_new(torch, dev, spec, 1, 0, qlen)
    o = torch.empty_like(q)

    def per_layer():
        s = torch.cuda.current_stream()
        for l in range(L):
            st.session_query(sid, q[l:l + 1], k[l:l + 1], v[l:l + 1], o[l:l + 1], layer=l, stream=s)
    # GT_CFGS: "cluster,merge ..." (SSA_OPT_CLUSTER, SSA_OPT_CM_MERGE)
    for cl, mk in (tuple(int(x) for x in c.split(",")) for c in os.environ.get("GT_CFGS", "0,1 4,1 0,2").split()):
        st.set_option(ssa.OPT_CLUSTER, cl)
        st.set_option(ssa.OPT_CM_MERGE, mk)
        per_layer()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            per_layer()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        buf[:] = 0
        ssa.lib.ssa_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
        t = buf.reshape(32, 256, 16).astype(np.int64)
        nct = st.last_plan()["ctas"]
        print(f"GT q={qlen} cluster={cl} merge={mk} plan={st.last_plan()}")
        prev_end = None
        spans = []
        for l in range(L):
            tl = t[l, :nct]
            t0 = tl[:, 0].min()
            rel = (tl - t0) / 1000.0
            end = tl[:, 6].max()
            gap = (t0 - prev_end) / 1000.0 if prev_end is not None else float("nan")
            prev_end = end
            spans.append(((end - t0) / 1000.0, gap))
            if l in (0, 1, 16, 31):
                row = " ".join(f"{nm}={np.median(rel[tl[:, i] > 0, i]):.2f}/{rel[tl[:, i] > 0, i].max():.2f}"
                               for i, nm in enumerate(names) if nm and (tl[:, i] > 0).any())
                print(f"GT   layer {l}: span {(end - t0) / 1000.0:.2f} us, gap from prev {gap:.2f} us | p50/max {row}")
        sp = np.array(spans)
        print(f"GT   mean span {sp[:, 0].mean():.2f} us, mean gap {np.nanmean(sp[:, 1]):.2f} us, "
              f"layer period {(t[L - 1, :nct, 6].max() - t[0, :nct, 0].min()) / 1000.0 / L:.2f} us")
