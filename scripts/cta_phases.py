"""Per-CTA phase times of an all-layer 256-token append at several contexts (a -DSSA_GTRACE
build, scripts/build_gtrace.sh): entry -> setup -> Q landed -> first K -> first S seen ->
last PV done (slot 0) -> CTA end, median over the CTAs of layers 0-31 (blockIdx.x < 256)."""
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
dev = torch.device("cuda:0")
st = ssa.Store(C["L"], C["hq"], C["hkv"], C["d"], page_size=C["P"], num_pages=C["n_ctx"] // C["P"] + 16, max_sessions=2)
spec = streams.StreamSpec("market", seed=2)
buf = np.zeros(32 * 256 * 16, dtype=np.uint64)
for n in (4096, 16384):
    sid = bench.build_session_n(st, torch, dev, spec, n)
    Qa, Ka, Va = bench.gen_new(torch, dev, spec, 0, n, C["m_append"])
    Oa = torch.empty_like(Qa)
    for _ in range(3):
        st.session_append(sid, Qa, Ka, Va, Oa)
        st.session_truncate(sid, n)
    torch.cuda.synchronize()
    buf[:] = 0
    st.session_append(sid, Qa, Ka, Va, Oa)
    torch.cuda.synchronize()
    ssa.lib.ssa_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    t = buf.reshape(32, 256, 16).astype(np.int64)
    ok = (t[:, :, 0] > 0) & (t[:, :, 6] > 0)
    names = ["setup", "q", "k0", "s0", "o_fin", "end"]
    cols = [1, 2, 3, 4, 5, 6]
    prev = 0
    out = []
    for nm, c in zip(names, cols):
        d = (t[:, :, c] - t[:, :, prev])[ok] / 1000.0
        out.append(f"{nm} +{np.median(d):.2f}")
        prev = c
    tot = (t[:, :, 6] - t[:, :, 0])[ok] / 1000.0
    print(f"PHASES n={n} ctas={ok.sum()} total {np.median(tot):.2f} us | " + " ".join(out), flush=True)
    st.session_destroy(sid)
