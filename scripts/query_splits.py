"""Query-plane split-count sweep (SSA_OPT_MAX_SPLITS) on the bench workload: one
32-token query over 32 layers at n = 32,768 and the 1-token variant."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import streams  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402

CFG = bench.CFG
dev = torch.device("cuda:0")
n = CFG["n_ctx"]
st = ssa.Store(CFG["L"], CFG["hq"], CFG["hkv"], CFG["d"], page_size=CFG["P"], num_pages=n // CFG["P"] + 16,
               max_sessions=2, dtype="bf16")
spec = streams.StreamSpec("market", seed=2)
sid = bench.build_session_n(st, torch, dev, spec, n)
stream = torch.cuda.current_stream()
for qn in (32, 1):
    q, k, v = bench.gen_new(torch, dev, spec, 1, 0, qn)
    o = torch.empty_like(q)
    nb = bench.query_bytes_per_layer(n, qn, CFG["hq"], CFG["hkv"], CFG["d"]) * CFG["L"]
    for ms_cap in (0, 2, 3, 4, 6, 8, 12, 16):
        st.set_option(ssa.OPT_MAX_SPLITS, ms_cap)
        t = bench._timed(torch, stream, lambda: st.session_query(sid, q, k, v, o, stream=stream), 10, 3)
        print(f"q{qn} max_splits {ms_cap:2d}: {t * 1e3 / 32:6.2f} us/layer  {nb / (t * 1e-3) / 1e9:7.0f} GB/s")
