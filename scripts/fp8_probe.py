"""One 32-token query over 32 layers at n = 32,768 on an E4M3 (or bf16) store, for ncu:
  ncu --set full -k regex:attn_tc_kernel -c 1 python scripts/fp8_probe.py [bf16]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402
import streams  # noqa: E402

fp8 = "bf16" not in sys.argv[1:]
C = bench.CFG
dev = torch.device("cuda", 0)
kw = dict(kv_format="e4m3", k_scale=1 / 32, v_scale=1 / 32) if fp8 else {}
st = ssa.Store(C["L"], C["hq"], C["hkv"], C["d"], page_size=C["P"], num_pages=C["n_ctx"] // C["P"] + 16,
               max_sessions=2, dtype="bf16", **kw)
spec = streams.StreamSpec("market", seed=2)
sid = bench.build_session(st, torch, dev, spec, C["n_ctx"])
q, k, v = bench.gen_new(torch, dev, spec, 1, 0, C["q_len"])
o = torch.empty_like(q)
st.session_query(sid, q, k, v, o)
torch.cuda.synchronize()
print("ok", fp8)
