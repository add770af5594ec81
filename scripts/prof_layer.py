"""One single-layer 32-token query at n = 32,768 (the cluster-merge launch + its merge kernel)
after a warm-up, for an ncu capture: `ncu -k regex:"attn_tc|cm_merge" -s 4 -c 2`."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402
import streams  # noqa: E402

C = bench.CFG
st = ssa.Store(C["L"], C["hq"], C["hkv"], C["d"], page_size=C["P"], num_pages=C["n_ctx"] // C["P"] + 16, max_sessions=2)
dev = torch.device("cuda", 0)
spec = streams.StreamSpec("market", seed=2)
sid = bench.build_session(st, torch, dev, spec, C["n_ctx"])
q, k, v = bench.gen_new(torch, dev, spec, 1, 0, int(os.environ.get("QLEN", "32")))
o = torch.empty_like(q)
for _ in range(3):
    st.session_query(sid, q[5:6], k[5:6], v[5:6], o[5:6], layer=5)
torch.cuda.synchronize()
st.session_query(sid, q[5:6], k[5:6], v[5:6], o[5:6], layer=5)
torch.cuda.synchronize()
print("plan", st.last_plan())
