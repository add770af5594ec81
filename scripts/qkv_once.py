"""One fused-projection call per m in argv (default 256 32) on a fresh W (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13784_b200 as ssa  # noqa: E402
import streams  # noqa: E402

dev = torch.device("cuda:0")
hq, hkv, d, hidden = 32, 8, 128, 4096
st = ssa.Store(1, hq, hkv, d, page_size=64, num_pages=4, dtype="bf16")
W = streams.gen_qkv_weight(9, 0, 6144, hidden, device=dev)
for m in [int(x) for x in (sys.argv[1:] or ["256", "32"])]:
    X = streams.gen_hidden(9, 0, 0, 0, 0, m, hidden, device=dev)
    Q = torch.empty(m, hq, d, dtype=torch.bfloat16, device=dev)
    K = torch.empty(m, hkv, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    st.qkv_rope(X, W, Q, K, V, pos0=1000)
    torch.cuda.synchronize()
st.close()
