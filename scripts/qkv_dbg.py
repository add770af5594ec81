"""Fused projection per-layer time (32 layers, distinct W, CUDA graph) under the
SSA_OPT_QKV_DEBUG experiments (0 full kernel, 1 no reduce/RoPE/store epilogue), with and
without RoPE (timing only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13784_b200 as ssa  # noqa: E402
import streams  # noqa: E402

dev = torch.device("cuda:0")
L, hq, hkv, d, hidden = 32, 32, 8, 128, 4096
st = ssa.Store(1, hq, hkv, d, page_size=64, num_pages=4, dtype="bf16")
W = [streams.gen_qkv_weight(9, l, 6144, hidden, device=dev) for l in range(L)]
gs = torch.cuda.Stream(device=dev)
for m in [int(x) for x in os.environ.get("QKV_MS", "256 32").split()]:
    X = [streams.gen_hidden(9, 0, 0, l, 0, m, hidden, device=dev) for l in range(L)]
    Q = torch.empty(m, hq, d, dtype=torch.bfloat16, device=dev)
    K = torch.empty(m, hkv, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    for dbg, th, pdl in (((0, 5e5, 1), (1, 5e5, 1)) if os.environ.get("QKV_SHORT") else
                         ((0, 5e5, 1), (1, 5e5, 1), (0, 5e5, 0), (1, 5e5, 0))):
        st.set_option(ssa.OPT_QKV_DEBUG, dbg)
        st.set_option(ssa.OPT_PDL, pdl)
        st.qkv_rope(X[0], W[0], Q, K, V, pos0=100, rope_theta=th, stream=gs)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=gs):
            for l in range(L):
                st.qkv_rope(X[l], W[l], Q, K, V, pos0=100, rope_theta=th, stream=gs)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            g.replay()
        b.record()
        b.synchronize()
        print(f"QKVDBG m={m} debug={dbg} theta={th} pdl={pdl} {a.elapsed_time(b) / 5 / L * 1e3:.1f} us/layer", flush=True)
st.close()
