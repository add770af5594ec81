"""Fused-projection experiments: max active clusters per split factor and the kernel
time per (m, splits, debug) on Llama-3-8B shapes, 32 distinct layer weights (CUDA graph)."""
import ctypes
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import torch
    import paper_2605_13784_b200 as ssa
    import streams
    m = int(sys.argv[2])
    dev = torch.device("cuda:0")
    L, hq, hkv, d, hidden = 32, 32, 8, 128, 4096
    st = ssa.Store(1, hq, hkv, d, page_size=64, num_pages=4, dtype="bf16")
    W = [streams.gen_qkv_weight(9, l, 6144, hidden, device=dev) for l in range(L)]
    X = [streams.gen_hidden(9, 0, 0, l, 0, m, hidden, device=dev) for l in range(L)]
    Q = torch.empty(m, hq, d, dtype=torch.bfloat16, device=dev)
    K = torch.empty(m, hkv, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    gs = torch.cuda.Stream()
    for l in range(L):
        st.qkv_rope(X[l], W[l], Q, K, V, pos0=100, stream=gs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for rep in range(5):
        e0.record(gs)
        for l in range(L):
            st.qkv_rope(X[l], W[l], Q, K, V, pos0=100, stream=gs)
        e1.record(gs)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / L)
    print(f"{best * 1e3:.2f}")
    sys.exit(0)

import paper_2605_13784_b200 as ssa  # noqa: E402
ssa.lib.ssa_debug_qkv_clusters.restype = ctypes.c_int32
ssa.lib.ssa_debug_qkv_clusters.argtypes = [ctypes.c_int32]
print("max active clusters:", {s: ssa.lib.ssa_debug_qkv_clusters(s) for s in range(1, 9)})
for m in (256, 32):
    for dbg in (os.environ.get("DBGS", "0,1").split(",")):
        row = []
        for s in os.environ.get("SPLITS", "1,2,3,4,6,8").split(","):
            env = dict(os.environ, SSA_QKV_SPLITS=s, SSA_QKV_DEBUG=dbg)
            out = subprocess.run([sys.executable, __file__, "child", str(m)], env=env, capture_output=True, text=True)
            row.append(f"S={s}:{out.stdout.strip() or out.stderr.strip()[-80:]}")
        print(f"m={m} debug={dbg} us/layer", " ".join(row), flush=True)
