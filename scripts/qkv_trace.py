"""Per-CTA phase timeline of the fused projection (ssa_debug_qkv_trace): median and max
over CTAs of each phase, for the Llama-3-8B shapes."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13784_b200 as ssa  # noqa: E402
import streams  # noqa: E402

ssa.lib.ssa_debug_qkv_trace.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda:0")
hq, hkv, d, hidden = 32, 8, 128, 4096
st = ssa.Store(1, hq, hkv, d, page_size=64, num_pages=4, dtype="bf16")
W = streams.gen_qkv_weight(9, 0, 6144, hidden, device=dev)
buf = torch.zeros(4096 * 10, dtype=torch.int64, device=dev)
names = ["setup", "mainloop", "dump", "csync1", "epilogue", "csync2"]
for m in [int(x) for x in (sys.argv[1:] or ["256", "32"])]:
    X = streams.gen_hidden(9, 0, 0, 0, 0, m, hidden, device=dev)
    Q = torch.empty(m, hq, d, dtype=torch.bfloat16, device=dev)
    K = torch.empty(m, hkv, d, dtype=torch.bfloat16, device=dev)
    V = torch.empty_like(K)
    for rep in range(3):
        buf.zero_()
        ssa.lib.ssa_debug_qkv_trace(buf.data_ptr() if rep == 2 else None)
        st.qkv_rope(X, W, Q, K, V, pos0=1000)
        torch.cuda.synchronize()
    ssa.lib.ssa_debug_qkv_trace(None)
    t = buf.view(-1, 10).cpu()
    t = t[t[:, 0] > 0].double()
    t0 = t[:, 0].min()
    print(f"m={m} ctas={len(t)} kernel span {(t[:, 6].max() - t0) / 1e3:.2f} us; start spread "
          f"{(t[:, 0].max() - t0) / 1e3:.2f} us")
    for nm, a, b in (("acc->csync", 2, 7), ("push", 7, 3), ("table done (after acc)", 2, 8)):
        dt = (t[:, b] - t[:, a]) / 1e3
        print(f"  {nm:9s} median {dt.median():7.2f} us  max {dt.max():7.2f} us")
    for i, nm in enumerate(names):
        dt = (t[:, i + 1] - t[:, i]) / 1e3
        print(f"  {nm:9s} median {dt.median():7.2f} us  max {dt.max():7.2f} us")
st.close()
