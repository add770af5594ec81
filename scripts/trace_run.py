"""Run the bench append + query once with a -DSSA_TRACE build and dump the kernel's
clock64 trace (ssa_debug_trace) to gpurun_out/trace_<kind>.npy."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import streams  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402

CFG = bench.CFG
dev = torch.device("cuda:0")
n0 = CFG["n_ctx"] - CFG["m_append"]
KV = os.environ.get("KV", "bf16")   # "e4m3": an E4M3 KV store (bench fp8_kv leg scales)
kvkw = dict(kv_format="e4m3", k_scale=1 / 32, v_scale=1 / 32) if KV == "e4m3" else {}
st = ssa.Store(CFG["L"], CFG["hq"], CFG["hkv"], CFG["d"], page_size=CFG["P"], num_pages=CFG["n_ctx"] // CFG["P"] + 16,
               max_sessions=4, dtype="bf16", **kvkw)
spec = streams.StreamSpec("market", seed=2)
sid = bench.build_session(st, torch, dev, spec, n0)
Qa, Ka, Va = bench.gen_new(torch, dev, spec, 0, n0, CFG["m_append"])
Oa = torch.empty_like(Qa)
Qq, Kq, Vq = bench.gen_new(torch, dev, spec, 1, 0, CFG["q_len"])
Oq = torch.empty_like(Qq)
buf = np.zeros(4 * 12 * 256 * 2 + 4 * 2 * 4 * 256 * 2, dtype=np.uint64)
n1 = 4 * 12 * 256 * 2
lib = ssa.lib
for kind in ("append", "query"):
    for _ in range(3):
        if kind == "append":
            st.session_append(sid, Qa, Ka, Va, Oa)
            st.session_truncate(sid, n0)
        else:
            st.session_query(sid, Qq, Kq, Vq, Oq)
    torch.cuda.synchronize()
    n = lib.ssa_debug_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
    print(kind, "trace bytes", n)
    os.makedirs("gpurun_out", exist_ok=True)
    np.save(f"gpurun_out/trace_{KV}_{kind}.npy", buf[:n1].reshape(4, 12, 256, 2).copy())
    np.save(f"gpurun_out/trace2_{KV}_{kind}.npy", buf[n1:].reshape(4, 2, 4, 256, 2).copy())
    buf[:] = 0
