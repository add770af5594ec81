"""e2e query pieces on the bench session shape: device-only query, H2D / D2H copy times,
and the host-buffer query with SSA_PIPE_CHUNKS (0 = unpipelined) from the environment."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_13784_b200 as ssa  # noqa: E402
import streams  # noqa: E402
import bench  # noqa: E402

dev = torch.device("cuda:0")
L, hq, hkv, d = 32, 32, 8, 128
st = ssa.Store(L, hq, hkv, d, page_size=64, num_pages=32768 // 64 + 64)
spec = streams.StreamSpec("market", seed=2)
sid = bench.build_session_n(st, torch, dev, spec, 32768)
Q, K, V = bench.gen_new(torch, dev, spec, 1, 0, 32)
O = torch.empty_like(Q)
hQ, hK, hV = (x.cpu().pin_memory() for x in (Q, K, V))
hO = torch.empty(O.shape, dtype=O.dtype).pin_memory()
s = torch.cuda.Stream()


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(n):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("device query ms", t(lambda: st.session_query(sid, Q, K, V, O, stream=s)))
os.environ["SSA_PIPE_FORCE"] = "1"
print("device query, chunked ms", t(lambda: st.session_query(sid, Q, K, V, O, stream=s)))
del os.environ["SSA_PIPE_FORCE"]
with torch.cuda.stream(s):
    print("H2D Q,K,V ms", t(lambda: [x.copy_(h, non_blocking=True) for x, h in ((Q, hQ), (K, hK), (V, hV))]))
    print("D2H O ms", t(lambda: hO.copy_(O, non_blocking=True)))
print("host query ms (SSA_PIPE_CHUNKS=%s)" % os.environ.get("SSA_PIPE_CHUNKS"),
      t(lambda: st.session_query(sid, hQ, hK, hV, hO, stream=s)))
