"""e2e query pieces on the bench session shape: device-only query, H2D / D2H copy times,
and the host-buffer query under SSA_OPT_PIPE_CHUNKS settings (-1 unpipelined, 0 default,
n chunks), interleaved over several rounds (tapered 1:3:3:1 chunks measured 1.14-1.19 ms vs 0.88-0.90 for 2, not kept)."""
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


def t(fn, n=20):
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


print("E2E device query ms", t(lambda: st.session_query(sid, Q, K, V, O, stream=s)))
with torch.cuda.stream(s):
    print("E2E H2D Q,K,V ms", t(lambda: [x.copy_(h, non_blocking=True) for x, h in ((Q, hQ), (K, hK), (V, hV))]))
    print("E2E D2H O ms", t(lambda: hO.copy_(O, non_blocking=True)))
res = {}
for rnd in range(3):
    for pc in (0, 4, 8, -1):
        st.set_option(ssa.OPT_PIPE_CHUNKS, pc)
        res.setdefault(pc, []).append(t(lambda: st.session_query(sid, hQ, hK, hV, hO, stream=s)))
for pc, v in res.items():
    print(f"E2E host query pipe_chunks={pc}: " + " ".join(f"{x:.3f}" for x in v) + " ms")
