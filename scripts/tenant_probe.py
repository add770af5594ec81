"""BJ.configs[2] by class: the 48-session varlen batch (one launch over 32 layers) timed whole and
with only its appends, only its queries, only its stateless prompts (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402
import streams  # noqa: E402

C = bench.CFG
dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream()
L, hq, hkv, d, P = C["L"], C["hq"], C["hkv"], C["d"], C["P"]
ns = [4096 + 256 * s for s in range(48)]
st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=sum(-(-(n + 256) // P) for n in ns) + 64, max_sessions=64)
spec = streams.StreamSpec("market", seed=3)
sids = [bench.build_session_n(st, torch, dev, spec, n, session=s) for s, n in enumerate(ns)]
items, Qs, Ks, Vs, row = [], [], [], [], 0
for s, n in enumerate(ns):
    m = 256 if s % 2 == 0 else 32
    q, k, v = bench.gen_new(torch, dev, spec, 0 if m == 256 else 1, n if m == 256 else 0, m, session=s)
    items.append((ssa.WORK_APPEND if m == 256 else ssa.WORK_QUERY, sids[s], m, row))
    Qs.append(q); Ks.append(k); Vs.append(v)
    row += m
for j in range(4):
    q, k, v = bench.gen_new(torch, dev, spec, 100 + j, 0, 1024, session=60 + j)
    items.append((ssa.WORK_STATELESS, -1, 1024, row))
    Qs.append(q); Ks.append(k); Vs.append(v)
    row += 1024
Q, K, V = (torch.cat(x, dim=1).contiguous() for x in (Qs, Ks, Vs))
O = torch.empty_like(Q)


def run(sel):
    its = [it for it in items if it[0] in sel]

    def step():
        st.batch_run(its, Q, K, V, O, stream=stream)
        for s in range(0, 48, 2):
            st.session_truncate(sids[s], ns[s])
    return bench._timed(torch, stream, step, 3, 1)


A, Qy, S = ssa.WORK_APPEND, ssa.WORK_QUERY, ssa.WORK_STATELESS
for name, sel in (("all", (A, Qy, S)), ("appends", (A,)), ("queries", (Qy,)), ("stateless", (S,)),
                  ("appends+stateless", (A, S))):
    print(f"TENANT {name}: {run(sel):.2f} ms / 32 layers", flush=True)
for ms in (0, 2, 4):
    st.set_option(ssa.OPT_MAX_SPLITS, ms)
    print(f"TENANT all max_splits={ms}: {run((A, Qy, S)):.2f} ms", flush=True)
