"""A/B of store options on the bench step (BJ.configs[1]: 256-token append + 32-token query
over 32 layers at n = 32,512 / 32,768): per-kernel device times (SSA_OPT_TIMING) and the
step time (events around the steps, PDL active) for each setting."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402
import streams  # noqa: E402

C = bench.CFG
L = C["L"]
dev = torch.device("cuda", 0)
st = ssa.Store(L, C["hq"], C["hkv"], C["d"], page_size=C["P"], num_pages=C["n_ctx"] // C["P"] + 16, max_sessions=2)
spec = streams.StreamSpec("market", seed=2)
n0 = C["n_ctx"] - C["m_append"]
sid = bench.build_session(st, torch, dev, spec, n0)
Qa, Ka, Va = bench.gen_new(torch, dev, spec, 0, n0, C["m_append"])
Oa = torch.empty_like(Qa)
Qq, Kq, Vq = bench.gen_new(torch, dev, spec, 1, 0, C["q_len"])
Oq = torch.empty_like(Qq)
s = torch.cuda.current_stream()


def step():
    st.session_append(sid, Qa, Ka, Va, Oa, stream=s)
    st.session_query(sid, Qq, Kq, Vq, Oq, stream=s)
    st.session_truncate(sid, n0)


if os.environ.get("AB_SET"):   # e.g. AB_SET=14:1,10:0 -> one setting
    settings = [{int(k): int(v) for k, v in (kv.split(":") for kv in os.environ["AB_SET"].split(","))}]
    os.environ["AB_ONLY_DEFAULT"] = "1"
elif os.environ.get("AB_ONLY_DEFAULT"):
    settings = [dict()]
else:
    settings = [dict(), {ssa.OPT_L2_HINT: 1}, {ssa.OPT_L2_HINT: 2}, {ssa.OPT_PDL: 0}, {ssa.OPT_PDL: 0, ssa.OPT_L2_HINT: 1}]
for rep in range(1 if os.environ.get("AB_ONLY_DEFAULT") else int(os.environ.get("AB_REPS", "2"))):
    for opts in settings:
        for k, v in opts.items():
            st.set_option(k, v)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        st.set_option(ssa.OPT_TIMING, 1)
        st.timing(reset=True)
        for _ in range(5):
            step()
        tm = st.timing(reset=True)
        st.set_option(ssa.OPT_TIMING, 0)
        step_ms = bench._timed(torch, s, step, 10, 2)
        qa = tm["attn_query"][0] / max(1, tm["attn_query"][1])
        aa = tm["attn_data"][0] / max(1, tm["attn_data"][1])
        print(f"AB {opts} step {step_ms:.3f} ms  append attn {aa:.3f} ms "
              f"({bench.append_flops_per_layer(n0, C['m_append'], C['hq'], C['d']) * L / (aa * 1e-3) / 1e12:.0f} TF)  "
              f"query attn {qa * 1e3:.1f} us ({bench.query_bytes_per_layer(C['n_ctx'], C['q_len'], C['hq'], C['hkv'], C['d']) * L / (qa * 1e-3) / 1e9:.0f} GB/s)",
              flush=True)
        for k in opts:
            st.set_option(k, {getattr(ssa, "OPT_PDL", -1): 1, getattr(ssa, "OPT_L2_HINT", -1): 0}.get(k, 0))
