"""Query-plane timing sweep (E4M3 vs bf16 store, page size, split cap) on the 32k session:
one 32-token query over 32 layers, CUDA events, mean of 10 after 3 warm-ups."""
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
for fp8 in (False, True):
    for P in (64, 128):
        kw = dict(kv_format="e4m3", k_scale=1 / 32, v_scale=1 / 32) if fp8 else {}
        st = ssa.Store(C["L"], C["hq"], C["hkv"], C["d"], page_size=P, num_pages=C["n_ctx"] // P + 16,
                       max_sessions=2, dtype="bf16", **kw)
        spec = streams.StreamSpec("market", seed=2)
        sid = bench.build_session(st, torch, dev, spec, C["n_ctx"])
        q, k, v = bench.gen_new(torch, dev, spec, 1, 0, C["q_len"])
        o = torch.empty_like(q)
        for splits in (0, 4, 8, 16):
            st.set_option(ssa.OPT_MAX_SPLITS, splits)
            ms = bench._timed(torch, stream, lambda: st.session_query(sid, q, k, v, o, stream=stream), 10, 3)
            print(f"TIME fp8={int(fp8)} P={P} max_splits={splits}: {ms * 1e3:.1f} us / 32 layers", flush=True)
        st.close()
        del st
        torch.cuda.empty_cache()
