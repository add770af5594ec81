"""Two processes on ONE GPU exercising A9 over peer memory for real (CUDA IPC mapped
symmetric memory, cross-process flags): rank r holds a token shard of one session,
sharded_query = push + flag merge; rank 0 checks against the fp64 oracle.
Run: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/p2p_two_process.py"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle  # noqa: E402
import streams  # noqa: E402
from helpers import from_dev, gen_qkv, to_dev, within  # noqa: E402
import paper_2605_13784_b200 as ssa  # noqa: E402
from paper_2605_13784_b200.sharding import attach_symmetric, chunk_floats, shard_range  # noqa: E402

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
torch.cuda.set_device(0)
dev = torch.device("cuda", 0)
L, hq, hkv, d, P, n = 2, 32, 8, 128, 64, 3001
spec = streams.StreamSpec("market", seed=43)
Q, K, V = gen_qkv(spec, L, hq, hkv, d, 0, 0, n)
lo, hi = shard_range(n, rank, world)
st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
sid = st.session_create(None, to_dev(K[:, lo:hi], dev), to_dev(V[:, lo:hi], dev))
keep = attach_symmetric(st, chunk_floats(32, L, hq, d))
ok_all = True
for rnd in range(3):
    Qq, Kq, Vq = gen_qkv(spec, L, hq, hkv, d, 1 + rnd, 0, 32)
    O = torch.empty(Qq.shape, dtype=torch.bfloat16, device=dev)
    st.sharded_query(sid, to_dev(Qq, dev), to_dev(Kq, dev), to_dev(Vq, dev), O)
    torch.cuda.synchronize()
    ref = oracle.OracleStore(L, hq, hkv, d, page_size=P, num_pages=64)
    rsid, _ = ref.session_create(n, Q, K, V, compute=False)
    ok, e = within(from_dev(O), ref.session_query(rsid, Qq, Kq, Vq), "bf16")
    print(f"rank {rank} round {rnd}: parity {ok} {e}", flush=True)
    ok_all &= ok
    dist.barrier()
st.close()
del keep
dist.destroy_process_group()
sys.exit(0 if ok_all else 1)
