"""World-size-2 CPU (gloo) tests of the multi-GPU host logic (no GPU needed):
shard ranges, NCCL-id bootstrap over a process group, max-over-ranks timing,
and the split-KV merge across ranks done on the oracle (R-11, R-12)."""
import os
import socket

import numpy as np
import pytest

from paper_2605_13784_b200.sharding import broadcast_unique_id, max_over_ranks, shard_range, tail_owner


def test_shard_ranges_cover_contiguously():
    for n in (0, 1, 7, 131072, 131071):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            for (a, b), (c, d) in zip(parts[:-1], parts[1:]):
                assert b == c
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    assert tail_owner(4) == 3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = bytes(range(128)) if rank == 0 else None
        got = broadcast_unique_id(uid)
        t = max_over_ranks(1.0 + rank)
        # each rank: partial of the same query rows over its token shard (oracle arithmetic),
        # all-gather of the packed (o, lse), merge -> must equal the unsplit attention
        rng = np.random.default_rng(0)
        n, d, rows = 50, 8, 3
        qv, k, v = rng.normal(size=(rows, d)) * 2, rng.normal(size=(n, d)), rng.normal(size=(n, d))
        lo, hi = shard_range(n, rank, world)
        o, lse = oracle.attention_rows(qv, k[lo:hi], v[lo:hi], [hi - lo] * rows, 0.5)
        import torch
        mine = torch.from_numpy(np.concatenate([o.ravel(), lse]))
        allp = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(allp, mine)
        O = np.stack([a[:rows * d].numpy().reshape(rows, d) for a in allp])
        L = np.stack([a[rows * d:].numpy() for a in allp])
        mo, _ = oracle.merge_partials(O, L)
        full, _ = oracle.attention_rows(qv, k, v, [n] * rows, 0.5)
        q.put((rank, got == bytes(range(128)), t, float(np.abs(mo - full).max())))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_bootstrap_and_merge():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, id_ok, t, err in res:
        assert id_ok
        assert t == 2.0
        assert err <= 1e-12
