"""Host-side helpers for multi-GPU use of libssa (one process per GPU).

* Independent sessions shard across GPUs with no communication: each rank owns
  a ``Store`` and its own sessions (SURVEY §8(e) case 1).
* One long session split by contiguous token ranges (reading R-12, §8(e) case 2):
  rank r holds tokens ``shard_range(n, r, world)`` of every layer as an ordinary
  session of its own store; ``Store.sharded_query`` computes the rank partial,
  exchanges (O, lse) with one NCCL all-gather and merges.  The NCCL unique id is
  bootstrapped through any torch.distributed process group (gloo or nccl).
* The same exchange over peer memory (``attach_symmetric``): the kernel that
  produces a rank partial stores it into every rank's buffer over NVLink and
  releases a flag; each rank's merge acquires all flags (no NCCL launch).
"""
from __future__ import annotations


def shard_range(n_tokens: int, rank: int, world: int):
    """Contiguous, balanced token range [lo, hi) of `rank` (the first n % world ranks get one more)."""
    if world <= 0 or not (0 <= rank < world) or n_tokens < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(n_tokens, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def tail_owner(world: int) -> int:
    """The rank that also covers the query's own tokens (reading R-12)."""
    return world - 1


def broadcast_unique_id(uid: bytes | None, group=None, src: int = 0) -> bytes:
    """Broadcast the 128-byte NCCL unique id from `src` over a torch.distributed group."""
    import torch
    import torch.distributed as dist
    buf = torch.zeros(128, dtype=torch.uint8)
    if dist.get_rank(group) == src:
        assert uid is not None and len(uid) == 128
        buf.copy_(torch.frombuffer(bytearray(uid), dtype=torch.uint8))
    backend = dist.get_backend(group)
    if backend == "nccl":
        buf = buf.cuda()
    dist.broadcast(buf, src=src, group=group)
    return bytes(buf.cpu().tolist())


def init_comm(store, group=None):
    """Join `store` to an NCCL communicator spanning the ranks of `group`."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = store.comm_unique_id() if rank == 0 else None
    uid = broadcast_unique_id(uid, group)
    store.comm_init(rank, world, uid)
    return rank, world


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a per-rank number (device timings are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        return value
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def chunk_floats(n_q: int, num_layers: int, num_q_heads: int, head_dim: int) -> int:
    """fp32 words of one rank partial of an all-layer query of n_q tokens (O rows + lse)."""
    return n_q * num_layers * num_q_heads * (head_dim + 1)


def attach_symmetric(store, max_chunk_floats: int, group=None):
    """Allocate the gathered buffer ([2][world][chunk]: halves alternate by epoch) and the flag
    array ([2][world]: ready, ack) in torch symmetric memory over `group`, exchange the peer
    addresses and attach them to `store` (ssa_comm_attach_peers).  Returns the (buffer, flags)
    tensors, which must stay alive."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    buf = symm_mem.empty(2 * world * max_chunk_floats, dtype=torch.float32, device=dev)
    flags = symm_mem.empty(max(2 * world, 4), dtype=torch.int32, device=dev)
    flags.zero_()
    gname = group.group_name if group is not None else dist.group.WORLD.group_name
    hb = symm_mem.rendezvous(buf, gname)
    hf = symm_mem.rendezvous(flags, gname)
    dist.barrier(group)
    store.comm_attach_peers(rank, world, list(hb.buffer_ptrs), list(hf.buffer_ptrs),
                            2 * world * max_chunk_floats * 4)
    return buf, flags
