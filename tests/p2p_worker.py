"""Worker of tests/test_gpu_parity.py::test_sharded_peer_push_two_processes: one rank of a
two-process A9 exchange over CUDA-IPC-mapped peer memory on one GPU."""
import numpy as np


def run(rank, world, bufs, flags, K, V, Qs, Ks, Vs, out_q, n, cfg):
    import torch
    import paper_2605_13784_b200 as ssa
    from paper_2605_13784_b200.sharding import shard_range
    L, hq, hkv, d, P = cfg
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)

    def dv(a):
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(dev)
    lo, hi = shard_range(n, rank, world)
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=64)
    sid = st.session_create(None, dv(K[:, lo:hi]), dv(V[:, lo:hi]))
    st.comm_attach_peers(rank, world, [b.data_ptr() for b in bufs], [f.data_ptr() for f in flags],
                         bufs[0].numel() * 4)   # [2][world][chunk] floats
    outs = []
    for Qq, Kq, Vq in zip(Qs, Ks, Vs):
        O = torch.empty(Qq.shape, dtype=torch.bfloat16, device=dev)
        st.sharded_query(sid, dv(Qq), dv(Kq), dv(Vq), O)
        torch.cuda.synchronize()
        outs.append(O.cpu().view(torch.int16).numpy().view(np.uint16))
    st.close()
    out_q.put((rank, outs))
