"""Shared test helpers: seeded inputs as numpy (oracle side) and torch (GPU side)."""
import numpy as np

import streams

TOL = {"bf16": (2e-2, 2e-3), "fp32": (1e-5, 1e-5)}   # BASELINE.json north_star


def gen_qkv(spec, L, hq, hkv, d, domain, tok0, n, dtype="bf16", session=0, layers=None):
    """Returns (Q, K, V) numpy arrays [L][n][H][d] in storage dtype (uint16 bf16 bits / float32)."""
    layers = range(L) if layers is None else layers
    out = []
    for t in (streams.TENSOR_Q, streams.TENSOR_K, streams.TENSOR_V):
        h = hq if t == streams.TENSOR_Q else hkv
        out.append(np.stack([streams.gen_tensor_np(spec, session, domain, l, t, tok0, n, h, d, hkv=hkv, dtype=dtype)
                             for l in layers]))
    return out


def to_dev(a, device):
    import torch
    if a.dtype == np.uint16:
        return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).view(torch.bfloat16).to(device)
    return torch.from_numpy(np.ascontiguousarray(a)).to(device)


def from_dev(t):
    import torch
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def f64(a):
    import oracle
    return oracle.to_f64(a)


def errors(got, ref):
    """(max-abs, mean-abs) between a GPU output (storage dtype) and the fp64 oracle."""
    g = f64(got)
    e = np.abs(g - ref)
    return float(e.max()), float(e.mean())


def within(got, ref, dtype):
    mx, mn = errors(got, ref)
    tmax, tmean = TOL[dtype]
    return mx <= tmax and mn <= tmean, (mx, mn)
