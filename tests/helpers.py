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


def abs_bits(x):
    """|x| of bf16 bit patterns (clear the sign bit) or floats, exactly."""
    x = np.asarray(x)
    return x & np.uint16(0x7FFF) if x.dtype == np.uint16 else np.abs(x)


def attention_bound(A, o_ref, n_keys, p_unit=2.0 ** -8):
    """Derived per-element error bound of a tcgen05 attention output against the fp64 oracle
    (parity bound).  The kernel rounds each weight p_j to bf16 (relative error
    <= 2^-8; fp16 for an E4M3 store: p_unit = 2^-11) before P V but normalises by the fp32 sum
    of the unrounded weights, so the weight rounding moves O_e by at most p_unit *
    sum_j w_j |v_j[e]| = p_unit * A_e, where A is the oracle's attention output with |V| in
    place of V; fp32 accumulation over n keys adds at most n * 2^-24 * A_e; the one rounding of
    O to bf16 adds 2^-8 |O_e|.  A 1.25 factor covers the fp32 score / exp2 / split-merge terms
    (each below 2^-12 relative)."""
    return 1.25 * (p_unit + n_keys * 2.0 ** -24) * np.asarray(A) + 2.0 ** -8 * np.abs(o_ref) + 1e-6


def within_bound(got, ref, bound):
    """(all errors within the derived bound, largest error / bound)."""
    e = np.abs(f64(got) - ref)
    r = e / bound
    return bool((r <= 1.0).all()), float(r.max())
