"""streams.py: the numpy and torch implementations of the seeded generator produce identical
bits (on CPU here; tests/test_gpu_parity.py repeats it on the GPU), every element is a pure
function of its coordinates (any chunking sees the same bits), and the stream
recipes have the statistics DESIGN.md §3 states."""
import numpy as np
import pytest

import streams


@pytest.mark.parametrize("name", streams.STREAMS)
@pytest.mark.parametrize("tensor", [streams.TENSOR_Q, streams.TENSOR_K, streams.TENSOR_V])
def test_torch_cpu_matches_numpy(name, tensor):
    import torch
    spec = streams.StreamSpec(name, seed=13, needles=(3, 70))
    heads = 32 if tensor == streams.TENSOR_Q else 8
    for domain in (0, 1, streams.FLASH_DOMAIN + 2):
        a = streams.gen_tensor_np(spec, 2, domain, 1, tensor, 50, 40, heads, 128, hkv=8)
        b = streams.gen_tensor_torch(spec, 2, domain, 1, tensor, 50, 40, heads, 128, hkv=8, device="cpu")
        assert np.array_equal(a, b.view(torch.int16).numpy().view(np.uint16)), (name, tensor, domain)


@pytest.mark.parametrize("name", streams.STREAMS)
def test_chunking_invariance(name):
    spec = streams.StreamSpec(name, seed=5, needles=(7, 600))
    whole = streams.gen_tensor_np(spec, 0, 0, 3, streams.TENSOR_K, 0, 700, 8, 64)
    parts = [streams.gen_tensor_np(spec, 0, 0, 3, streams.TENSOR_K, a, b - a, 8, 64)
             for a, b in ((0, 1), (1, 129), (129, 600), (600, 700))]
    assert np.array_equal(whole, np.concatenate(parts, axis=0))


def test_stream_statistics():
    f = streams.bf16_bits_to_f32_np
    spec = streams.StreamSpec("peaked", seed=1)
    k = f(streams.gen_tensor_np(spec, 0, 0, 0, streams.TENSOR_K, 0, 4096, 8, 128))
    q = f(streams.gen_tensor_np(spec, 0, 1, 0, streams.TENSOR_Q, 0, 512, 32, 128))
    assert abs(k.mean()) < 0.01 and abs(k.std() - 1.0) < 0.01 and np.abs(k).max() <= 3.5   # Irwin-Hall(4), unit var
    assert abs(q.std() - 3.0) < 0.05                                                     # Q ~ N(0, 3^2)
    spec = streams.StreamSpec("needle", seed=1, needles=(10,))
    kn = f(streams.gen_tensor_np(spec, 0, 0, 0, streams.TENSOR_K, 0, 64, 8, 128))
    assert abs(np.linalg.norm(kn[10, 0]) - spec.gamma) < 0.2 * spec.gamma                 # the needle key
    assert np.linalg.norm(kn[11, 0]) < 2.0                                               # background ~ 0.1 N(0,1)
