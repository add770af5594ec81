"""Pins for the oracle's fused-projection functions (reading
R-21): brute force, closed forms, the RoPE invariants, and an independent library
implementation (transformers' Llama rotary embedding).  CPU only."""
import math

import numpy as np
import pytest
import torch

import oracle


def test_round_bf16_special_cases():
    # exact values stay, ties go to the even significand, signs and scales carry
    x = np.array([1.0, 1 + 2**-8, 1 + 3 * 2**-8, 1 + 2**-8 + 2**-30, -2.5, 2.0**-100, 3.0 * 2**100])
    got = oracle.to_f64(oracle.round_bf16(x))
    want = np.array([1.0, 1.0, 1 + 2**-6, 1 + 2**-7, -2.5, 2.0**-100, 3.0 * 2**100])
    assert np.array_equal(got, want)


def test_round_bf16_matches_torch_on_fp32_inputs():
    # for fp32-representable inputs torch's fp32 -> bf16 cast is a single RNE
    rng = np.random.default_rng(7)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-20, 20, 100000))).astype(np.float32)
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(oracle.round_bf16(x.astype(np.float64)), want)


def test_projection_brute_force():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((3, 8))
    w = rng.standard_normal((6, 8))
    y = oracle.qkv_projection(x, w)
    for i in range(3):
        for o in range(6):
            acc = 0.0
            for k in range(8):
                acc += x[i, k] * w[o, k]
            assert abs(y[i, o] - acc) <= 1e-12 * (1 + abs(acc))


def test_projection_decodes_bf16_bits():
    x = np.array([[0x3F80, 0x4000]], dtype=np.uint16)        # [1, 2]
    w = np.array([[0x4040, 0xBF80], [0, 0x3F00]], dtype=np.uint16)   # [3, -1], [0, 0.5]
    assert np.array_equal(oracle.qkv_projection(x, w), np.array([[1.0, 1.0]]))


def test_rope_position_zero_is_identity():
    x = np.random.default_rng(2).standard_normal((1, 3, 16))
    assert np.array_equal(oracle.rope(x, [0], 10000.0), x)


def test_rope_closed_form_unit_vectors():
    # d = 4: pair (0, 2) turns at 1 rad/position, pair (1, 3) at theta^-1/2
    theta, p = 100.0, 3
    e0 = np.zeros((1, 1, 4)); e0[0, 0, 0] = 1
    e2 = np.zeros((1, 1, 4)); e2[0, 0, 2] = 1
    e1 = np.zeros((1, 1, 4)); e1[0, 0, 1] = 1
    assert np.allclose(oracle.rope(e0, [p], theta)[0, 0], [math.cos(p), 0, math.sin(p), 0], atol=1e-15)
    assert np.allclose(oracle.rope(e2, [p], theta)[0, 0], [-math.sin(p), 0, math.cos(p), 0], atol=1e-15)
    a = p * theta ** -0.5
    assert np.allclose(oracle.rope(e1, [p], theta)[0, 0], [0, math.cos(a), 0, math.sin(a)], atol=1e-15)


def test_rope_is_complex_rotation():
    # (x_j + i x_{j+d/2}) * exp(i pos theta^(-2j/d))
    rng = np.random.default_rng(3)
    d, theta = 8, 500000.0
    x = rng.standard_normal((5, 2, d))
    pos = np.array([0, 1, 7, 1000, 123456])
    got = oracle.rope(x, pos, theta)
    for i in range(5):
        for h in range(2):
            for j in range(d // 2):
                z = complex(x[i, h, j], x[i, h, j + d // 2]) * complex(
                    math.cos(pos[i] * theta ** (-2 * j / d)), math.sin(pos[i] * theta ** (-2 * j / d)))
                assert abs(got[i, h, j] - z.real) < 1e-12 and abs(got[i, h, j + d // 2] - z.imag) < 1e-12


def test_rope_invariants_norm_and_relative_position():
    rng = np.random.default_rng(4)
    d, theta = 128, 500000.0
    q = rng.standard_normal((1, 1, d))
    k = rng.standard_normal((1, 1, d))
    rq = oracle.rope(q, [17], theta)
    # per-pair norm preserved
    n0 = q[0, 0, :64] ** 2 + q[0, 0, 64:] ** 2
    n1 = rq[0, 0, :64] ** 2 + rq[0, 0, 64:] ** 2
    assert np.allclose(n0, n1, rtol=1e-13)
    # <R(p) q, R(s) k> depends on p - s only
    for p, s, t in [(17, 5, 1000), (0, 300, 31), (4096, 4095, 20000)]:
        a = np.dot(oracle.rope(q, [p], theta).ravel(), oracle.rope(k, [s], theta).ravel())
        b = np.dot(oracle.rope(q, [p + t], theta).ravel(), oracle.rope(k, [s + t], theta).ravel())
        assert abs(a - b) < 1e-9 * (1 + abs(a))


def test_rope_matches_transformers_llama():
    lm = pytest.importorskip("transformers.models.llama.modeling_llama")
    from transformers import LlamaConfig
    cfg = LlamaConfig(hidden_size=256, num_attention_heads=2, num_key_value_heads=1, head_dim=128,
                      rope_theta=500000.0, max_position_embeddings=4096)
    emb = lm.LlamaRotaryEmbedding(cfg)
    rng = np.random.default_rng(5)
    n = 6
    pos = np.array([0, 1, 2, 100, 999, 1000])
    q = rng.standard_normal((n, 2, 128))
    k = rng.standard_normal((n, 1, 128))
    x = torch.zeros(1, n, 128, dtype=torch.float64)
    cos, sin = emb(x, torch.from_numpy(pos)[None])
    qt = torch.from_numpy(q).permute(1, 0, 2)[None]      # [1, H, n, d]
    kt = torch.from_numpy(k).permute(1, 0, 2)[None]
    qr, kr = lm.apply_rotary_pos_emb(qt, kt, cos.double(), sin.double())
    # transformers builds inv_freq in fp32: angles agree to ~6e-8 * pos
    assert np.allclose(oracle.rope(q, pos, 500000.0), qr[0].permute(1, 0, 2).numpy(), atol=2e-4)
    assert np.allclose(oracle.rope(k, pos, 500000.0), kr[0].permute(1, 0, 2).numpy(), atol=2e-4)


def test_qkv_rope_splits_heads_in_weight_order():
    # W rows: Q heads, then K heads, then V heads; V is never rotated
    hq, hkv, d, hidden = 2, 1, 4, 3
    rng = np.random.default_rng(6)
    x = rng.standard_normal((2, hidden))
    w = rng.standard_normal(((hq + 2 * hkv) * d, hidden))
    q, k, v = oracle.qkv_rope(x, w, hq, hkv, d, pos0=5, theta=10.0)
    y = x @ w.T
    assert np.allclose(v.reshape(2, -1), y[:, (hq + hkv) * d:], atol=0)
    assert np.allclose(q, oracle.rope(y[:, : hq * d].reshape(2, hq, d), [5, 6], 10.0), atol=1e-15)
    assert np.allclose(k, oracle.rope(y[:, hq * d: (hq + hkv) * d].reshape(2, hkv, d), [5, 6], 10.0), atol=1e-15)
    q0, k0, _ = oracle.qkv_rope(x, w, hq, hkv, d, pos0=5, theta=0.0)
    assert np.allclose(q0.reshape(2, -1), y[:, : hq * d], atol=0)
