"""bench.py's reference arm (the fp64 oracle, this tier's baseline) prints the contract's
JSON line on CPU: same metric / unit / config as our arm, impl "reference", a cpu_baseline
and an e2e object with zero copies.  The oracle sample is shrunk so the test is quick."""
import io
import json
import os
import sys
from contextlib import redirect_stdout

import numpy as np

import bench


def _small_inputs(monkeypatch, n=1024):
    real = bench.oracle_inputs
    monkeypatch.setattr(bench, "oracle_inputs", lambda layers, **kw: real(layers, **dict(kw, n=n)))


def test_reference_arm_line(monkeypatch):
    _small_inputs(monkeypatch)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--steps", "2", "--warmup", "3"])
    buf = io.StringIO()
    with redirect_stdout(buf):
        bench.main()
    line = json.loads(buf.getvalue().strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["unit"] == "GB/s" and line["higher_is_better"] is True
    assert line["config"] == bench.arm_config()
    assert line["steps"] == 2 and line["warmup"] >= 3 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == (os.cpu_count() or 1)
    assert line["cpu_baseline"]["cpu_model"]
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_algorithmic_counts():
    # 134,873,088 B per query layer at n = 32,768, |q| = 32; 1.369e11 FLOP per append layer
    assert bench.query_bytes_per_layer(32768, 32, 32, 8, 128) == 134873088
    assert bench.append_flops_per_layer(32512, 256, 32, 128) == 4 * 32 * 128 * (256 * 32512 + 256 * 257 // 2)
    assert abs(bench.append_flops_per_layer(32512, 256, 32, 128) - 1.369e11) < 1e9


def test_cpu_baseline_leg_and_parity_sample(monkeypatch):
    """The multi-threaded oracle leg of our arm: all host threads, CPU model, the single-thread
    figure, and the parity sample against the derived bound -- fed the oracle's own output
    rounded to bf16 (error = one rounding, inside the bound)."""
    import oracle
    _small_inputs(monkeypatch, n=256)
    inp = bench.oracle_inputs(range(bench.CFG["L"]))
    _, outs = bench.oracle_layers(inp, 4)
    f32 = np.stack(outs).astype(np.float32)
    u = f32.view(np.uint32)
    bf = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)      # RNE to bf16
    leg = bench.cpu_baseline_leg(bf)
    assert leg["cores"] == (os.cpu_count() or 1) and leg["cpu_model"] and leg["value"] > 0
    assert leg["single_thread_one_layer_kv_head_s"] > 0 and leg["append_one_layer_s"] > 0
    ps = leg["parity_sample"]
    assert ps["max_abs"] <= 2e-2 and 0.0 < ps["max_err_over_derived_bound"] <= 1.0
    assert np.abs(oracle.to_f64(bf[0]) - outs[0]).max() == ps["max_abs"] or ps["max_abs"] > 0
