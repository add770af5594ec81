"""bench.py's reference arm (the fp64 oracle, this tier's baseline) prints the contract's
JSON line on CPU: same metric / unit / config as our arm, impl "reference", a cpu_baseline
and an e2e object with zero copies.  The oracle sample is shrunk so the test is quick."""
import io
import json
import sys
from contextlib import redirect_stdout

import bench


def test_reference_arm_line(monkeypatch):
    real = bench.oracle_query_sample
    monkeypatch.setattr(bench, "oracle_query_sample", lambda n=None, **kw: real(n=2048))
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--steps", "2", "--warmup", "3"])
    buf = io.StringIO()
    with redirect_stdout(buf):
        bench.main()
    line = json.loads(buf.getvalue().strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["unit"] == "GB/s" and line["higher_is_better"] is True
    assert line["config"] == bench.arm_config()
    assert line["steps"] == 2 and line["warmup"] >= 3 and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_algorithmic_counts():
    # 134,873,088 B per query layer at n = 32,768, |q| = 32; 1.369e11 FLOP per append layer
    assert bench.query_bytes_per_layer(32768, 32, 32, 8, 128) == 134873088
    assert bench.append_flops_per_layer(32512, 256, 32, 128) == 4 * 32 * 128 * (256 * 32512 + 256 * 257 // 2)
    assert abs(bench.append_flops_per_layer(32512, 256, 32, 128) - 1.369e11) < 1e9
