"""CPU-only checks of the boundary and the host logic (no GPU needed)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "ssa.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ssa_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    import paper_2605_13784_b200 as ssa
    out = subprocess.check_output(["nm", "-D", "--defined-only", ssa.LIB_PATH]).decode()
    exported = set(re.findall(r" T (ssa_\w+)", out))
    declared = _declared_symbols()
    assert len(declared) >= 30
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    for s in declared:
        assert hasattr(ssa.lib, s)


def test_library_is_sm100a_only():
    import paper_2605_13784_b200 as ssa
    out = subprocess.check_output(["cuobjdump", "--list-elf", ssa.LIB_PATH]).decode()
    assert "sm_100a" in out
    assert not re.search(r"sm_(8\d|9\d)\b", out)


def test_abi_version_and_status_strings():
    import paper_2605_13784_b200 as ssa
    assert ssa.lib.ssa_abi_version() == 3
    assert ssa.lib.ssa_status_str(-3) == b"SSA_ERR_POOL_EXHAUSTED"


def test_pool_bytes_matches_memory_model():
    """Eq. (memory) P:778-781 with the GQA KV width (reading R-13)."""
    import paper_2605_13784_b200 as ssa
    # 32k tokens of Llama-3-8B-shaped KV = 512 pages of 64 tokens per layer
    assert ssa.Store.pool_bytes(32, 32, 8, 128, 64, 512, "bf16") == 2 * 32 * 8 * 128 * 32768 * 2 == 4294967296
    assert ssa.Store.pool_bytes(1, 4, 4, 64, 16, 40, "fp32") == 2 * 1 * 4 * 64 * 640 * 4
    assert ssa.Store.pool_bytes(32, 32, 7, 128, 64, 512, "bf16") == 0      # Hkv must divide Hq
    assert ssa.Store.pool_bytes(32, 32, 8, 128, 48, 512, "bf16") == 0      # page size power of two
    # E4M3 KV (reading R-22): one byte per element -> 2 GiB at 32k; needs bf16, d=128, scales > 0
    e4 = dict(kv_format="e4m3", k_scale=1 / 16, v_scale=1 / 32)
    assert ssa.Store.pool_bytes(32, 32, 8, 128, 64, 512, "bf16", **e4) == 2147483648
    assert ssa.Store.pool_bytes(32, 32, 8, 64, 64, 512, "bf16", **e4) == 0
    assert ssa.Store.pool_bytes(32, 32, 8, 128, 64, 512, "fp32", **e4) == 0
    assert ssa.Store.pool_bytes(32, 32, 8, 128, 64, 512, "bf16", kv_format="e4m3", k_scale=0.0) == 0
    assert ssa.Store.pool_bytes(32, 32, 8, 128, 64, 512, "bf16", kv_format="e4m3", v_scale=float("inf")) == 0


def test_store_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2605_13784_b200 as ssa
    with pytest.raises(ssa.SsaError) as e:
        ssa.Store(1, 4, 4, 64, page_size=16, num_pages=8, dtype="fp32")
    assert e.value.name == "SSA_ERR_CUDA"


def _check_cover(units, seg_m, seg_slots, hkv, qt, bk):
    """Every (segment, q tile, kv head) covers its causal key tiles exactly once."""
    from collections import defaultdict
    cover = defaultdict(list)
    for (seg, kvh, tok0, ntok, lo, hi, group, split) in units:
        assert 0 <= lo <= hi
        cover[(seg, kvh, tok0, ntok)].append((split, lo, hi, group))
    expect = set()
    for s, (m, n) in enumerate(zip(seg_m, seg_slots)):
        for tok0 in range(0, m, qt):
            ntok = min(qt, m - tok0)
            for h in range(hkv):
                expect.add((s, h, tok0, ntok))
                parts = sorted(cover[(s, h, tok0, ntok)])
                tiles = -(-n // bk) + -(-(tok0 + ntok) // bk)
                assert [p[0] for p in parts] == list(range(len(parts)))
                assert parts[0][1] == 0 and parts[-1][2] == tiles
                for a, b in zip(parts[:-1], parts[1:]):
                    assert a[2] == b[1]
                groups = {p[3] for p in parts}
                assert len(groups) == 1 and ((len(parts) == 1) == (groups == {-1}))
    assert set(cover) == expect


@pytest.mark.parametrize("case", [
    ([32], [32768], 8, 32, 128, 1),           # config 2 query, one layer
    ([32], [32768], 8, 32, 128, 32),          # all 32 layers in one launch
    ([256], [32512], 8, 32, 128, 1),          # config 2 append
    ([1], [131072], 8, 32, 128, 1),           # config 5 1-token query
    ([32] * 64, [8192] * 64, 8, 32, 128, 1),  # config 4 flash batch
    ([37, 91, 5, 256, 1024], [0, 4096, 777, 16128, 0], 8, 8, 64, 2),   # varlen batch incl. stateless
    ([16], [640], 4, 32, 64, 1),              # config 1 toy
])
def test_planner_covers_every_key_tile_once(case):
    import paper_2605_13784_b200 as ssa
    seg_m, seg_slots, hkv, qt, bk, L = case
    units = ssa.debug_plan(seg_m, seg_slots, hkv, qt, bk, n_layers=L)
    _check_cover(units, seg_m, seg_slots, hkv, qt, bk)


def test_planner_fills_the_gpu_for_the_query():
    import paper_2605_13784_b200 as ssa
    units = ssa.debug_plan([32], [32768], 8, 32, 128, n_layers=1, num_sms=148, ctas_per_sm=2)
    assert 240 <= len(units) <= 296          # one wave of two-slot CTAs on 148 SMs
    units = ssa.debug_plan([32], [32768], 8, 32, 128, n_layers=1, num_sms=148, ctas_per_sm=2, max_splits=4)
    assert len(units) == 32


def test_planner_does_not_shred_heterogeneous_batches():
    """Config 3 (48 sessions + stateless prompts, 32 layers): enough CTAs already, so no splits."""
    import paper_2605_13784_b200 as ssa
    ns = [4096 + 256 * s for s in range(48)]
    seg_m = [256 if s % 2 == 0 else 32 for s in range(48)] + [1024] * 4
    units = ssa.debug_plan(seg_m, ns + [0] * 4, 8, 32, 128, n_layers=32, num_sms=148, ctas_per_sm=2)
    for u in units:
        if seg_m[u[0]] == 32:
            # a lone 32-token query (one q tile, private pool) is halved so its two key
            # ranges fill both softmax slots of one tcgen05 CTA
            assert u[6] >= 0 and u[7] in (0, 1)
        else:
            assert u[6] == -1          # appends and stateless prompts pair their own q tiles
    assert sum(1 for u in units if seg_m[u[0]] == 32) == 24 * 8 * 2
