#!/usr/bin/env python
"""Benchmark of the stateful-session attention hot path on B200 (BASELINE.json).

Workload (BJ.configs[1]): Llama-3-8B-shaped attention (32 Q / 8 KV
heads, d=128, 32 layers, bf16, page size 64), one market-feed session at
n = 32,512 tokens.  One step = one pass of the whole hot path:
  1. data plane:  append D_k of 256 tokens over all 32 layers (ssa_session_append:
                  KV scatter into pages + chunked-prefill attention), n -> 32,768;
  2. query plane: a 32-token query over all 32 layers at n = 32,768
                  (ssa_session_query), no state change;
  3. SeqRemove(s, 32512, inf) (ssa_session_truncate, host metadata only) so every
     step sees the same context size.
Inputs are resident in HBM before the timed region; the per-step KV traffic
(4.3 GB over 32 layers) is larger than L2 (126 MB), so no flush is needed.

value = query-plane algorithmic HBM GB/s (134,873,088 B/layer x 32 layers per
query / device time of the query call); the JSON line also carries the append
prefill tok/s and TC utilisation, per-kernel rooflines, the fp64 oracle timed on
the host cores (cpu_baseline) and an end-to-end number through host buffers.

`--impl reference` times the fp64 CPU oracle (this tier's reference arm) on a
bounded sample of the same workload.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "query-plane attn latency & HBM GB/s at 32k ctx; append prefill tok/s & TC util"
CFG = dict(L=32, hq=32, hkv=8, d=128, P=64, n_ctx=32768, m_append=256, q_len=32)
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def query_bytes_per_layer(n, q, hq, hkv, d, elem=2):
    """Algorithmic bytes of one query-plane layer: cached K+V of n
    tokens, Q, own K/V, O."""
    return n * 2 * hkv * d * elem + q * hq * d * elem + q * 2 * hkv * d * elem + q * hq * d * elem


def append_flops_per_layer(n_cached, m, hq, d):
    """Algorithmic FLOPs of one data-plane layer: QK^T and PV, 2 FLOP/MAC,
    Hq*d*sum_i (n + i + 1) MACs each ("O(m*n)")."""
    return 4 * hq * d * (m * n_cached + m * (m + 1) // 2)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return dict(FALLBACK_PEAKS), "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ----------------------------------------------------------------------------- oracle legs
def oracle_query_sample(n=CFG["n_ctx"], kv_heads=1, q_len=CFG["q_len"]):
    """The fp64 oracle on a bounded sample of the workload: one layer, `kv_heads` KV
    heads (and their 4 q heads each), a 32-token query over n cached tokens.
    Returns (seconds, algorithmic bytes of the sample)."""
    import numpy as np
    import oracle
    import streams
    spec = streams.StreamSpec("market", seed=2)
    hq_s = kv_heads * (CFG["hq"] // CFG["hkv"])
    K = streams.gen_tensor_np(spec, 0, 0, 0, streams.TENSOR_K, 0, n, kv_heads, CFG["d"])
    V = streams.gen_tensor_np(spec, 0, 0, 0, streams.TENSOR_V, 0, n, kv_heads, CFG["d"])
    Q = streams.gen_tensor_np(spec, 0, 1, 0, streams.TENSOR_Q, 0, q_len, hq_s, CFG["d"])
    Kq = streams.gen_tensor_np(spec, 0, 1, 0, streams.TENSOR_K, 0, q_len, kv_heads, CFG["d"])
    Vq = streams.gen_tensor_np(spec, 0, 1, 0, streams.TENSOR_V, 0, q_len, kv_heads, CFG["d"])
    t0 = time.perf_counter()
    oracle.segment_rows(K, V, Q, Kq, Vq, kv_heads, oracle.default_scale(CFG["d"]))
    dt = time.perf_counter() - t0
    nbytes = query_bytes_per_layer(n, q_len, hq_s, kv_heads, CFG["d"])
    return dt, nbytes


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    oracle.build()
    for _ in range(args.warmup):
        oracle_query_sample(n=4096)
    times, nbytes = [], 0
    for _ in range(args.steps):
        dt, nbytes = oracle_query_sample()
        times.append(dt)
    v = nbytes / statistics.mean(times) / 1e9
    line = {"metric": METRIC, "value": v, "unit": "GB/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (streams.py market stream)",
            "config": {"workload": "llama3-8b-shape GQA 32/8 d128, 32-token query at n=32768 (1 layer, 1 KV head sample)"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": "fp64 C oracle: one layer, one KV head (4 q heads), 32-token query over 32,768 cached tokens, per step"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def build_session(st, torch, dev, spec, n, chunk=4096):
    """Bulk-import an n-token market-feed session (K/V generated on the GPU)."""
    import streams
    sid = None
    tok = 0
    while tok < n:
        m = min(chunk, n - tok)
        K = torch.stack([streams.gen_tensor_torch(spec, 0, 0, l, streams.TENSOR_K, tok, m, CFG["hkv"], CFG["d"],
                                                  device=dev) for l in range(CFG["L"])])
        V = torch.stack([streams.gen_tensor_torch(spec, 0, 0, l, streams.TENSOR_V, tok, m, CFG["hkv"], CFG["d"],
                                                  device=dev) for l in range(CFG["L"])])
        if sid is None:
            sid = st.session_create(None, K, V, n_prefix=m)   # R0 = first chunk (S)
        else:
            st.load_kv(sid, K, V)
        tok += m
    return sid


def gen_new(torch, dev, spec, domain, tok0, m):
    import streams
    out = []
    for t in (streams.TENSOR_Q, streams.TENSOR_K, streams.TENSOR_V):
        h = CFG["hq"] if t == streams.TENSOR_Q else CFG["hkv"]
        out.append(torch.stack([streams.gen_tensor_torch(spec, 0, domain, l, t, tok0, m, h, CFG["d"], hkv=CFG["hkv"],
                                                         device=dev) for l in range(CFG["L"])]).contiguous())
    return out


def run_ours(args):
    import torch
    import streams
    import paper_2605_13784_b200 as ssa

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    L, hq, hkv, d, P = CFG["L"], CFG["hq"], CFG["hkv"], CFG["d"], CFG["P"]
    n_ctx, m_app, q_len = CFG["n_ctx"], CFG["m_append"], CFG["q_len"]
    n0 = n_ctx - m_app
    num_pages = n_ctx // P + 16
    st = ssa.Store(L, hq, hkv, d, page_size=P, num_pages=num_pages, max_sessions=4, device=local, dtype="bf16")
    spec = streams.StreamSpec("market", seed=2 + rank)   # independent session per rank (weak scaling)
    sid = build_session(st, torch, dev, spec, n0)
    Qa, Ka, Va = gen_new(torch, dev, spec, 0, n0, m_app)
    Oa = torch.empty_like(Qa)
    Qq, Kq, Vq = gen_new(torch, dev, spec, 1, 0, q_len)
    Oq = torch.empty_like(Qq)
    stream = torch.cuda.current_stream()

    def step():
        st.session_append(sid, Qa, Ka, Va, Oa, stream=stream)
        st.session_query(sid, Qq, Kq, Vq, Oq, stream=stream)
        st.session_truncate(sid, n0)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    st.set_option(ssa.OPT_TIMING, 1)
    st.timing(reset=True)
    st.stats(reset=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev[0].record(stream)
        for _ in range(args.steps):
            step()
        ev[1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    step_ms = ev[0].elapsed_time(ev[1]) / args.steps
    tm = st.timing(reset=True)
    stats = st.stats()
    st.set_option(ssa.OPT_TIMING, 0)
    launches = stats["kernel_launches"]

    q_bytes = query_bytes_per_layer(n_ctx, q_len, hq, hkv, d) * L
    a_flops = append_flops_per_layer(n0, m_app, hq, d) * L
    attn_q_ms = tm["attn_query"][0] / max(1, tm["attn_query"][1])
    attn_a_ms = tm["attn_data"][0] / max(1, tm["attn_data"][1])
    comb_q_ms = tm["combine_query"][0] / args.steps
    comb_a_ms = tm["combine_data"][0] / args.steps
    scat_ms = tm["scatter"][0] / args.steps
    # query call = query attention + its combine; data call = scatter + attention + combine
    query_call_ms = attn_q_ms + comb_q_ms
    append_call_ms = attn_a_ms + scat_ms + comb_a_ms

    # max over ranks
    vals = torch.tensor([step_ms, query_call_ms, append_call_ms, attn_q_ms, attn_a_ms], device=dev, dtype=torch.float64)
    if world > 1:
        torch.distributed.all_reduce(vals, op=torch.distributed.ReduceOp.MAX)
    step_ms, query_call_ms, append_call_ms, attn_q_ms, attn_a_ms = vals.tolist()

    peaks, peak_src = load_peaks()
    hbm = peaks["hbm_gbs"]
    tc = peaks["bf16_tflops"]
    q_gbs = q_bytes / (query_call_ms * 1e-3) / 1e9
    kern_q_gbs = q_bytes / (attn_q_ms * 1e-3) / 1e9
    a_tflops = a_flops / (attn_a_ms * 1e-3) / 1e12
    append_tok_s = m_app / (append_call_ms * 1e-3)

    # ---- end-to-end through the C ABI with host (pinned) buffers
    hQ, hK, hV = (x.cpu().pin_memory() for x in (Qq, Kq, Vq))
    hO = torch.empty(Oq.shape, dtype=Oq.dtype).pin_memory()
    for _ in range(2):
        st.session_query(sid, hQ, hK, hV, hO, stream=stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        st.session_query(sid, hQ, hK, hV, hO, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    e2e_t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
    if world > 1:
        torch.distributed.all_reduce(e2e_t, op=torch.distributed.ReduceOp.MAX)
    e2e_ms = e2e_t.item()
    h2d = sum(x.numel() * x.element_size() for x in (hQ, hK, hV))
    d2h = hO.numel() * hO.element_size()

    line = None
    if rank == 0:
        clocks = clk.summary()
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get("attn_data_bytes_per_launch")
            except Exception:
                traffic = None
        dominant_is_append = attn_a_ms >= attn_q_ms
        roof_append = {"bound": "tensor", "achieved": a_tflops, "peak": tc, "unit": "TFLOP/s",
                       "frac": a_tflops / tc, "traffic": traffic,
                       "kernel": "data-plane attention (256-token append, 32 layers/launch)",
                       "peak_source": f"{peak_src} bf16_tflops (burst)"}
        roof_query = {"bound": "hbm", "achieved": kern_q_gbs, "peak": hbm, "unit": "GB/s",
                      "frac": kern_q_gbs / hbm, "traffic": None,
                      "kernel": "query-plane attention (32-token query, 32 layers/launch)",
                      "peak_source": f"{peak_src} hbm_gbs"}
        line = {
            "metric": METRIC, "value": q_gbs * world, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic market-feed stream (streams.py), random K/V/Q of Llama-3-8B attention shapes",
            "config": {"workload": "BJ.configs[1]: Llama-3-8B-shaped GQA 32/8 d=128 x 32 layers, one session at "
                                   "n=32,512 -> 256-token append -> 32-token query at n=32,768",
                       "page_size": P, "l2": "inputs larger than L2 (4.3 GB of KV read per step)",
                       "sessions_per_gpu": 1},
            "query_latency_us_32_layers": query_call_ms * 1e3,
            "query_latency_us_per_layer": query_call_ms * 1e3 / L,
            "query_hbm_gbs": q_gbs,
            "append_tok_per_s": append_tok_s * world,
            "append_tflops": a_tflops,
            "append_tc_util": a_tflops / tc,
            "kernel_ms": {"attn_data": attn_a_ms, "attn_query": attn_q_ms, "combine_data": comb_a_ms,
                          "combine_query": comb_q_ms, "scatter": scat_ms},
            "roofline": roof_append if dominant_is_append else roof_query,
            "roofline_query": roof_query,
            "roofline_append": roof_append,
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": {"value": q_bytes / (e2e_ms * 1e-3) / 1e9 * world, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_query": e2e_ms,
                    "what": "ssa_session_query with pinned host Q/K/V/O (H2D + kernels + D2H in the timed region)"},
            "paper_context": "paper: ~43 ms end-to-end standard query (full Llama-3.1-8B forward) on 1x L40S "
                             "(P:645, Table 1 P:672); not comparable to this attention-only path",
        }
        if not args.no_cpu_baseline:
            import oracle
            oracle.build()
            dt, nb = oracle_query_sample()
            line["cpu_baseline"] = {"value": nb / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
                                    "sample": "fp64 C oracle, single thread: one layer, one KV head (4 q heads), "
                                              f"32-token query over 32,768 cached tokens ({dt:.1f} s)"}
        print(json.dumps(line), flush=True)
    st.close()
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
