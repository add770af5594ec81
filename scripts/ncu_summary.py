#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the files gpurun brought back).

    python scripts/ncu_summary.py raw  <raw.csv>  [--traffic profiles/traffic.json]
    python scripts/ncu_summary.py launches <launches.csv> [--slice a:b]

`raw` reads an `ncu -i rep --page raw --csv` export (one row per profiled launch) and
prints duration, DRAM bytes, tensor-pipe / XU / issue utilisation per launch.  With
--traffic it writes dram__bytes_read.sum + dram__bytes_write.sum of launch 0 (the
data-plane append launch of the bench step) and launch 1 (the query launch) as the
`traffic` figure bench.py reports beside the roofline.
`launches` aggregates an `ncu --metrics gpu__time_duration.sum --csv` launch list by
kernel name (count, mean, share of the total time)."""
import collections
import csv
import json
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "s": 1.0, "second": 1.0}

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor_%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu_%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma_%"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu_%"),
    ("sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active", "tmem_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clk"),
    ("launch__grid_size", "grid"),
    ("launch__registers_per_thread", "regs"),
]


def read_raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = {}
        for full, short in METRICS:
            for i, h in enumerate(hdr):
                if h == full or h.endswith("." + full) or h.split(".", 1)[-1] == full:
                    try:
                        v = float(r[i].replace(",", ""))
                    except ValueError:
                        continue
                    d[short] = v * UNITS.get(units[i], 1.0)
                    break
        for i, h in enumerate(hdr):
            if h == "Kernel Name":
                d["kernel"] = r[i][:60]
        out.append(d)
    return out


def cmd_raw(path, traffic_path=None):
    launches = read_raw(path)
    for i, d in enumerate(launches):
        parts = [f"launch {i}: {d.get('kernel', '?')}"]
        if "duration" in d:
            parts.append(f"{d['duration'] * 1e3:.3f} ms")
        if "dram_read" in d:
            parts.append(f"DRAM r {d['dram_read'] / 1e9:.3f} GB w {d.get('dram_write', 0) / 1e9:.3f} GB")
        for k in ("dram_%peak", "tensor_%", "xu_%", "fma_%", "alu_%", "tmem_%", "issue_%"):
            if k in d:
                parts.append(f"{k} {d[k]:.1f}")
        if "sm_clk" in d:
            parts.append(f"clk {d['sm_clk'] / 1e6:.0f} MHz")
        print(" | ".join(parts))
    if traffic_path and launches:
        t = {"source": path, "note": "dram__bytes_read.sum + dram__bytes_write.sum per launch (ncu --set full)"}
        names = ["attn_data_bytes_per_launch", "attn_query_bytes_per_launch"]
        for i, name in enumerate(names):
            if i < len(launches) and "dram_read" in launches[i]:
                t[name] = launches[i]["dram_read"] + launches[i].get("dram_write", 0.0)
        json.dump(t, open(traffic_path, "w"), indent=1)
        print("wrote", traffic_path)


def cmd_launches(path, sl=None):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(list)
    if sl:
        a, b = (int(x) for x in sl.split(":"))
        data = data[a:b]      # the launches of the timed steps
        for d in data:
            print("  ", d["Kernel Name"].split("(")[0].split("::")[-1], d["Metric Value"], d["Metric Unit"])
    for d in data:
        name = d["Kernel Name"].split("(")[0].split("::")[-1]
        agg[name].append(float(d["Metric Value"].replace(",", "")) * UNITS.get(d["Metric Unit"], 1.0))
    tot = sum(sum(v) for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:32s} n={len(v):4d} mean {sum(v) / len(v) * 1e6:10.1f} us  share {sum(v) / tot:6.1%}")


if __name__ == "__main__":
    if sys.argv[1] == "raw":
        tp = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
        cmd_raw(sys.argv[2], tp)
    else:
        cmd_launches(sys.argv[2], sys.argv[sys.argv.index("--slice") + 1] if "--slice" in sys.argv else None)
