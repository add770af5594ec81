#!/usr/bin/env python
"""Hottest SASS lines of an `ncu --page source --csv --print-source sass` export
(first kernel block): warp-stall samples per instruction and the top reasons."""
import csv, sys
path = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; blocks.append(cur); continue
    if r and r[0] == "Address":
        cur["hdr"] = r; continue
    if cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
        cur["rows"].append(dict(zip(cur["hdr"], r)))
b = blocks[int(sys.argv[3]) if len(sys.argv) > 3 else 0]
stalls = [h for h in b["hdr"] if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in b["rows"])
agg = {s: sum(int(x[s] or 0) for x in b["rows"]) for s in stalls}
print("total samples", tot, " by reason:", ", ".join(f"{k[6:]} {v/tot:.1%}" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))
rs = sorted(enumerate(b["rows"]), key=lambda ix: -int(ix[1]["Warp Stall Sampling (All Samples)"] or 0))
for i, x in rs[:top]:
    n = int(x["Warp Stall Sampling (All Samples)"] or 0)
    why = sorted(((int(x[s] or 0), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"{i:5d} {n/tot:6.2%} {x['Source'].strip()[:70]:70s} " + " ".join(f"{w}:{c}" for c, w in why if c))
