"""Steady-state statistics of an SSA_TRACE timeline (scripts/trace_run.py output)."""
import sys
import numpy as np
t = np.load(sys.argv[1]).astype(np.int64)
lo, hi = int(sys.argv[2]) if len(sys.argv) > 2 else 20, int(sys.argv[3]) if len(sys.argv) > 3 else 200
for c in range(t.shape[0]):
    n = hi - lo
    sm = [np.median(t[c, k, lo:hi, 1] - t[c, k, lo:hi, 0]) for k in (0, 1)]
    per = [np.median(np.diff(t[c, k, lo:hi, 0])) for k in (0, 1)]
    p2i = [np.median(t[c, 2 + k, lo:hi, 0] - t[c, k, lo:hi, 1]) for k in (0, 1)]
    iss = [np.median(t[c, 2 + k, lo + 1:hi + 1, 1] - t[c, 2 + k, lo:hi, 0]) for k in (0, 1)]
    s2s = [np.median(t[c, k, lo + 1:hi + 1, 0] - t[c, 2 + k, lo + 1:hi + 1, 1]) for k in (0, 1)]
    ov = np.median(np.minimum(t[c, 0, lo:hi, 1], t[c, 1, lo:hi, 1]) - np.maximum(t[c, 0, lo:hi, 0], t[c, 1, lo:hi, 0]))
    print(f"cta {c}: softmax {sm} period {per} P->issuer {p2i} issuer P->Scommit {iss} Scommit->Sseen {s2s} softmax overlap {ov}")
