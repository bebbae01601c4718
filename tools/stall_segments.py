"""Stall reasons per code segment (segments delimited by BAR.SYNC) from an ncu
source-page CSV: python tools/stall_segments.py X.csv [units_per_step]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ie = h.index("Instructions Executed")
reasons = [k for k in h if k.startswith("stall_") and "(Not Issued)" not in k]
idx = {k: h.index(k) for k in reasons}
segs, cur, start, n_inst = [], defaultdict(float), 0, 0.0
for i, r in enumerate(rows[2:]):
    if len(r) < len(h):
        continue
    s = r[1].strip()
    e = float(r[ie] or 0)
    n_inst += e
    for k in reasons:
        cur[k] += float(r[idx[k]] or 0)
    if s.startswith("BAR") and e > 0:
        segs.append((start, i, n_inst, dict(cur)))
        cur, start, n_inst = defaultdict(float), i + 1, 0.0
segs.append((start, len(rows), n_inst, dict(cur)))
tot = sum(sum(c.values()) for *_, c in segs)
for a, b, n, c in segs:
    t = sum(c.values())
    if t / tot < 0.01:
        continue
    top = sorted(c.items(), key=lambda x: -x[1])[:6]
    print(f"[{a:5d},{b:5d}) instr/unit {n / units:8.0f}  samples {100 * t / tot:5.1f}%  " +
          "  ".join(f"{k[6:]}={100 * v / t:.0f}%" for k, v in top))
