"""Stall reasons of one kernel region from an ncu source-page CSV (--print-source sass):
    ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv
    python tools/ncu_stalls.py X.csv FIRST LAST [WINDOW]
FIRST/LAST: SASS row range (e.g. the compute-warp code, excluding the loader loop)."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
lo, hi = int(sys.argv[2]), int(sys.argv[3])
ie = h.index("Instructions Executed"); ns = h.index("Warp Stall Sampling (All Samples)")
reasons = [k for k in h if k.startswith("stall_") and "(Not Issued)" not in k]
idx = {k: h.index(k) for k in reasons}
data = []
for i, r in enumerate(rows[2:]):
    if len(r) < len(h) or not (lo <= i < hi): continue
    data.append((i, r[1].strip(), float(r[ie] or 0), float(r[ns] or 0), {k: float(r[idx[k]] or 0) for k in reasons}))
tot = sum(d[3] for d in data); ex = sum(d[2] for d in data)
print(f"region [{lo},{hi}): samples {tot:.0f}, executed warp-instr {ex:.0f}")
allr = defaultdict(float)
for d in data:
    for k, v in d[4].items(): allr[k] += v
print("by reason:", " ".join(f"{k[6:]}={100*v/tot:.1f}%" for k, v in sorted(allr.items(), key=lambda x: -x[1])[:12]))
byop = defaultdict(lambda: [0.0, 0.0, defaultdict(float)])
for i, s, e, samp, rs in data:
    t = s.split(); op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
    op = op.split(".")[0]
    byop[op][0] += samp; byop[op][1] += e
    for k, v in rs.items(): byop[op][2][k] += v
for op, (samp, e, rs) in sorted(byop.items(), key=lambda x: -x[1][0])[:22]:
    top = sorted(rs.items(), key=lambda x: -x[1])[:4]
    print(f"  {op:10s} {100*samp/tot:5.1f}%  exec {100*e/ex:5.1f}%  " + " ".join(f"{k[6:]}={100*v/max(samp,1):.0f}%" for k, v in top))
# windows of 50 instructions
print("windows:")
w = int(sys.argv[4]) if len(sys.argv) > 4 else 100
for s0 in range(lo, hi, w):
    seg = [d for d in data if s0 <= d[0] < s0 + w]
    st = sum(d[3] for d in seg)
    if st / tot < 0.015: continue
    rr = defaultdict(float)
    for d in seg:
        for k, v in d[4].items(): rr[k] += v
    top = sorted(rr.items(), key=lambda x: -x[1])[:4]
    ops = defaultdict(int)
    for d in seg:
        t = d[1].split(); op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?"); ops[op.split(".")[0]] += 1
    mix = " ".join(f"{k}:{v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:5])
    print(f"  [{s0:5d}+{w}] {100*st/tot:5.1f}%  " + " ".join(f"{k[6:]}={100*v/max(st,1):.0f}%" for k, v in top) + "   | " + mix)
