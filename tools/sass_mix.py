"""Instruction mix + stall samples by SASS opcode from an ncu source-page CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass)."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ie, ss = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
cnt, smp = defaultdict(float), defaultdict(float)
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    op = r[1].strip().split()
    if not op:
        continue
    o = op[0] if not op[0].startswith("@") else op[1]
    o = o.split(".")[0]
    cnt[o] += float(r[ie] or 0)
    smp[o] += float(r[ss] or 0)
tot, tots = sum(cnt.values()), sum(smp.values())
print(f"total warp-instr {tot:.4g}")
for o, c in sorted(cnt.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"  {o:10s} {c:12.4g} {100 * c / tot:6.2f}%   stall-samples {100 * smp[o] / tots:6.2f}%")
