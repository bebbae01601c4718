"""Static SASS opcode histogram of one kernel: cuobjdump -sass LIB | this NAME_SUBSTR"""
import re
import sys
from collections import Counter

name = sys.argv[1]
txt = sys.stdin.read().split("Function : ")
for blk in txt[1:]:
    fn = blk.split("\n", 1)[0].strip()
    if name not in fn:
        continue
    c = Counter()
    for line in blk.split("\n"):
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            c[m.group(2)] += 1
    print(fn, sum(c.values()))
    print("  " + "  ".join(f"{k}:{v}" for k, v in c.most_common(30)))
