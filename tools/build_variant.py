"""Compile the current csrc/ into variants/lib_<name>.so (A/B timing within one
gpurun call: GATEWAVE_B200_LIB=variants/lib_<name>.so python tools/br_time.py)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_11006_b200 import build as B  # noqa: E402

name = sys.argv[1]
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
out = os.path.join(ROOT, "variants", f"lib_{name}.so")
cmd = [B.nvcc(), *B.ARCH, *B.FLAGS, *sys.argv[2:], "-o", out, os.path.join(B.CSRC, "gw_api.cu")]
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stdout + r.stderr)
    sys.exit(1)
print(out)
