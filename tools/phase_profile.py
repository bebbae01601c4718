"""Per-phase cycle breakdown of the TMEM blind rotation (GATEWAVE_BR_PROFILE=1; for v5 at
1 or 3 gates per SM build with -DGW_V5_PHASE_PROF=1, e.g. tools/build_variant.py)."""
import os
import sys

os.environ["GATEWAVE_BR_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2306_11006_b200.cggi import PARAM_128, keygen  # noqa: E402

gates = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ks = keygen(PARAM_128, 7)
eng = ks.eval_key().engine()
rng = np.random.default_rng(0)
lin = rng.integers(0, 2 ** 32, (gates, PARAM_128.n + 1), dtype=np.uint32)
tv = np.zeros((2, PARAM_128.N), np.uint32)
tv[1] = PARAM_128.mu
eng.blind_rotate(lin, tv)
eng.blind_rotate(lin, tv)
cyc = eng.br_phase_cycles()
names = ["F", "wait B1", "M", "wait B2", "I", "wait B3"]  # br_v3.cuh phase marks
tot = sum(cyc[0])
print(f"gates={gates}: cycles per step (warp o of gate 0), total {tot / PARAM_128.n:.0f}")
for w in range(4):
    print(f"  warp {w}: " + "  ".join(f"{n}={c / PARAM_128.n:7.0f}" for n, c in zip(names, cyc[w])))
