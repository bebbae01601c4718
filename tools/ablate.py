"""Timing ablations of the TMEM blind rotation (debug; results are NOT exact
when any ablation bit is set).  1 = no decomposition, 2 = no MAC, 4 = no key
streaming, 8 = no accumulator atomics, 16 = no forward FFT, 32 = no inverse FFT."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2306_11006_b200 import engine as E  # noqa: E402
from paper_2306_11006_b200.cggi import PARAM_128, keygen  # noqa: E402

gates = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ks = keygen(PARAM_128, 7)
rng = np.random.default_rng(0)
lin = rng.integers(0, 2 ** 32, (gates, PARAM_128.n + 1), dtype=np.uint32)
tv = np.zeros((2, PARAM_128.N), np.uint32)
tv[1] = PARAM_128.mu
base = None
for ab in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else "0,1,2,4,8,16,32,48,15,63".split(","))]:
    os.environ["GATEWAVE_BR_ABLATE"] = str(ab)
    eng = E.Engine(*E.params_tuple(PARAM_128))
    eng.upload_keys(ks.bootstrapping_key.data, None)
    eng.blind_rotate(lin, tv)
    ts = []
    for _ in range(3):
        eng.timer_start()
        eng.blind_rotate(lin, tv)
        ts.append(eng.timer_stop())
    t = min(ts)
    base = base or t
    print(f"gates={gates} ablate={ab:3d}  {t:7.3f} ms  (saves {base - t:6.3f} ms, {100 * (base - t) / base:5.1f}%)")
    eng.close()
