"""One blind rotation of G random samples (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2306_11006_b200.cggi import PARAM_128, keygen  # noqa: E402

gates = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ks = keygen(PARAM_128, 7)
eng = ks.eval_key().engine()
lin = np.random.default_rng(0).integers(0, 2 ** 32, (gates, PARAM_128.n + 1), dtype=np.uint32)
tv = np.zeros((2, PARAM_128.N), np.uint32)
tv[1] = PARAM_128.mu
for _ in range(2):
    eng.blind_rotate(lin, tv)
