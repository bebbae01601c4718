"""A few config-1 NAND batches (for ncu captures of the keyswitch kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2306_11006_b200.cggi import PARAM_128, GateKind, eval_gate_batch, keygen  # noqa: E402

gates = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ks = keygen(PARAM_128, 7)
ek = ks.eval_key()
rng = np.random.default_rng(0)
a = rng.integers(0, 2 ** 32, (gates, PARAM_128.n + 1), dtype=np.uint32)
b = rng.integers(0, 2 ** 32, (gates, PARAM_128.n + 1), dtype=np.uint32)
for _ in range(3):
    eval_gate_batch(GateKind.NAND, [a, b], ek)
