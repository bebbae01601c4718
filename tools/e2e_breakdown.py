"""Where the end-to-end time of one config-1 call goes (host layers vs device):
    python tools/e2e_breakdown.py"""
import statistics
import sys
import time

sys.path.insert(0, '.')
import ctypes  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_11006_b200 import engine as E  # noqa: E402
from paper_2306_11006_b200.cggi import PARAM_128, GateKind, encrypt_bits, eval_gate_batch, keygen  # noqa: E402
from paper_2306_11006_b200.rng import SeededRng  # noqa: E402

ks = keygen(PARAM_128, seed=7)
ek = ks.eval_key()
eng = ek.engine()
rng = np.random.default_rng(0)
A = encrypt_bits(PARAM_128, ks.lwe_sk, rng.integers(0, 2, 256).astype(np.uint8), SeededRng(1))
B = encrypt_bits(PARAM_128, ks.lwe_sk, rng.integers(0, 2, 256).astype(np.uint8), SeededRng(2))
pa = torch.from_numpy(A.view(np.int32)).pin_memory().numpy().view(np.uint32)
pb = torch.from_numpy(B.view(np.int32)).pin_memory().numpy().view(np.uint32)
out = torch.empty((256, PARAM_128.n + 1), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
nand = E.OPCODES["NAND"]
for _ in range(5):
    eval_gate_batch(GateKind.NAND, [pa, pb], ek)


def timed(fn, n=40):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e6


arr = (E._P * 2)(E._addr(pa), E._addr(pb))
res = {
    "cggi.eval_gate_batch": timed(lambda: eval_gate_batch(GateKind.NAND, [pa, pb], ek)),
    "Engine.eval_gate_batch": timed(lambda: eng.eval_gate_batch(nand, [pa, pb], 256)),
    "C gw_eval_gate_batch (ctypes)": timed(lambda: eng._lib.gw_eval_gate_batch(eng._ctx, nand, arr, 2, 256, E._addr(out))),
}
eng.set_profiling(True)
eng.stage_times(reset=True)
for _ in range(20):
    eng._lib.gw_eval_gate_batch(eng._ctx, nand, arr, 2, 256, E._addr(out))
st = eng.stage_times(reset=True)
eng.set_profiling(False)
res["device kernels (sum of stages)"] = sum(v[0] for v in st.values()) / 20 * 1e3
for k, v in res.items():
    print(f"{k:40s} {v:9.1f} us")
