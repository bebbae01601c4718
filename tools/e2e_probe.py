"""e2e latency distribution of one config-1 batch through cggi.eval_gate_batch (pinned host
buffers), with and without an L2 flush before each call, plus the per-stage device time:
    python tools/e2e_probe.py"""
import sys, time, statistics
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2306_11006_b200.cggi import PARAM_128, GateKind, keygen, encrypt_bits, eval_gate_batch
from paper_2306_11006_b200.rng import SeededRng
ks = keygen(PARAM_128, seed=7); ek = ks.eval_key(); eng = ek.engine()
rng = np.random.default_rng(0)
A = encrypt_bits(PARAM_128, ks.lwe_sk, rng.integers(0, 2, 256).astype(np.uint8), SeededRng(1))
B = encrypt_bits(PARAM_128, ks.lwe_sk, rng.integers(0, 2, 256).astype(np.uint8), SeededRng(2))
pa = torch.from_numpy(A.view(np.int32)).pin_memory().numpy().view(np.uint32)
pb = torch.from_numpy(B.view(np.int32)).pin_memory().numpy().view(np.uint32)
for _ in range(5): eval_gate_batch(GateKind.NAND, [pa, pb], ek)
for label, flush in (("no flush", False), ("flush", True)):
    buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for _ in range(60):
        if flush: buf.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter(); eval_gate_batch(GateKind.NAND, [pa, pb], ek); ts.append(time.perf_counter() - t0)
    print(label, "mean %.1f us median %.1f min %.1f max %.1f" % tuple(x * 1e6 for x in (statistics.mean(ts), statistics.median(ts), min(ts), max(ts))))
# device-only pieces
eng.set_profiling(True); eng.stage_times(reset=True)
for _ in range(20): eval_gate_batch(GateKind.NAND, [pa, pb], ek)
st = eng.stage_times(reset=True); eng.set_profiling(False)
print({k: round(v[0] / 20 * 1e3, 1) for k, v in st.items()}, "us per call")
