"""Event-timed blind rotation (device-resident inputs) for several batch sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_11006_b200 import engine as E  # noqa: E402
from paper_2306_11006_b200.cggi import PARAM_128, keygen  # noqa: E402

ks = keygen(PARAM_128, 7)
ek = ks.eval_key()
eng = ek.engine()
P = PARAM_128
W = P.n + 1
Wp = (W + 3) & ~3
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
eng.set_stream(stream.cuda_stream)
nand = E.OPCODES["NAND"]
for G in [int(x) for x in (sys.argv[1:] or ["148", "256", "296", "444", "592", "1184"])]:
    rng = np.random.default_rng(G)
    ops = torch.from_numpy(rng.integers(0, 2 ** 32, (2 * G, Wp), dtype=np.uint32).view(np.int32)).cuda()
    out = torch.zeros((G, Wp), dtype=torch.int32, device="cuda")
    pa, pb = ops.data_ptr(), ops.data_ptr() + G * Wp * 4
    for _ in range(3):
        eng.eval_gate_batch_device(nand, [pa, pb], Wp, G, out.data_ptr(), Wp)
    torch.cuda.synchronize()
    eng.stage_times(reset=True)
    eng.set_profiling(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 5
    e0.record(stream)
    for _ in range(K):
        eng.eval_gate_batch_device(nand, [pa, pb], Wp, G, out.data_ptr(), Wp)
    e1.record(stream)
    torch.cuda.synchronize()
    eng.set_profiling(False)
    st = eng.stage_times(reset=True)
    ms = e0.elapsed_time(e1) / K
    br = st["blind_rotate"][0] / K
    print(f"G={G:5d}  step {ms:7.3f} ms  blind_rotate {br:7.3f} ms  -> {G / ms * 1e3:9.0f} gates/s"
          f"  ({br / P.n * 1e3:6.2f} us/step, {br * 1e-3 * 1.965e9 / P.n:7.0f} cyc/step)")
