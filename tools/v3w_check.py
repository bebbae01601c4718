"""v3w (gate-interleaved warps) vs v3: bit-exact blind rotation and event-timed
step cost for several batch sizes.  Env GATEWAVE_BR_W selects the kernel in
NEW contexts, so each variant gets its own engine (different device)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2306_11006_b200 import engine as E  # noqa: E402
from paper_2306_11006_b200.cggi import PARAM_128, keygen  # noqa: E402

P = PARAM_128
ks = keygen(P, 7)
bk, ksk = ks.bootstrapping_key.data, ks.keyswitch_key.data
variants = [v for v in (sys.argv[1].split(";") if len(sys.argv) > 1 else ["", "2,1", "2,2", "3,1"])]
sizes = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["148", "256", "296", "444", "592"])]
W = P.n + 1
Wp = (W + 3) & ~3
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
engines = {}
for v in variants:
    if v:
        os.environ["GATEWAVE_BR_W"] = v
    else:
        os.environ.pop("GATEWAVE_BR_W", None)
    eng = E.Engine(*E.params_tuple(P), device=0)
    eng.upload_keys(bk, ksk)
    eng.set_stream(stream.cuda_stream)
    engines[v or "v3"] = eng
nand = E.OPCODES["NAND"]
for G in sizes:
    rng = np.random.default_rng(G)
    ops = torch.from_numpy(rng.integers(0, 2 ** 32, (2 * G, Wp), dtype=np.uint32).view(np.int32)).cuda()
    ref = None
    for name, eng in engines.items():
        out = torch.zeros((G, Wp), dtype=torch.int32, device="cuda")
        pa, pb = ops.data_ptr(), ops.data_ptr() + G * Wp * 4
        for _ in range(2):
            eng.eval_gate_batch_device(nand, [pa, pb], Wp, G, out.data_ptr(), Wp)
        torch.cuda.synchronize()
        res = out.cpu().numpy()
        same = "ref" if ref is None else ("bit-exact" if np.array_equal(res, ref) else "MISMATCH")
        if ref is None:
            ref = res
        eng.stage_times(reset=True)
        eng.set_profiling(True)
        K = 5
        for _ in range(K):
            eng.eval_gate_batch_device(nand, [pa, pb], Wp, G, out.data_ptr(), Wp)
        torch.cuda.synchronize()
        eng.set_profiling(False)
        st = eng.stage_times(reset=True)
        br = st["blind_rotate"][0] / K
        tot = sum(x[0] for x in st.values()) / K
        print(f"{name:5s} G={G:5d}  blind_rotate {br:7.3f} ms ({br * 1e-3 * 1.965e9 / P.n:7.0f} cyc/step)  "
              f"step {tot:7.3f} ms -> {G / tot * 1e3:9.0f} gates/s  {same}", flush=True)
