"""Stage breakdown (blind rotation / keyswitch / other kernels, CUDA events per
launch) of one netlist evaluation through runtime.evaluate:
    python tools/netlist_stages.py --config 3"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    args = ap.parse_args()
    import torch
    from netlist_run import build
    from paper_2306_11006_b200.cggi import PARAM_128, encrypt_bits, keygen
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import evaluate
    from paper_2306_11006_b200.scheduler import build_schedule
    ks = keygen(PARAM_128, seed=7)
    ek = ks.eval_key()
    eng = ek.engine()
    out = []
    for name, c, seed in build(args.config):
        rng = np.random.default_rng(seed)
        inputs = {p.name: encrypt_bits(PARAM_128, ks.lwe_sk, rng.integers(0, 2, p.width).astype(np.uint8),
                                       SeededRng(seed)) for p in c.inputs}
        sched = build_schedule(c, 1)
        evaluate(c, sched, inputs, ek)  # warm (plan compile, scratch)
        eng.stage_times(reset=True)
        eng.set_profiling(True)
        torch.cuda.synchronize()
        t = time.monotonic()
        _, met = evaluate(c, sched, inputs, ek)
        torch.cuda.synchronize()
        wall = time.monotonic() - t
        eng.set_profiling(False)
        st = eng.stage_times(reset=True)
        out.append({"netlist": name, "wall_s": wall, "device_s": met.device_time_seconds,
                    "stages_ms": {k: v[0] for k, v in st.items()},
                    "stage_items": {k: v[1] for k, v in st.items()}})
    print(json.dumps({"config": args.config, "results": out}))


if __name__ == "__main__":
    main()
