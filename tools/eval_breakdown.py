"""Host-side breakdown of runtime.evaluate for config 2's netlists: where the
wall time goes besides the device levels (wire store, plan, copies)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2306_11006_b200 import circuit as C  # noqa: E402
from paper_2306_11006_b200 import netlists as NL  # noqa: E402
from paper_2306_11006_b200 import runtime as RT  # noqa: E402
from paper_2306_11006_b200.cggi import PARAM_128, encrypt_bits, keygen  # noqa: E402
from paper_2306_11006_b200.rng import SeededRng  # noqa: E402
from paper_2306_11006_b200.scheduler import build_schedule  # noqa: E402

ks = keygen(PARAM_128, 7)
ek = ks.eval_key()
eng = ek.engine()
rng = np.random.default_rng(80)
for name, c in (("adder8", C.gen_adder(8)), ("multiplier8", NL.gen_multiplier(8))):
    vals = {p.name: int(rng.integers(0, 1 << p.width)) for p in c.inputs}
    srng = SeededRng(8000)
    inputs = {p.name: encrypt_bits(PARAM_128, ks.lwe_sk, C.value_to_bits(vals[p.name], p.width), srng)
              for p in c.inputs}
    sched = build_schedule(c, 1)
    RT.evaluate(c, sched, inputs, ks)
    for rep in range(3):
        T = {}
        t = time.perf_counter()
        mats = RT.check_inputs(c, inputs, PARAM_128.n); T["check"] = time.perf_counter() - t
        t = time.perf_counter(); plan = RT._cached_plan(c, sched); T["plan_cache"] = time.perf_counter() - t
        with eng._mtx:
            t = time.perf_counter(); eng.wires_alloc(c.max_wire + 1); T["wires_alloc"] = time.perf_counter() - t
            t = time.perf_counter()
            for port in c.inputs:
                eng.wires_put(np.asarray(port.wires, np.int64), mats[port.name])
            T["wires_put"] = time.perf_counter() - t
            t = time.perf_counter()
            h = eng.plan_create(plan.level_offsets, plan.opcodes, plan.operands, plan.out_ids)
            T["plan_create"] = time.perf_counter() - t
            t = time.perf_counter(); ms = h.run_timed(0, len(sched.waves)); T["run"] = time.perf_counter() - t
            t = time.perf_counter(); h.close(); T["plan_close"] = time.perf_counter() - t
            t = time.perf_counter()
            outs = {p.name: eng.wires_get(np.asarray(p.wires, np.int64)) for p in c.outputs}
            T["wires_get"] = time.perf_counter() - t
            t = time.perf_counter(); eng.wires_alloc(0); T["wires_free"] = time.perf_counter() - t
        t = time.perf_counter(); RT.evaluate(c, sched, inputs, ks); T["evaluate_total"] = time.perf_counter() - t
        print(name, f"device {sum(ms):.2f} ms over {len(ms)} levels;",
              " ".join(f"{k}={v * 1e3:.2f}ms" for k, v in T.items()))
