"""Config-2 app latency only (bench.config2_latency), one line: for same-box A/Bs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2306_11006_b200.cggi import PARAM_128, keygen  # noqa: E402

ks = keygen(PARAM_128, seed=7)
eng = ks.eval_key().engine()
r = bench.config2_latency(ks, PARAM_128, eng, repeats=5)
print("adder8 %.2f ms  multiplier8 %.2f ms  combined %.2f ms  (device %.2f / %.2f / %.2f)" % (
    1e3 * r["adder8"]["app_latency_s"], 1e3 * r["multiplier8"]["app_latency_s"],
    1e3 * r["combined_netlist"]["app_latency_s"], 1e3 * r["adder8"]["device_time_s"],
    1e3 * r["multiplier8"]["device_time_s"], 1e3 * r["combined_netlist"]["device_time_s"]))
