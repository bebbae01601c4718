#!/usr/bin/env python
"""bench.py -- bootstrapped gates/s of the B200 CGGI engine (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (BASELINE.json configs[0], the config its metric is quoted on and the
CPU oracle runs): one step = one batch of 256 independent homomorphic NAND
gate bootstraps at the 128-bit parameter set (PARAM_128: n=630, N=1024,
Bg=2^9, l=2, t=8, gamma=2) with keygen(PARAM_128, seed=7) and the config-1
inputs of SURVEY.md Appendix A.  With N GPUs every rank evaluates its own
256-gate batch (independent gates: weak scaling, no data-path collective).

* value      -- whole-job gates/s with inputs resident in HBM, CUDA events on
                the engine stream around exactly K steps (L2 flushed between
                steps, outside the events), max over ranks.
* e2e        -- the same metric through the public API
                `cggi.eval_gate_batch(NAND, [A, B], ek)` with pinned host
                buffers: H2D of both operand matrices + D2H of the result
                inside the timed region (wall clock, max over ranks).
* roofline   -- the blind-rotation kernel against the FP64 pipe: algorithmic
                FLOPs (249,856 n per bootstrap) / its live
                event-timed duration, vs the DFMA peak measured on this pool.
* cpu_baseline / --impl reference -- the C restatement of the reference's
                algorithm (oracle/, "port") on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GATES = 256
CONFIG1_DIGEST = "6b796965e2579b67"
# tools/microbench/pipes.cu on this pool's B200 (profiles/r01_microbench_pipes.txt)
FP64_PEAK_TFLOPS = 37.05


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--gates", type=int, default=GATES)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-netlist", action="store_true")
    return ap.parse_args()


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cpu_info():
    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count() or 1


def _workload(params, rank: int, gates: int):
    from paper_2306_11006_b200.cggi import encrypt_bits, keygen
    from paper_2306_11006_b200.rng import SeededRng
    ks = keygen(params, seed=7)
    # SURVEY.md Appendix A; other ranks shift the plaintext seeds
    bits_a = np.random.default_rng(0 + 1000 * rank).integers(0, 2, gates)
    bits_b = np.random.default_rng(1 + 1000 * rank).integers(0, 2, gates)
    rng = SeededRng(1 + 1000 * rank)
    A = encrypt_bits(params, ks.lwe_sk, bits_a, rng)
    B = encrypt_bits(params, ks.lwe_sk, bits_b, rng)
    return ks, A, B, bits_a, bits_b


class ClockSampler:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self._nv is not None:
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


def cpu_oracle_run(params, ks, A, B, threads: int):
    """Time the oracle (C restatement of the reference path) on host cores."""
    import oracle as O
    keys = O.Keys.from_params(params, ks.bootstrapping_key.data, ks.keyswitch_key.data)
    t0 = time.perf_counter()
    out = O.eval_gate_batch("NAND", [A, B], keys, threads=threads)
    dt = time.perf_counter() - t0
    return out, dt


def _load_reference():
    """The unmodified reference package, pip-installed into baseline/_ref
    (DESIGN.md §6); None if it is not there."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "gatewave")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gatewave_numba_cache")
    sys.path.insert(0, path)
    try:
        import gatewave.cggi  # noqa: F401
        import gatewave.circuit  # noqa: F401
        import gatewave.runtime  # noqa: F401
        import gatewave.scheduler  # noqa: F401
        return sys.modules["gatewave"]
    except Exception:
        return None


def run_reference(args):
    """Reference arm: the reference's own CPU implementation of the path on all
    host cores -- `runtime.evaluate(gen_flat(256, NAND), build_schedule(c, K))`
    with K = os.cpu_count() (BASELINE.md CPU-baseline plan), one full config-1
    batch per step.  Falls back to the oracle port if baseline/_ref is absent."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    from paper_2306_11006_b200.cggi import PARAM_128
    model, cores = _cpu_info()
    ks, A, B, _, _ = _workload(PARAM_128, 0, args.gates)
    ref = _load_reference()
    if ref is not None:
        from gatewave import cggi as rc, circuit as rcirc, runtime as rrt, scheduler as rsch
        rks = rc.keygen(rc.PARAM_128, seed=7)       # same bytes as ours (tests pin the digests)
        c = rcirc.gen_flat(args.gates, rc.GateKind.NAND)
        sched = rsch.build_schedule(c, cores)
        inputs = {"a": A, "b": B}

        def step():
            t0 = time.perf_counter()
            outs, _ = rrt.evaluate(c, sched, inputs, rks)
            return outs["y"], time.perf_counter() - t0
        kind = "reference"
        sample = (f"full config-1 batch ({args.gates} NAND) per step through the unmodified "
                  f"reference (baseline/_ref gatewave.runtime.evaluate, K={cores} workers, "
                  f"numba JIT warm) on {model}")
    else:
        def step():
            return cpu_oracle_run(PARAM_128, ks, A, B, cores)
        kind = "port"
        sample = (f"full config-1 batch ({args.gates} NAND) per step; oracle/gw_oracle.c on "
                  f"{cores} threads of {model} (baseline/_ref unavailable)")
    for _ in range(max(args.warmup, 1)):
        step()
    times = [step()[1] for _ in range(args.steps)]
    mean = statistics.mean(times)
    value = args.gates / mean
    line = {
        "impl": "reference", "metric": "bootstrapped gates/sec", "value": value, "unit": "gates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64 (Goldilocks NTT)", "data": "synthetic",
        "config": {"workload": f"config1: {args.gates} independent NAND gate bootstraps per GPU, "
                               "PARAM_128 (n=630, N=1024, l=2, Bg=2^9, t=8, gamma=2)",
                   "gates_per_gpu": args.gates},
        "cpu_baseline": {"value": value, "unit": "gates/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config2_latency(ks, P, eng, repeats: int = 3):
    """BASELINE configs[1]: 8-bit ripple-carry adder + 8-bit multiplier,
    level-scheduled on one GPU through runtime.evaluate (host rows in, host
    rows out).  Returns app latency (median over repeats) and level shapes;
    decrypted outputs are checked against simulate_plain."""
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200 import netlists as NL
    from paper_2306_11006_b200.cggi import decrypt_rows, encrypt_bits
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import evaluate
    from paper_2306_11006_b200.scheduler import build_schedule
    res = {}
    rng = np.random.default_rng(80)
    for name, c in (("adder8", C.gen_adder(8)), ("multiplier8", NL.gen_multiplier(8))):
        vals = {p.name: int(rng.integers(0, 1 << p.width)) for p in c.inputs}
        srng = SeededRng(8000)
        inputs = {p.name: encrypt_bits(P, ks.lwe_sk, C.value_to_bits(vals[p.name], p.width), srng)
                  for p in c.inputs}
        sched = build_schedule(c, 1)
        evaluate(c, sched, inputs, ks)  # warm
        lat, met, outs = [], None, None
        for _ in range(repeats):
            t0 = time.perf_counter()
            outs, met = evaluate(c, sched, inputs, ks)
            lat.append(time.perf_counter() - t0)
        plain = C.simulate_plain(c, vals)
        ok = all(C.bits_to_value(decrypt_rows(ks.lwe_sk, outs[k])) == v for k, v in plain.items())
        res[name] = {"app_latency_s": statistics.median(lat), "gates": len(c.gates),
                     "bootstraps": met.bootstrap_count, "levels": len(sched.waves),
                     "device_time_s": met.device_time_seconds, "decrypt_ok": ok}
    res["total_app_latency_s"] = sum(v["app_latency_s"] for v in res.values())
    return res


def run_ours(args):
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
        torch.cuda.set_device(local)
    from paper_2306_11006_b200 import engine as E
    from paper_2306_11006_b200.cggi import PARAM_128, GateKind, eval_gate_batch

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    P = PARAM_128
    E.set_device(local)
    ks, A, B, bits_a, bits_b = _workload(P, rank, args.gates)
    ek = ks.eval_key()
    eng = ek.engine()
    # a dedicated (non-default) stream: the engine and the timing events share it
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    eng.set_stream(stream.cuda_stream)
    G = args.gates
    W = P.n + 1
    Wp = (W + 3) & ~3
    nand = E.OPCODES["NAND"]

    # device-resident operands (stacked a-rows then b-rows) and output
    ops = torch.zeros((2 * G, Wp), dtype=torch.int32, device="cuda")
    ops[:G, :W] = torch.from_numpy(A.view(np.int32))
    ops[G:, :W] = torch.from_numpy(B.view(np.int32))
    out = torch.zeros((G, Wp), dtype=torch.int32, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    pa, pb, po = ops.data_ptr(), ops.data_ptr() + G * Wp * 4, out.data_ptr()

    def step():
        eng.eval_gate_batch_device(nand, [pa, pb], Wp, G, po, Wp)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    res = out[:, :W].cpu().numpy().view(np.uint32)
    from paper_2306_11006_b200.cggi import decrypt_rows
    import hashlib
    parity = {"decrypt_ok": bool(np.array_equal(decrypt_rows(ks.lwe_sk, res),
                                                (1 - (bits_a & bits_b)).astype(np.uint8)))}
    if rank == 0 and G == GATES:
        parity["digest"] = hashlib.sha256(np.ascontiguousarray(res).tobytes()).hexdigest()[:16]
        parity["digest_ok"] = parity["digest"] == CONFIG1_DIGEST

    # ---- timed region: exactly K steps -----------------------------------
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    eng.stage_times(reset=True)
    eng.set_profiling(True)
    launches0 = eng.launch_count()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()                      # L2 flush, outside the events
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = eng.launch_count() - launches0
    eng.set_profiling(False)
    stages = eng.stage_times(reset=True)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = max_over_ranks(statistics.mean(step_ms))
    value = G * ws / (ms / 1e3)

    # ---- roofline of the dominant kernel (blind rotation) ------------------
    br_ms, br_items = stages["blind_rotate"]
    ks_ms, ks_items = stages["keyswitch"]
    launches_br = args.steps
    flops_per_bootstrap = 249_856 * P.n                      # SURVEY.md §8(d), FP64 path
    achieved = flops_per_bootstrap * br_items / (br_ms / 1e3) / 1e12 if br_ms > 0 else 0.0
    bk_bytes = P.n * 2 * (2 * P.l) * 2 * (P.N // 2) * 16    # FFT-domain key, one pass
    # the kernel the engine launches for this batch (gw_api.cu launch_v3: gates per CTA
    # minimising waves x measured step time; loader-warp key streaming below 4 per CTA)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    step_kcyc = {1: 7.8, 2: 9.6, 3: 12.6, 4: 17.7}   # gw_api.cu launch_v3 policy
    gc = min(step_kcyc, key=lambda g: (-(-G // (sms * g)) * step_kcyc[g], g))
    kname = f"k_blind_rotate_v3<{gc},{0 if gc == 4 else 2}>"
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")) as f:
            t = json.load(f).get(kname)
        if t and t["gates"] == G:
            traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
    except (OSError, ValueError, KeyError):
        pass
    roofline = {"bound": "fp64", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                "traffic_unit": "bytes per launch (ncu dram read+write, profiles/r01_ncu_traffic.json)",
                "kernel": kname,
                "per_launch_ms": br_ms / launches_br,
                "work_per_launch": f"{G} bootstraps x {flops_per_bootstrap} FLOP",
                "kernel_share_of_step": br_ms / max(sum(step_ms), 1e-9),
                "keyswitch_ms_per_launch": ks_ms / launches_br,
                "bk_stream_gbs": bk_bytes / (br_ms / launches_br / 1e3) / 1e9,
                "peak_source": "measured DFMA peak, tools/microbench/pipes.cu "
                               "(profiles/r01_microbench_pipes.txt); not in MEASURED_PEAKS.json"}

    # ---- informational: a wide level (12 x 148 gates, 3 per SM, 4 waves) -----
    wide = None
    if not args.no_netlist:
        Gw = 12 * torch.cuda.get_device_properties(local).multi_processor_count
        rng_w = np.random.default_rng(4242 + rank)
        opsw = torch.from_numpy(rng_w.integers(0, 2 ** 32, (2 * Gw, Wp), dtype=np.uint32).view(np.int32)).cuda()
        outw = torch.zeros((Gw, Wp), dtype=torch.int32, device="cuda")
        pw, qw = opsw.data_ptr(), opsw.data_ptr() + Gw * Wp * 4
        for _ in range(2):
            eng.eval_gate_batch_device(nand, [pw, qw], Wp, Gw, outw.data_ptr(), Wp)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(3):
            eng.eval_gate_batch_device(nand, [pw, qw], Wp, Gw, outw.data_ptr(), Wp)
        e1.record(stream)
        torch.cuda.synchronize()
        wms = e0.elapsed_time(e1) / 3
        wide = {"gates": Gw, "ms": wms, "gates_per_s": Gw / (wms / 1e3),
                "fp64_frac": 157_409_280 * Gw / (wms / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
                "note": "device-resident NAND batch, 3 gates per SM (the netlists' wide levels)"}
        del opsw, outw

    # ---- informational: the secondary parameter set (PARAM_110, n = 512) ----
    p110 = None
    if not args.no_netlist:
        from paper_2306_11006_b200.cggi import PARAM_110
        ks110, A110, B110, a110, b110 = _workload(PARAM_110, rank, G)
        ek110 = ks110.eval_key()
        e110 = ek110.engine()
        e110.set_stream(stream.cuda_stream)
        W1 = PARAM_110.n + 1
        Wp1 = (W1 + 3) & ~3
        ops1 = torch.zeros((2 * G, Wp1), dtype=torch.int32, device="cuda")
        ops1[:G, :W1] = torch.from_numpy(A110.view(np.int32))
        ops1[G:, :W1] = torch.from_numpy(B110.view(np.int32))
        out1 = torch.zeros((G, Wp1), dtype=torch.int32, device="cuda")
        q0, q1 = ops1.data_ptr(), ops1.data_ptr() + G * Wp1 * 4
        for _ in range(2):
            e110.eval_gate_batch_device(nand, [q0, q1], Wp1, G, out1.data_ptr(), Wp1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(5):
            e110.eval_gate_batch_device(nand, [q0, q1], Wp1, G, out1.data_ptr(), Wp1)
        e1.record(stream)
        torch.cuda.synchronize()
        pms = e0.elapsed_time(e1) / 5
        ok110 = bool(np.array_equal(decrypt_rows(ks110.lwe_sk, out1[:, :W1].cpu().numpy().view(np.uint32)),
                                    (1 - (a110 & b110)).astype(np.uint8)))
        p110 = {"params": "PARAM_110 (n=512)", "gates": G, "ms": pms, "gates_per_s": G / (pms / 1e3),
                "decrypt_ok": ok110}
        del ops1, out1

    # ---- end to end through the public API (pinned host buffers) ----------
    pa_h = torch.from_numpy(A.view(np.int32)).pin_memory().numpy().view(np.uint32)
    pb_h = torch.from_numpy(B.view(np.int32)).pin_memory().numpy().view(np.uint32)
    for _ in range(2):
        eval_gate_batch(GateKind.NAND, [pa_h, pb_h], ek)
    e2e_times = []
    barrier()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = eval_gate_batch(GateKind.NAND, [pa_h, pb_h], ek)
        e2e_times.append(time.perf_counter() - t0)
    barrier()
    e2e_s = max_over_ranks(statistics.mean(e2e_times))
    parity["e2e_matches_device"] = bool(np.array_equal(r, res))

    # ---- config 2 app latency: adder8 + 8-bit multiplier through evaluate() --
    # BASELINE configs[1] is a one-GPU latency workload: measured at N = 1 only
    netlist = None
    if not args.no_netlist and ws == 1:
        netlist = config2_latency(ks, P, eng)

    # ---- CPU baseline (oracle port), rank 0 at N=1 only --------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        model, cores = _cpu_info()
        ref_out, dt = cpu_oracle_run(P, ks, A, B, cores)
        cpu = {"value": G / dt, "unit": "gates/s", "cores": cores, "kind": "port",
               "sample": f"full config-1 batch ({G} NAND bootstraps), oracle/gw_oracle.c "
                         f"on {cores} threads of {model}; {dt:.2f} s",
               "bit_exact_vs_gpu": bool(np.array_equal(ref_out, res))}

    if rank == 0:
        line = {
            "metric": "bootstrapped gates/sec", "value": value, "unit": "gates/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: keygen(PARAM_128, seed=7) + SURVEY Appendix A config-1 inputs",
            "config": {"workload": f"config1: {G} independent NAND gate bootstraps per GPU, "
                                   "PARAM_128 (n=630, N=1024, l=2, Bg=2^9, t=8, gamma=2)",
                       "gates_per_gpu": G, "bootstraps_per_gate": 1,
                       "l2": "flushed (512 MB write) between timed steps",
                       "parallelism": f"dp{ws} (independent gate batches)"},
            "e2e": {"value": G * ws / e2e_s, "unit": "gates/s",
                    "h2d_bytes_per_step": 2 * G * W * 4, "d2h_bytes_per_step": G * W * 4,
                    "app_latency_s": e2e_s, "api": "paper_2306_11006_b200.cggi.eval_gate_batch"},
            "gpu_launches": launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "app_latency_config2": netlist,
            "throughput_wide_level": wide,
            "param110": p110,
            "clocks": clk.summary(),
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    args = _args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
