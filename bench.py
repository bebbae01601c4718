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
                FLOPs of the kernel that ran (v5: 171,008 n per bootstrap; the
                split-key v3 of exact mode: SURVEY.md §8(d)'s 249,856 n) / its
                live event-timed duration, vs the DFMA peak measured on this pool.
* cpu_baseline / --impl reference -- the UNMODIFIED reference (numba,
                pip-installed into baseline/_ref) through its own
                runtime.evaluate on all host cores ("reference"); the C
                restatement (oracle/, rebuilt -march=native for the host,
                "port") only when baseline/_ref cannot be imported.  Config-2
                CPU app latency is measured the same way; configs 3-5 are
                extrapolated from the measured per-bootstrap cost and the
                netlists' per-level bootstrap counts (labelled).
* --gpus N   -- one process per GPU: under torchrun (WORLD_SIZE must equal N)
                or, without it, bench.py re-launches itself under
                torch.distributed.run.  Besides the per-rank config-1 batches
                (weak scaling), N > 1 evaluates config 4 (and config 5 at N = 8)
                sharded by netlist level across the N GPUs with the NCCL
                point-to-point wire exchange, and reports its app latency,
                exchange bytes and an output digest that must not depend on N.
"""
from __future__ import annotations

import argparse
import gc
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
    ap.add_argument("--sharded-timeout", type=float, default=600.0,
                    help="deadline (s) for the sharded netlists at N > 1; on expiry the line is printed without them")
    ap.add_argument("--sharded", default="auto",
                    help="netlists evaluated sharded over the GPUs: auto (config4 at N>1, + config5 at "
                         "N=8), none, or a comma list of config4,config5,config3")
    ap.add_argument("--no-cpu-netlists", action="store_true")
    # test-only: exercise the N > 1 flow on a single-GPU box (every rank on GPU 0, gloo
    # process group, host-staged wire exchange) -- NCCL cannot put two ranks on one GPU
    ap.add_argument("--backend", choices=("nccl", "gloo"), default="nccl", help=argparse.SUPPRESS)
    ap.add_argument("--same-device", action="store_true", help=argparse.SUPPRESS)
    return ap.parse_args()


def config_dict(gates: int, n_gpus: int) -> dict:
    """The workload description both arms print (identical, so the driver can
    match them)."""
    return {"workload": f"config1: {gates} independent NAND gate bootstraps per GPU, "
                        "PARAM_128 (n=630, N=1024, l=2, Bg=2^9, t=8, gamma=2)",
            "gates_per_gpu": gates, "bootstraps_per_gate": 1,
            "l2": "flushed (512 MB write) between timed GPU steps",
            "parallelism": f"dp{n_gpus} (independent gate batches per GPU)"}


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


def _load_reference():
    """The unmodified reference package, pip-installed into baseline/_ref
    (DESIGN.md §6); None if it is not there."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "gatewave")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/gatewave_numba_cache")
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import gatewave.cggi  # noqa: F401
        import gatewave.circuit  # noqa: F401
        import gatewave.runtime  # noqa: F401
        import gatewave.scheduler  # noqa: F401
        return sys.modules["gatewave"]
    except Exception:
        return None


class CpuReference:
    """The reference's own CPU path on this host: `runtime.evaluate(c,
    build_schedule(c, K), inputs, keys)` with K = os.cpu_count() workers
    (BASELINE.md CPU-baseline plan).  Falls back to the oracle port (rebuilt
    -march=native here) when baseline/_ref cannot be imported."""

    def __init__(self, gates: int):
        from paper_2306_11006_b200.cggi import PARAM_128
        self.model, self.cores = _cpu_info()
        self.G = gates
        self.ks, self.A, self.B, _, _ = _workload(PARAM_128, 0, gates)
        self.ref = _load_reference()
        self.kind = "reference" if self.ref is not None else "port"
        if self.ref is not None:
            from gatewave import cggi as rc, circuit as rcirc, scheduler as rsch
            self.rc, self.rcirc, self.rsch = rc, rcirc, rsch
            from gatewave import runtime as rrt
            self.rrt = rrt
            self.rks = rc.keygen(rc.PARAM_128, seed=7)      # same bytes as ours (tests pin the digests)
            self.c1 = rcirc.gen_flat(gates, rc.GateKind.NAND)
            self.s1 = rsch.build_schedule(self.c1, self.cores)
        else:
            import oracle as O
            import oracle.oracle as OO
            OO.use_native()
            self.okeys = O.Keys.from_params(PARAM_128, self.ks.bootstrapping_key.data,
                                            self.ks.keyswitch_key.data)

    def step(self):
        """One full config-1 batch; returns (outputs, seconds)."""
        t0 = time.perf_counter()
        if self.ref is not None:
            outs, _ = self.rrt.evaluate(self.c1, self.s1, {"a": self.A, "b": self.B}, self.rks)
            out = outs["y"]
        else:
            import oracle as O
            out = O.eval_gate_batch("NAND", [self.A, self.B], self.okeys, threads=self.cores)
        return out, time.perf_counter() - t0

    def sample(self) -> str:
        if self.ref is not None:
            return (f"full config-1 batch ({self.G} NAND) per step through the unmodified reference "
                    f"(baseline/_ref gatewave.runtime.evaluate, K={self.cores} workers, numba JIT warm) "
                    f"on {self.model}")
        return (f"full config-1 batch ({self.G} NAND) per step; oracle/gw_oracle.c -march=native on "
                f"{self.cores} threads of {self.model} (baseline/_ref unavailable)")

    def config2(self, repeats: int = 3):
        """Config 2 app latency on the CPU: adder8 + 8x8 multiplier, median of
        `repeats` full runs each (reference runtime, K = cores)."""
        if self.ref is None:
            return None
        from paper_2306_11006_b200 import circuit as C
        from paper_2306_11006_b200 import netlists as NL
        from paper_2306_11006_b200.cggi import PARAM_128, encrypt_bits
        from paper_2306_11006_b200.rng import SeededRng
        res = {}
        rng = np.random.default_rng(80)
        for name, c in (("adder8", C.gen_adder(8)), ("multiplier8", NL.gen_multiplier(8))):
            vals = {p.name: int(rng.integers(0, 1 << p.width)) for p in c.inputs}
            srng = SeededRng(8000)
            inputs = {p.name: encrypt_bits(PARAM_128, self.ks.lwe_sk, C.value_to_bits(vals[p.name], p.width),
                                           srng) for p in c.inputs}
            rcirc = self.rcirc.parse_circuit(C.serialize_circuit(c))
            sched = self.rsch.build_schedule(rcirc, self.cores)
            lat = []
            for _ in range(repeats):
                t0 = time.perf_counter()
                self.rrt.evaluate(rcirc, sched, inputs, self.rks)
                lat.append(time.perf_counter() - t0)
            res[name] = {"app_latency_s": statistics.median(lat), "gates": len(c.gates), "repeats": repeats}
        res["total_app_latency_s"] = sum(v["app_latency_s"] for v in res.values())
        # the same two circuits as one netlist through the reference's own parser and runtime
        c = NL.merge_circuits([("add", C.gen_adder(8)), ("mul", NL.gen_multiplier(8))])
        vals = {p.name: int(rng.integers(0, 1 << p.width)) for p in c.inputs}
        srng = SeededRng(8100)
        inputs = {p.name: encrypt_bits(PARAM_128, self.ks.lwe_sk, C.value_to_bits(vals[p.name], p.width),
                                       srng) for p in c.inputs}
        rcirc = self.rcirc.parse_circuit(C.serialize_circuit(c))
        sched = self.rsch.build_schedule(rcirc, self.cores)
        lat = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            self.rrt.evaluate(rcirc, sched, inputs, self.rks)
            lat.append(time.perf_counter() - t0)
        res["combined_netlist"] = {"app_latency_s": statistics.median(lat), "gates": len(c.gates),
                                   "repeats": repeats}
        res["workers"] = self.cores
        return res

    def extrapolated_netlists(self, per_bootstrap_s: float):
        """Configs 3-5 on the CPU, EXTRAPOLATED: level L costs ceil(b_L / K)
        serial bootstraps of one worker, at the per-bootstrap time measured on
        this host (config-1 batch through the reference runtime)."""
        try:
            with open(os.path.join(ROOT, "tools", "level_profiles.json")) as f:
                prof = json.load(f)
        except OSError:
            return None
        out = {}
        K = self.cores
        for name, p in prof.items():
            if not name.startswith(("config3", "config4", "config5")):
                continue
            t = sum(-(-b // K) * per_bootstrap_s for b in p["bootstraps_per_level"])
            boots = sum(p["bootstraps_per_level"])
            out[name] = {"app_latency_s": t, "gates_per_s": p["gates"] / t, "bootstraps_per_s": boots / t,
                         "gates": p["gates"], "levels": p["levels"], "extrapolated": True}
        out["method"] = (f"extrapolated: sum over levels of ceil(bootstraps_L / K) x {per_bootstrap_s * 1e3:.1f} ms "
                         f"(one worker's per-bootstrap time, measured here on the config-1 batch), K = {K}; "
                         "level profiles from tools/level_profiles.json")
        return out


def run_reference(args):
    """Reference arm: the reference's own CPU implementation of the path on all
    host cores -- `runtime.evaluate(gen_flat(256, NAND), build_schedule(c, K))`
    with K = os.cpu_count() (BASELINE.md CPU-baseline plan), one full config-1
    batch per step.  Falls back to the oracle port if baseline/_ref is absent."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    cpu = CpuReference(args.gates)
    for _ in range(max(args.warmup, 1)):
        cpu.step()
    times = [cpu.step()[1] for _ in range(args.steps)]
    mean = statistics.mean(times)
    value = args.gates / mean
    line = {
        "impl": "reference", "metric": "bootstrapped gates/sec", "value": value, "unit": "gates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": mean * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64 (Goldilocks NTT)" if cpu.kind == "reference" else "u64 (port)",
        "data": "synthetic: keygen(PARAM_128, seed=7) + SURVEY Appendix A config-1 inputs",
        "config": config_dict(args.gates, args.gpus),
        "cpu_baseline": {"value": value, "unit": "gates/s", "cores": cpu.cores, "kind": cpu.kind,
                         "sample": cpu.sample()},
        "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def config2_latency(ks, P, eng, repeats: int = 5):
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
        lat, met, outs, phases = [], None, None, []
        for _ in range(repeats):
            gc.collect()          # a collection inside the timed call would be host noise, not the app
            gc.disable()
            try:
                t0 = time.perf_counter()
                outs, met = evaluate(c, sched, inputs, ks)
                lat.append(time.perf_counter() - t0)
            finally:
                gc.enable()
            phases.append({k: round(v, 6) for k, v in met.host_phases.items()})
        plain = C.simulate_plain(c, vals)
        ok = all(C.bits_to_value(decrypt_rows(ks.lwe_sk, outs[k])) == v for k, v in plain.items())
        res[name] = {"app_latency_s": statistics.median(lat), "gates": len(c.gates),
                     "bootstraps": met.bootstrap_count, "levels": len(sched.waves),
                     "device_time_s": met.device_time_seconds, "wall_runs_s": lat,
                     "evaluate_wall_s": met.wall_time_seconds, "host_phases_s": phases, "decrypt_ok": ok}
    res["total_app_latency_s"] = sum(v["app_latency_s"] for v in res.values())
    # the two circuits as ONE level-scheduled netlist (netlists.merge_circuits): their level-k
    # gates share each level's launch, so the evaluation takes as many levels as the deeper one
    c = NL.merge_circuits([("add", C.gen_adder(8)), ("mul", NL.gen_multiplier(8))])
    rng = np.random.default_rng(81)
    vals = {p.name: int(rng.integers(0, 1 << p.width)) for p in c.inputs}
    srng = SeededRng(8100)
    inputs = {p.name: encrypt_bits(P, ks.lwe_sk, C.value_to_bits(vals[p.name], p.width), srng)
              for p in c.inputs}
    sched = build_schedule(c, 1)
    evaluate(c, sched, inputs, ks)  # warm
    lat = []
    for _ in range(repeats):
        gc.collect()
        gc.disable()
        try:
            t0 = time.perf_counter()
            outs, met = evaluate(c, sched, inputs, ks)
            lat.append(time.perf_counter() - t0)
        finally:
            gc.enable()
    plain = C.simulate_plain(c, vals)
    ok = all(C.bits_to_value(decrypt_rows(ks.lwe_sk, outs[k])) == v for k, v in plain.items())
    res["combined_netlist"] = {"app_latency_s": statistics.median(lat), "gates": len(c.gates),
                               "levels": len(sched.waves), "device_time_s": met.device_time_seconds,
                               "wall_runs_s": lat, "decrypt_ok": ok,
                               "note": "adder8 and multiplier8 side by side in one netlist "
                                       "(netlists.merge_circuits), one level-scheduled evaluation"}
    return res


def run_ours(args):
    import torch
    ws, rank, local = _dist()
    if args.same_device:
        local = 0
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
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
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")
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
    # Algorithmic FP64 work per bootstrap, SURVEY.md §8(d) (the FP64 16-bit-split FFT path):
    # W_alg = n * 249,856 FLOP (4 fwd + 4 inv FFT-512 at 5 M log2 M, 16 x 512 complex MACs at
    # 8 FLOP) -- the figure `achieved` is defined on.  The FP64 work the kernel actually
    # executes is reported beside it (`frac_executed`):
    #   v5 (default, one key image): 4 fwd + 2 inv FFT-512 + 8 x 512 complex MACs = 171,008 per step
    #   v3 (exact mode, split key): 249,856 per step, the same as W_alg
    exact = eng.exact()
    flops_per_step = 249_856
    flops_per_bootstrap = flops_per_step * P.n
    executed_per_bootstrap = (249_856 if exact else 171_008) * P.n
    achieved = flops_per_bootstrap * br_items / (br_ms / 1e3) / 1e12 if br_ms > 0 else 0.0
    cidx = 64 if exact else 32                               # key complexes per TMEM lane and step
    bk_bytes = P.n * cidx * 128 * 16                         # FFT-domain key image, one pass
    # the kernel the engine launches for this batch (gw_api.cu launch_v5 / launch_v3: gates
    # per CTA minimising waves x measured step time)
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    if exact:
        step_kcyc = {1: 7.8, 2: 9.2, 3: 12.6, 4: 17.7}   # gw_api.cu launch_v3 policy
        gc = min(step_kcyc, key=lambda g: (-(-G // (sms * g)) * step_kcyc[g], g))
        kname = f"k_blind_rotate_v3<{gc}, {0 if gc == 4 else 2}, false>"
    else:
        step_kcyc = {1: 4.75, 2: 7.22, 3: 9.45}          # gw_api.cu launch_v5 policy
        gc = min(step_kcyc, key=lambda g: (-(-G // (sms * g)) * step_kcyc[g], g))
        kname = f"k_blind_rotate_v5<{gc}, false>"
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")) as f:
            t = json.load(f).get(kname)
        if t and t["gates"] == G:
            traffic = t["dram_bytes_read"] + t["dram_bytes_write"]
    except (OSError, ValueError, KeyError):
        pass
    roofline = {"bound": "fp64", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                "traffic_unit": "bytes per launch (ncu dram read+write, profiles/r02_ncu_traffic.json)",
                "kernel": kname,
                "per_launch_ms": br_ms / launches_br,
                "work_per_launch": f"{G} bootstraps x {flops_per_bootstrap} FLOP (SURVEY.md §8(d) W_alg = "
                                   f"n x 249,856)",
                "flop_count": "W_alg: 4 fwd + 4 inv FFT-512 + 16 x 512 complex MACs per step (SURVEY.md §8(d))",
                "executed_flop_count": ("v3 split key: 4 fwd + 4 inv FFT-512 + 16 x 512 complex MACs per step"
                                        if exact else
                                        "v5 one key image: 4 fwd + 2 inv FFT-512 + 8 x 512 complex MACs "
                                        "per step"),
                "frac_executed": executed_per_bootstrap * br_items / (br_ms / 1e3) / 1e12 / FP64_PEAK_TFLOPS
                if br_ms > 0 else 0.0,
                "kernel_share_of_step": br_ms / max(sum(step_ms), 1e-9),
                "keyswitch_ms_per_launch": ks_ms / launches_br,
                "bk_stream_gbs": bk_bytes / (br_ms / launches_br / 1e3) / 1e9,
                "peak_source": "measured DFMA peak, tools/microbench/pipes.cu "
                               "(profiles/r01_microbench_pipes.txt); not in MEASURED_PEAKS.json"}

    # ---- informational: the same batch in exact mode (split-key v3 kernel) -----
    exact_mode = None
    if not args.no_netlist and not eng.exact():
        eng.set_exact(True)
        try:
            for _ in range(2):
                step()
            torch.cuda.synchronize()
            res_x = out[:, :W].cpu().numpy().view(np.uint32)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(5):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
            xms = e0.elapsed_time(e1) / 5
            exact_mode = {"kernel": "k_blind_rotate_v3 (16-bit split key, provably exact rounding)",
                          "ms_per_step": xms, "gates_per_s": G / (xms / 1e3),
                          "outputs_equal_default_kernel": bool(np.array_equal(res_x, res)),
                          "note": "device-resident, L2 not flushed; gw_set_exact / GATEWAVE_BR_EXACT=1"}
        finally:
            eng.set_exact(False)

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
                "fp64_frac": flops_per_bootstrap * Gw / (wms / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
                "fp64_frac_executed": executed_per_bootstrap * Gw / (wms / 1e3) / 1e12 / FP64_PEAK_TFLOPS,
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

    # ---- CPU baseline: the unmodified reference, rank 0 at N=1 only ---------
    cpu = cpu_c2 = cpu_c345 = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        ref = CpuReference(G)
        ref.step()                                  # numba JIT warm (cached in NUMBA_CACHE_DIR)
        times, ref_out = [], None
        for _ in range(3):
            ref_out, dt = ref.step()
            times.append(dt)
        dt = statistics.median(times)
        cpu = {"value": G / dt, "unit": "gates/s", "cores": ref.cores, "kind": ref.kind,
               "sample": ref.sample() + f"; median of {len(times)} steps, {dt:.2f} s per step",
               "bit_exact_vs_gpu": bool(np.array_equal(ref_out, res))}
        if not args.no_cpu_netlists:
            # one worker's per-bootstrap time: each of the K workers ran ceil(G / K) bootstraps
            per_boot = dt / -(-G // ref.cores)
            cpu_c2 = ref.config2()
            cpu_c345 = ref.extrapolated_netlists(per_boot)

    if rank == 0:
        line = {
            "metric": "bootstrapped gates/sec", "value": value, "unit": "gates/s",
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: keygen(PARAM_128, seed=7) + SURVEY Appendix A config-1 inputs",
            "config": config_dict(G, ws),
            "e2e": {"value": G * ws / e2e_s, "unit": "gates/s",
                    "h2d_bytes_per_step": 2 * G * W * 4, "d2h_bytes_per_step": G * W * 4,
                    "app_latency_s": e2e_s, "api": "paper_2306_11006_b200.cggi.eval_gate_batch"},
            "gpu_launches": launches,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "app_latency_config2": netlist,
            "app_latency_config2_cpu": cpu_c2,
            "cpu_netlists_extrapolated": cpu_c345,
            "netlists_sharded": None,
            "throughput_wide_level": wide,
            "exact_mode": exact_mode,
            "param110": p110,
            "clocks": clk.summary(),
            "parity": parity,
        }
    # ---- netlists sharded over the GPUs (config 4; config 5 at N = 8) --------
    # Run last, under a deadline: a stuck collective must not cost the config-1 line.
    # On expiry rank 0 prints the line with the timeout recorded and every rank exits 0.
    which = []
    if not args.no_netlist and args.sharded != "none":
        which = ([] if ws == 1 else ["config4"] + (["config5"] if ws == 8 else [])) \
            if args.sharded == "auto" else [x for x in args.sharded.split(",") if x]
    if which:
        sharded = {}

        def _deadline():
            if rank == 0:
                sharded["error"] = f"timeout after {args.sharded_timeout:.0f} s (completed: {sorted(sharded)})"
                line["netlists_sharded"] = sharded
                print(json.dumps(line), flush=True)
            os._exit(0)

        timer = threading.Timer(args.sharded_timeout, _deadline)
        timer.daemon = True
        timer.start()
        for name in which:
            # a failure here must not cost the config-1 line: report it instead
            try:
                sharded[name] = netlist_sharded(name, ks, P, dist, rank, ws)
            except Exception as e:  # noqa: BLE001
                sharded[name] = {"error": f"{type(e).__name__}: {e}"[:500]}
        timer.cancel()
        if rank == 0:
            line["netlists_sharded"] = sharded
    if dist is not None:
        # Under NCCL_DEBUG=INFO NCCL logs each communicator's teardown to stdout: tear the
        # engines' and torch's communicators down first so the JSON line is the last line.
        from paper_2306_11006_b200 import engine as E
        E.clear_cache()
        dist.barrier()                  # every rank's engine communicator is gone
        dist.destroy_process_group()
        if rank == 0:
            time.sleep(1.0)             # the other ranks' process-group teardown logs land first
    if rank == 0:
        print(json.dumps(line), flush=True)
    return 0


NETLIST_SEEDS = {"config3": 3, "config4": 4, "config5": 5}


def netlist_sharded(name, ks, P, dist, rank, ws):
    """One BASELINE netlist config evaluated with its levels sharded over the
    ws GPUs (runtime.evaluate -> exchange.evaluate_distributed: the
    reference's per-opcode split of every level, scheduler.py:133-157, and the
    NCCL point-to-point wire exchange).  App latency = host rows in -> host
    rows out on every rank, max over ranks."""
    import hashlib
    import torch
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200 import netlists as NL
    from paper_2306_11006_b200.cggi import decrypt_rows, encrypt_bits
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import _cached_plan, evaluate
    from paper_2306_11006_b200.scheduler import bootstraps_of, build_schedule
    gen = {"config3": lambda: NL.gen_dot_product(500), "config4": lambda: NL.gen_fc_layer(256, 30),
           "config5": lambda: NL.gen_matmul_sigmoid(10)}[name]
    t = time.monotonic()
    c = gen()
    prep = {"generate_s": time.monotonic() - t}
    t = time.monotonic()
    sched = build_schedule(c, ws)
    prep["schedule_s"] = time.monotonic() - t
    t = time.monotonic()
    _cached_plan(c, sched, *((None, None) if ws == 1 else (rank, ws)))
    prep["plan_compile_s"] = time.monotonic() - t
    seed = NETLIST_SEEDS[name]
    rng = np.random.default_rng(seed)
    bits = {p.name: rng.integers(0, 2, p.width).astype(np.uint8) for p in c.inputs}
    srng = SeededRng(1000 * seed)
    inputs = {p.name: encrypt_bits(P, ks.lwe_sk, bits[p.name], srng) for p in c.inputs}
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.monotonic()
    outs, met = evaluate(c, sched, inputs, ks)
    torch.cuda.synchronize()
    app = time.monotonic() - t0
    if dist is not None:
        tl = torch.tensor([app], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tl, op=dist.ReduceOp.MAX)
        app = float(tl.item())
    h = hashlib.sha256()
    for p in c.outputs:
        h.update(np.ascontiguousarray(outs[p.name]).tobytes())
    ok = None
    if rank == 0:
        plain = C.simulate_plain_bits(c, {k: v[:, None] for k, v in bits.items()})
        ok = all(np.array_equal(decrypt_rows(ks.lwe_sk, outs[k]), plain[k][:, 0]) for k in plain)
    nb = bootstraps_of(sched)
    return {"gates": len(c.gates), "bootstraps": nb, "levels": len(sched.waves), "n_gpus": ws,
            "app_latency_s": app, "gates_per_s": len(c.gates) / app, "bootstraps_per_s": nb / app,
            "device_time_s": met.device_time_seconds,
            "exchange_bytes": getattr(met, "exchange_bytes", 0), "transport": getattr(met, "transport", "local"),
            "output_digest": h.hexdigest()[:16], "decrypt_ok": ok, "host_prep": prep,
            "seeds": f"default_rng({seed}) bits, SeededRng({1000 * seed}) encryption, keygen(PARAM_128, 7)"}


def _self_launch(args) -> int:
    """--gpus N without torchrun: re-run this script under torch.distributed.run
    (one process per GPU, 127.0.0.1 rendezvous), exactly as the driver does."""
    import socket
    import subprocess
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = _args()
    if args.impl == "reference":
        return run_reference(args)
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        return _self_launch(args)
    if int(ws_env or 1) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}: one process per GPU required\n")
        return 2
    if args.gpus > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # the driver checks the communicator's rank count
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
