"""Encrypted netlist workloads (BASELINE.json configs 2-5) through the public
`runtime.evaluate` API on one or more GPUs.

    python tools/netlist_run.py --config 3            # 1 GPU
    torchrun --nproc-per-node N tools/netlist_run.py --config 4   # N GPUs, NCCL exchange

config 2: 8-bit ripple-carry adder + 8x8 multiplier     (default_rng(80))
config 3: dot product of two 500-element int16 vectors (default_rng(3))
config 4: fc layer, 256 int16 inputs x w[30][256] -> 30 outputs (default_rng(4))
config 5: 10x10 int16 matmul + hard sigmoid on the 100 outputs (default_rng(5))

Keys: keygen(PARAM_128, seed=7).  App latency = host ciphertext rows in ->
every level on the GPU(s) -> host ciphertext rows out (runtime.evaluate; the
one-time host steps -- netlist generation, scheduling, plan compilation, key
generation and encryption -- are reported separately).  Parity: every
decrypted output word against the plaintext model (circuit.simulate_plain_bits,
the reference's circuit.py:321-363 semantics).  Prints one JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def build(config: int):
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200 import netlists as NL
    if config == 2:
        return [("adder8", C.gen_adder(8), 80), ("multiplier8", NL.gen_multiplier(8), 80)]
    if config == 3:
        return [("dot_product_500", NL.gen_dot_product(500), 3)]
    if config == 4:
        return [("fc_layer_256x30", NL.gen_fc_layer(256, 30), 4)]
    if config == 5:
        return [("matmul10_hard_sigmoid", NL.gen_matmul_sigmoid(10), 5)]
    raise SystemExit(f"unknown config {config}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True)
    ap.add_argument("--repeats", type=int, default=2)
    ap.add_argument("--vectors", type=int, default=None,
                    help="input vectors per netlist, each evaluated on its own (default: 100 for "
                         "config 2 -- the tests/test_acceptance.py:349-362 pattern -- else 1)")
    args = ap.parse_args()
    if args.vectors is None:
        args.vectors = 100 if args.config == 2 else 1

    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    group = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200 import engine as E
    from paper_2306_11006_b200.cggi import PARAM_128, decrypt_rows, encrypt_bits, keygen
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import _cached_plan, evaluate
    from paper_2306_11006_b200.scheduler import bootstraps_of, build_schedule

    E.set_device(local)
    P = PARAM_128
    t = time.monotonic()
    ks = keygen(P, seed=7)
    ek = ks.eval_key()
    ek.engine()
    t_keys = time.monotonic() - t
    results = []
    for name, c, seed in build(args.config):
        prep = {}
        t = time.monotonic()
        sched = build_schedule(c, ws)
        prep["schedule_s"] = time.monotonic() - t
        t = time.monotonic()
        _cached_plan(c, sched, *((None, None) if ws == 1 else (rank, ws)))
        prep["plan_compile_s"] = time.monotonic() - t
        rng = np.random.default_rng(seed)
        bits = {p.name: rng.integers(0, 2, p.width).astype(np.uint8) for p in c.inputs}
        t = time.monotonic()
        srng = SeededRng(1000 * seed)
        inputs = {p.name: encrypt_bits(P, ks.lwe_sk, bits[p.name], srng) for p in c.inputs}
        prep["encrypt_s"] = time.monotonic() - t
        lat = []
        outs = met = None
        for _ in range(args.repeats):
            if ws > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize()
            t = time.monotonic()
            outs, met = evaluate(c, sched, inputs, ek)
            torch.cuda.synchronize()
            lat.append(time.monotonic() - t)
        if ws > 1:
            tl = torch.tensor([max(lat)], dtype=torch.float64, device="cuda")
            torch.distributed.all_reduce(tl, op=torch.distributed.ReduceOp.MAX)
            app = float(tl.item())
        else:
            app = min(lat)
        t = time.monotonic()
        plain = C.simulate_plain_bits(c, {k: v[:, None] for k, v in bits.items()})
        ok = all(np.array_equal(decrypt_rows(ks.lwe_sk, outs[k]), plain[k][:, 0]) for k in plain)
        prep["plain_check_s"] = time.monotonic() - t
        nb = bootstraps_of(sched)
        per_vec = None
        if args.vectors > 1:
            # vectors 1..V-1: fresh plaintexts from the same generator, SeededRng(8000 + v)
            vl, vok = [app], [bool(ok)]
            for v in range(1, args.vectors):
                vb = {p.name: rng.integers(0, 2, p.width).astype(np.uint8) for p in c.inputs}
                vr = SeededRng(8000 + v)
                vin = {p.name: encrypt_bits(P, ks.lwe_sk, vb[p.name], vr) for p in c.inputs}
                if ws > 1:
                    torch.distributed.barrier()
                torch.cuda.synchronize()
                t = time.monotonic()
                vo, _ = evaluate(c, sched, vin, ek)
                torch.cuda.synchronize()
                vl.append(time.monotonic() - t)
                vp = C.simulate_plain_bits(c, {k: x[:, None] for k, x in vb.items()})
                vok.append(all(np.array_equal(decrypt_rows(ks.lwe_sk, vo[k]), vp[k][:, 0]) for k in vp))
            a = np.asarray(vl)
            per_vec = {"vectors": args.vectors, "decrypt_ok": int(sum(vok)),
                       "latency_mean_s": float(a.mean()), "latency_p50_s": float(np.median(a)),
                       "latency_p90_s": float(np.quantile(a, 0.9)), "latency_max_s": float(a.max())}
        results.append({
            "netlist": name, "gates": len(c.gates), "bootstraps": nb, "levels": len(sched.waves),
            "max_level_gates": max(sum(len(b.gate_ids) for b in w) for w in sched.waves),
            "app_latency_s": app, "app_latency_first_s": lat[0], "gates_per_s": len(c.gates) / app, "bootstraps_per_s": nb / app,
            "device_time_s": met.device_time_seconds, "metrics_wall_time_s": met.wall_time_seconds,
            "wall_over_device": met.wall_time_seconds / met.device_time_seconds if met.device_time_seconds else None,
            "decrypt_ok": bool(ok),
            "input_bits": int(sum(p.width for p in c.inputs)), "output_bits": int(sum(p.width for p in c.outputs)),
            "host_prep": prep, **({"per_vector": per_vec} if per_vec else {})})
    if rank == 0:
        print(json.dumps({"config": args.config, "n_gpus": ws, "params": "PARAM_128",
                          "keygen_and_upload_s": t_keys, "results": results}), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
