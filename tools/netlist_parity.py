"""Paper-scale parity for one BASELINE config (SURVEY.md §8(d) protocol), as a
tool for the configs too long for the test-suite (config 4: 11.8M gates):
every decrypted output against the plaintext model, plus SAMPLES gates of
every level batch recomputed by the oracle (oracle/, test infrastructure) from
the GPU's own operand ciphertexts and compared bit for bit with the GPU's
output ciphertexts.  Prints one JSON line.

    python tools/netlist_parity.py --config 4 [--samples 16]
"""
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
    ap.add_argument("--samples", type=int, default=16)
    args = ap.parse_args()
    import oracle as O
    from netlist_run import build
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200.cggi import PARAM_128, decrypt_rows, encrypt_bits, keygen
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import evaluate
    from paper_2306_11006_b200.scheduler import build_schedule

    ks = keygen(PARAM_128, seed=7)
    ek = ks.eval_key()
    okeys = O.Keys.from_params(PARAM_128, ks.bootstrapping_key.data, ks.keyswitch_key.data)
    report = []
    for name, c, seed in build(args.config):
        rng = np.random.default_rng(seed)
        bits = {p.name: rng.integers(0, 2, p.width).astype(np.uint8) for p in c.inputs}
        srng = SeededRng(1000 * seed)
        inputs = {p.name: encrypt_bits(PARAM_128, ks.lwe_sk, bits[p.name], srng) for p in c.inputs}
        sched = build_schedule(c, 1)
        t = time.monotonic()
        outs, met = evaluate(c, sched, inputs, ek)
        t_eval = time.monotonic() - t
        plain = C.simulate_plain_bits(c, {k: v[:, None] for k, v in bits.items()})
        dec_ok = all(np.array_equal(decrypt_rows(ks.lwe_sk, outs[k]), plain[k][:, 0]) for k in plain)
        eng = ek.engine()
        by_id = {g.id: g for g in c.gates}
        pick = np.random.default_rng(seed + 1)
        checked = mismatched = batches = 0
        t = time.monotonic()
        for wave in sched.waves:
            for b in wave:
                ids = np.asarray(b.gate_ids)
                take = ids[pick.choice(len(ids), size=min(args.samples, len(ids)), replace=False)]
                gates = [by_id[int(g)] for g in take]
                ar = len(gates[0].operands)
                ops = [eng.wires_get(np.asarray([g.operands[k] for g in gates], np.int64)) for k in range(ar)]
                want = O.eval_gate_batch(b.opcode.value, ops, okeys, count=len(gates), threads=os.cpu_count())
                got = eng.wires_get(np.asarray(take, np.int64))
                mismatched += int((got != want).any(axis=1).sum())
                checked += len(gates)
                batches += 1
        report.append({"netlist": name, "gates": len(c.gates), "levels": len(sched.waves),
                       "level_batches": batches, "decrypt_ok": bool(dec_ok),
                       "output_bits": int(sum(p.width for p in c.outputs)),
                       "sampled_gates": checked, "sampled_mismatches": mismatched,
                       "evaluate_s": t_eval, "oracle_s": time.monotonic() - t,
                       "bootstraps": met.bootstrap_count})
    print(json.dumps({"config": args.config, "params": "PARAM_128", "samples_per_batch": args.samples,
                      "oracle_threads": os.cpu_count(), "results": report}), flush=True)


if __name__ == "__main__":
    main()
