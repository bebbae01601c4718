"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Run here (never on the GPU box):
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports the unmodified reference package from /root/reference/pkg/src and
records, at fixed seeds:
  * mini.npz   -- MINI-parameter keys (coefficient + NTT domain), gate outputs
                  for every GateKind, raw blind-rotation accumulators for a
                  random test vector, keyswitch outputs, NTT vectors, and an
                  adder4 netlist evaluation (tests/conftest.py:7-16 params).
  * p128.npz / p110.npz -- the first rows of the config-1 computation
                  (SURVEY.md Appendix A recipe) plus blind-rotation
                  accumulators and keyswitch outputs for a few gates.
  * golden.json -- sha256[:16] digests of the full artefacts (keys, config-1
                  inputs and outputs) and the counter tallies.
These fixtures pin oracle/ (the CPU restatement) and, through it, the CUDA path.
"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from gatewave import cggi, circuit, runtime, scheduler, torus  # noqa: E402
from gatewave.cggi import (  # noqa: E402
    GateKind, OpCounter, ParamSet, PARAM_110, PARAM_128, _blind_rotate_kernel,
    _decompose_offset, _extract_rows, _keyswitch_kernel, encrypt_bits, eval_gate_batch,
    keygen)
from gatewave.rng import SeededRng  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

MINI = ParamSet(n=16, N=64, lwe_noise_std=2.0 ** -20, rlwe_noise_std=1e-9,
                Bg_bits=9, l=2, ks_base_bits=2, ks_levels=8)


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def raw_rotate(lin, tv, ek):
    p = ek.params
    counts = np.zeros(2, dtype=np.int64)
    acc = _blind_rotate_kernel(lin, tv, ek.bk.ntt, ek.tables.psi_brv, ek.tables.ipsi_brv,
                               ek.tables.n_inv, ek.tables.log_n, p.Bg_bits, p.l,
                               _decompose_offset(p.Bg_bits, p.l), counts)
    return acc, counts


def mini_fixture(js):
    ks = keygen(MINI, seed=2024)
    ek = ks.eval_key()
    out = dict(lwe_sk=ks.lwe_sk, rlwe_sk=ks.rlwe_sk, bk_data=ks.bootstrapping_key.data,
               bk_ntt=ks.bootstrapping_key.ntt, ksk_data=ks.keyswitch_key.data,
               psi_brv=ek.tables.psi_brv, ipsi_brv=ek.tables.ipsi_brv)
    B = 8
    bits = np.random.default_rng(100).integers(0, 2, (3, B))
    rng = SeededRng(100)
    ops = [encrypt_bits(MINI, ks.lwe_sk, bits[k], rng) for k in range(3)]
    out.update(bits=bits, op0=ops[0], op1=ops[1], op2=ops[2])
    counters = {}
    for kind in GateKind:
        ar = cggi.GATE_ARITY[kind]
        ctr = OpCounter()
        res = eval_gate_batch(kind, ops[:ar], ek, ctr, count=B)
        out[f"gate_{kind.value}"] = res
        counters[kind.value] = [ctr.ntt_forward, ctr.ntt_inverse, ctr.bootstraps]
    js["mini_counters"] = counters
    # raw blind rotation with an arbitrary test vector and arbitrary lin rows
    r = np.random.default_rng(101)
    lin = r.integers(0, 2**32, (5, MINI.n + 1), dtype=np.uint32)
    tv = r.integers(0, 2**32, (2, MINI.N), dtype=np.uint32)
    acc, counts = raw_rotate(lin, tv, ek)
    out.update(br_lin=lin, br_tv=tv, br_acc=acc)
    js["mini_br_counts"] = [int(c) for c in counts]
    ext = r.integers(0, 2**32, (6, MINI.N + 1), dtype=np.uint32)
    out.update(ks_in=ext, ks_out=_keyswitch_kernel(ext, ek.ksk.data, MINI.ks_levels,
                                                      MINI.ks_base_bits))
    out.update(extract_in=acc, extract_out=_extract_rows(acc))
    # torus layer: NTT ordering + exact negacyclic product
    tabs = torus.build_ntt_tables(64)
    vec = r.integers(0, torus.Q, (3, 64), dtype=np.uint64)
    out.update(ntt_in=vec, ntt_fwd=torus.ntt_forward(vec, tabs),
               ntt_inv=torus.ntt_inverse(vec, tabs))
    pint = r.integers(-256, 256, (3, 64)).astype(np.int64)
    q = r.integers(0, 2**32, (3, 64), dtype=np.uint32)
    out.update(nm_p=pint, nm_q=q,
               nm_out=np.stack([torus.negacyclic_mul_naive(pint[k], q[k]) for k in range(3)]))
    # adder4 evaluated through the reference runtime (K=2 workers)
    c = circuit.gen_adder(4)
    sched = scheduler.build_schedule(c, 2)
    rng2 = SeededRng(77)
    inputs = {"a": encrypt_bits(MINI, ks.lwe_sk, circuit.value_to_bits(9, 4), rng2),
              "b": encrypt_bits(MINI, ks.lwe_sk, circuit.value_to_bits(8, 4), rng2)}
    outs, met = runtime.evaluate(c, sched, inputs, ek)
    out.update(adder_a=inputs["a"], adder_b=inputs["b"], adder_s=outs["s"])
    js["mini_adder4"] = dict(value=int(circuit.bits_to_value(cggi.decrypt_rows(ks.lwe_sk, outs["s"]))),
                            bootstraps=met.bootstrap_count, fwd=met.ntt_forward_count,
                            inv=met.ntt_inverse_count, total_gates=met.total_gates,
                            waves=[len(w) for w in sched.waves])
    js["mini_digests"] = {k: digest(v) for k, v in out.items()}
    np.savez_compressed(os.path.join(HERE, "mini.npz"), **out)


def real_fixture(js, params, tag, gates):
    ks = keygen(params, seed=7)
    ek = ks.eval_key()
    d = dict(lwe_sk=digest(ks.lwe_sk), rlwe_sk=digest(ks.rlwe_sk),
             bk_data=digest(ks.bootstrapping_key.data), bk_ntt=digest(ks.bootstrapping_key.ntt),
             ksk_data=digest(ks.keyswitch_key.data))
    # config-1 inputs
    bits_a = np.random.default_rng(0).integers(0, 2, gates)
    bits_b = np.random.default_rng(1).integers(0, 2, gates)
    rng = SeededRng(1)
    A = encrypt_bits(params, ks.lwe_sk, bits_a, rng)
    Bm = encrypt_bits(params, ks.lwe_sk, bits_b, rng)
    ctr = OpCounter()
    out = eval_gate_batch(GateKind.NAND, [A, Bm], ek, ctr)
    d.update(in_a=digest(A), in_b=digest(Bm), out_nand=digest(out),
             counters=[ctr.ntt_forward, ctr.ntt_inverse, ctr.bootstraps], gates=gates)
    assert np.array_equal(cggi.decrypt_rows(ks.lwe_sk, out), (1 - (bits_a & bits_b)).astype(np.uint8))
    # per-stage intermediates for the first two gates
    lin = (A[:2].astype(np.int64) * -1 + Bm[:2].astype(np.int64) * -1)
    lin[:, -1] += params.mu
    lin = (lin & 0xFFFFFFFF).astype(np.uint32)
    tv = np.zeros((2, params.N), dtype=np.uint32)
    tv[1, :] = params.mu
    acc, _ = raw_rotate(lin, tv, ek)
    ext = _extract_rows(acc)
    ksout = _keyswitch_kernel(ext, ek.ksk.data, params.ks_levels, params.ks_base_bits)
    assert np.array_equal(ksout, out[:2])
    arrs = dict(out_head=out[:8], in_a_head=A[:8], in_b_head=Bm[:8], lin2=lin, acc2=acc,
                bits_a=bits_a, bits_b=bits_b)
    # Goldilocks NTT ordering at N=1024 and the first BK slab in NTT domain
    r = np.random.default_rng(102)
    vec = r.integers(0, 2**32, (2, params.N), dtype=np.uint64)
    arrs.update(ntt_in=vec, ntt_fwd=torus.ntt_forward(vec, ek.tables),
                bk_ntt_slab0=ks.bootstrapping_key.ntt[0])
    js[tag] = d
    np.savez_compressed(os.path.join(HERE, f"{tag}.npz"), **arrs)


def main():
    js = {"reference": "/root/reference/pkg/src/gatewave (unmodified)",
          "generator": "tests/golden/make_golden.py"}
    mini_fixture(js)
    real_fixture(js, PARAM_128, "p128", 256)
    real_fixture(js, PARAM_110, "p110", 32)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(js, f, indent=1, sort_keys=True)
    print(json.dumps(js["p128"], indent=1))


if __name__ == "__main__":
    main()
