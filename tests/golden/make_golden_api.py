"""Golden vectors for the single-sample API wrappers, from the REFERENCE itself.

Run here (never on the GPU box):
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_api.py

Imports the unmodified reference from /root/reference/pkg/src and records, at
fixed seeds, the outputs of the public single-sample entry points
(cggi.py:730-777, 857-873): gate_bootstrap, blind_rotate, sample_extract,
keyswitch and eval_gate, with their counter tallies, for MINI keys
(keygen(MINI, 2024)) and PARAM_128 keys (keygen(PARAM_128, 7)).
Writes tests/golden/api.npz + api.json.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from gatewave import cggi  # noqa: E402
from gatewave.cggi import (GateKind, LweCiphertext, OpCounter, ParamSet, PARAM_128,  # noqa: E402
                           TlweCiphertext, encrypt_bits, keygen)
from gatewave.rng import SeededRng  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
MINI = ParamSet(n=16, N=64, lwe_noise_std=2.0 ** -20, rlwe_noise_std=1e-9,
                Bg_bits=9, l=2, ks_base_bits=2, ks_levels=8)


def record(tag, params, seed, n_cts, out, js):
    ks = keygen(params, seed=seed)
    ek = ks.eval_key()
    bits = np.random.default_rng(500 + seed).integers(0, 2, (3, n_cts))
    rng = SeededRng(500 + seed)
    cts = [encrypt_bits(params, ks.lwe_sk, bits[k], rng) for k in range(3)]
    out[f"{tag}_bits"] = bits
    for k in range(3):
        out[f"{tag}_ct{k}"] = cts[k]
    tally = {}
    # gate_bootstrap (cggi.py:770-777) on every sample of operand 0
    gb, ctr = [], OpCounter()
    for j in range(n_cts):
        gb.append(cggi.gate_bootstrap(LweCiphertext(cts[0][j]), ek, ctr).vec)
    out[f"{tag}_gate_bootstrap"] = np.stack(gb)
    tally["gate_bootstrap"] = [ctr.ntt_forward, ctr.ntt_inverse, ctr.bootstraps]
    # blind_rotate with the bootstrap test vector and a random one (cggi.py:730-753)
    r = np.random.default_rng(600 + seed)
    tv_mu = np.zeros((2, params.N), np.uint32)
    tv_mu[1, :] = params.mu
    tv_rand = r.integers(0, 2 ** 32, (2, params.N), dtype=np.uint32)
    out[f"{tag}_tv_rand"] = tv_rand
    br = []
    ctr = OpCounter()
    for j in range(n_cts):
        for tv in (tv_mu, tv_rand):
            br.append(cggi.blind_rotate(TlweCiphertext(tv), LweCiphertext(cts[1][j]),
                                        ek.bk, ek.tables, ctr).data)
    out[f"{tag}_blind_rotate"] = np.stack(br)
    tally["blind_rotate"] = [ctr.ntt_forward, ctr.ntt_inverse]
    # sample_extract (cggi.py:756-758) and keyswitch (cggi.py:761-767) of those
    ext = [cggi.sample_extract(TlweCiphertext(a)).vec for a in br]
    out[f"{tag}_sample_extract"] = np.stack(ext)
    out[f"{tag}_keyswitch"] = np.stack([cggi.keyswitch(LweCiphertext(e), ek.ksk).vec for e in ext])
    # eval_gate (cggi.py:857-873), every kind on sample 0
    for kind in GateKind:
        ar = cggi.GATE_ARITY[kind]
        ctr = OpCounter()
        res = cggi.eval_gate(kind, [LweCiphertext(cts[k][0]) for k in range(ar)], ek, ctr)
        out[f"{tag}_eval_gate_{kind.value}"] = res.vec
        tally[f"eval_gate_{kind.value}"] = [ctr.ntt_forward, ctr.ntt_inverse, ctr.bootstraps]
    js[tag] = tally


def main():
    out, js = {}, {"reference": "/root/reference/pkg/src/gatewave (unmodified)",
                   "generator": "tests/golden/make_golden_api.py"}
    record("mini", MINI, 2024, 6, out, js)
    record("p128", PARAM_128, 7, 2, out, js)
    np.savez_compressed(os.path.join(HERE, "api.npz"), **out)
    with open(os.path.join(HERE, "api.json"), "w") as f:
        json.dump(js, f, indent=1, sort_keys=True)
    print(json.dumps(js, indent=1))


if __name__ == "__main__":
    main()
