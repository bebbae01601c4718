"""Golden ARFX files written by the UNMODIFIED reference (gatewave.serial) in
this container, for tests/test_serial.py.  Run once here (the reference is
not on the GPU box; the files are committed):

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \\
        python tests/golden/make_arfx.py

MINI keys (keygen seed 2024, tests/conftest.py), PARAM_128 parameter block,
and a 5-wire MINI bundle; digests.json holds sha256 of every file.
"""
import hashlib
import json
import os

import numpy as np
from gatewave import serial
from gatewave.cggi import PARAM_128, ParamSet, encrypt_bits, keygen
from gatewave.rng import SeededRng

OUT = os.path.dirname(os.path.abspath(__file__)) + "/arfx"
MINI = ParamSet(n=16, N=64, lwe_noise_std=2.0 ** -20, rlwe_noise_std=1e-9, Bg_bits=9, l=2,
                ks_base_bits=2, ks_levels=8)
os.makedirs(OUT, exist_ok=True)
ks = keygen(MINI, seed=2024)
serial.write_secret_key(f"{OUT}/mini.sk", ks)
serial.write_eval_key(f"{OUT}/mini.ek", ks)
rows = encrypt_bits(MINI, ks.lwe_sk, np.array([1, 0, 1, 1, 0], np.uint8), SeededRng(77))
serial.write_bundle(f"{OUT}/mini.bundle", MINI, {w: rows[k] for k, w in enumerate([9, 3, 41, 0, 7])})
with open(f"{OUT}/p128.params", "wb") as f:
    f.write(serial.params_to_bytes(PARAM_128))
dig = {name: hashlib.sha256(open(f"{OUT}/{name}", "rb").read()).hexdigest()
       for name in sorted(os.listdir(OUT)) if not name.endswith(".json")}
dig["p128_params_digest"] = serial.params_digest(PARAM_128).hex()
json.dump(dig, open(f"{OUT}/digests.json", "w"), indent=1)
print(dig)
