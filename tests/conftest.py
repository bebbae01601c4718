"""Shared fixtures.  `-m gpu` tests need a B200 and the built engine library;
everything else runs on the CPU (oracle, host logic, C-ABI symbol checks)."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

from paper_2306_11006_b200.cggi import ParamSet  # noqa: E402

# tests/conftest.py:7-16 of the reference
MINI = ParamSet(n=16, N=64, lwe_noise_std=2.0 ** -20, rlwe_noise_std=1e-9, Bg_bits=9, l=2,
                ks_base_bits=2, ks_levels=8)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 and the built CUDA engine")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden_json():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_mini():
    return dict(np.load(os.path.join(GOLDEN, "mini.npz")))


@pytest.fixture(scope="session")
def golden_p128():
    return dict(np.load(os.path.join(GOLDEN, "p128.npz")))


@pytest.fixture(scope="session")
def golden_p110():
    return dict(np.load(os.path.join(GOLDEN, "p110.npz")))


@pytest.fixture(scope="session")
def mini_keys():
    from paper_2306_11006_b200.cggi import keygen
    return keygen(MINI, seed=2024)


@pytest.fixture(scope="session")
def p128_keys():
    from paper_2306_11006_b200.cggi import PARAM_128, keygen
    return keygen(PARAM_128, seed=7)


@pytest.fixture(scope="session")
def p110_keys():
    from paper_2306_11006_b200.cggi import PARAM_110, keygen
    return keygen(PARAM_110, seed=7)


def digest(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]
