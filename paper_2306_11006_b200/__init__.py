"""B200-native CGGI gate-bootstrapping engine with the `gatewave` Python API.

Drop-in for the reference package's hot path (arxiv 2306.11006 / ArctyrEX,
CPU re-creation `gatewave`): key generation, encryption, homomorphic gates and
level-scheduled netlist evaluation, with the bootstrapping pipeline in
hand-written sm_100a CUDA kernels.
"""
from .cggi import (  # noqa: F401
    GATE_ARITY, BOOTSTRAPS_PER_GATE, PARAM_110, PARAM_128, PARAM_SETS, TWO_INPUT_KINDS,
    DimensionError, EvalKey, GateKind, KeySet, LweCiphertext, OpCounter, ParameterError,
    ParamSet, SecretKey, TlweCiphertext, TransformCounter, blind_rotate, decrypt_bit,
    decrypt_rows, encrypt_bit, encrypt_bits, eval_gate, eval_gate_batch, gate_bootstrap, keygen,
    keyswitch, lwe_linear, lwe_trivial, phase, phase_rows, sample_extract, tlwe_trivial)
from .rng import SeededRng  # noqa: F401

__version__ = "0.1.0"
