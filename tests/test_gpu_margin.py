"""Exactness margin of the FP64 external product, measured on the device.

The engine rounds every inverse-transform value of the blind rotation to the
nearest integer; that recovers the exact integer (hence ciphertexts
bit-identical to the reference's Goldilocks NTT) whenever |x - rint(x)| < 0.5.
The probe build records the worst distance over every rounded value
(DESIGN.md §3).  At PARAM_128 / PARAM_110 the default kernel (v5) transforms the
full 32-bit key words (coefficients up to 2^51; measured margin ~0.03); at the
engine envelope's edge (Bg = 10, l = 2, N = 1024), where v5 does not apply, the
split-key kernel (v3, coefficients up to 2^36; ~7e-7) runs.  Assert < 0.1 in
both regimes, bit-exact against the oracle / the reference's golden vectors."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _probe(ek, lin, tv):
    eng = ek.engine()
    eng.set_margin_probe(True)
    try:
        acc = eng.blind_rotate(lin, tv)
        return acc, eng.margin(reset=True)
    finally:
        eng.set_margin_probe(False)


def test_margin_config1_p128(golden_p128, p128_keys):
    from paper_2306_11006_b200.cggi import PARAM_128, GateKind, eval_gate_batch
    ek = p128_keys.eval_key()
    eng = ek.engine()
    eng.set_margin_probe(True)
    try:
        from conftest import digest
        import bench
        ks, A, B, _, _ = bench._workload(PARAM_128, 0, 256)
        out = eval_gate_batch(GateKind.NAND, [A, B], ek)
        worst = eng.margin(reset=True)
    finally:
        eng.set_margin_probe(False)
    assert digest(out) == "6b796965e2579b67"    # probe build is the same arithmetic
    print(f"PARAM_128 config 1: worst |x - rint(x)| = {worst:.3e}")
    assert 0 < worst < 0.1


def test_margin_p110(golden_p110, p110_keys):
    from paper_2306_11006_b200.cggi import PARAM_110
    ek = p110_keys.eval_key()
    tv = np.zeros((2, PARAM_110.N), np.uint32)
    tv[1, :] = PARAM_110.mu
    acc, worst = _probe(ek, golden_p110["lin2"], tv)
    assert np.array_equal(acc, golden_p110["acc2"])
    assert 0 < worst < 0.1


def test_margin_at_envelope_edge_bg10():
    """Bg = 10, l = 2, N = 1024 (|coefficients| up to 2^36, the largest the
    engine accepts): random keys and random rows with a random test vector,
    bit-exact against the oracle, margin measured."""
    import oracle as O
    from paper_2306_11006_b200.cggi import ParamSet, keygen
    p = ParamSet(n=24, N=1024, lwe_noise_std=2.0 ** -15, rlwe_noise_std=2.5e-8, Bg_bits=10, l=2,
                 ks_base_bits=2, ks_levels=8)
    ks = keygen(p, seed=31)
    ek = ks.eval_key()
    r = np.random.default_rng(32)
    lin = r.integers(0, 2 ** 32, (40, p.n + 1), dtype=np.uint32)
    tv = r.integers(0, 2 ** 32, (2, p.N), dtype=np.uint32)
    acc, worst = _probe(ek, lin, tv)
    okeys = O.Keys.from_params(p, ks.bootstrapping_key.data, ks.keyswitch_key.data)
    want = O.blind_rotate(lin, tv, okeys.bk_ntt, p.Bg_bits, p.l, threads=8)
    assert np.array_equal(acc, want)
    print(f"Bg=10 envelope edge: worst |x - rint(x)| = {worst:.3e}")
    assert 0 < worst < 0.1


def test_envelope_beyond_edge_rejected():
    from paper_2306_11006_b200.cggi import ParameterError, ParamSet
    from paper_2306_11006_b200.engine import Engine, params_tuple
    p = ParamSet(n=24, N=1024, lwe_noise_std=2.0 ** -15, rlwe_noise_std=2.5e-8, Bg_bits=11, l=2,
                 ks_base_bits=2, ks_levels=8)
    with pytest.raises(ParameterError):
        Engine(*params_tuple(p), device=0)
