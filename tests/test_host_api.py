"""Host-side API parity with the reference (cggi.py client side, rng.py):
parameter envelope, key generation, encryption, decryption, sample algebra.
Keys and ciphertexts must be byte-identical to the reference's from the same
seeds (pinned by the reference-generated digests in tests/golden)."""
import numpy as np
import pytest

from conftest import MINI, digest
from paper_2306_11006_b200 import cggi
from paper_2306_11006_b200.cggi import (PARAM_110, PARAM_128, DimensionError, GateKind,
                                        ParameterError, ParamSet, decrypt_bit, decrypt_rows,
                                        encrypt_bit, encrypt_bits, keygen, lwe_linear, lwe_trivial,
                                        phase, phase_rows, torus_signed)
from paper_2306_11006_b200.rng import SeededRng


def test_builtin_parameter_sets():
    assert (PARAM_110.n, PARAM_110.N, PARAM_110.mu) == (512, 1024, 2 ** 29)
    assert (PARAM_128.n, PARAM_128.N) == (630, 1024)


def test_parameter_validation():
    ok = dict(n=16, N=64, lwe_noise_std=1e-6, rlwe_noise_std=1e-9, Bg_bits=9, l=2,
              ks_base_bits=2, ks_levels=8)
    ParamSet(**ok)
    for bad in ({"N": 48}, {"Bg_bits": 17}, {"N": 1024, "l": 1, "Bg_bits": 23},
                {"ks_base_bits": 5, "ks_levels": 7}, {"lwe_noise_std": 0.7}, {"mu": 0}):
        with pytest.raises(ParameterError):
            ParamSet(**{**ok, **bad})


@pytest.mark.parametrize("tag,params", [("p128", PARAM_128), ("p110", PARAM_110)])
def test_keygen_and_config1_inputs_match_reference(golden_json, tag, params):
    g = golden_json[tag]
    ks = keygen(params, seed=7)
    assert digest(ks.lwe_sk) == g["lwe_sk"]
    assert digest(ks.rlwe_sk) == g["rlwe_sk"]
    assert digest(ks.bootstrapping_key.data) == g["bk_data"]
    assert digest(ks.keyswitch_key.data) == g["ksk_data"]
    bits_a = np.random.default_rng(0).integers(0, 2, g["gates"])
    bits_b = np.random.default_rng(1).integers(0, 2, g["gates"])
    rng = SeededRng(1)
    assert digest(encrypt_bits(params, ks.lwe_sk, bits_a, rng)) == g["in_a"]
    assert digest(encrypt_bits(params, ks.lwe_sk, bits_b, rng)) == g["in_b"]


def test_mini_keygen_matches_reference(golden_mini):
    ks = keygen(MINI, seed=2024)
    assert np.array_equal(ks.lwe_sk, golden_mini["lwe_sk"])
    assert np.array_equal(ks.bootstrapping_key.data, golden_mini["bk_data"])
    assert np.array_equal(ks.keyswitch_key.data, golden_mini["ksk_data"])
    rng = SeededRng(100)
    for k in range(3):
        assert np.array_equal(encrypt_bits(MINI, ks.lwe_sk, golden_mini["bits"][k], rng),
                              golden_mini[f"op{k}"])


def test_keygen_is_deterministic():
    a, b, c = keygen(MINI, 99), keygen(MINI, 99), keygen(MINI, 100)
    assert np.array_equal(a.bootstrapping_key.data, b.bootstrapping_key.data)
    assert np.array_equal(a.keyswitch_key.data, b.keyswitch_key.data)
    assert not np.array_equal(a.bootstrapping_key.data, c.bootstrapping_key.data)


def test_encrypt_decrypt_roundtrip(mini_keys):
    bits = np.array([0, 1] * 100, dtype=np.uint32)
    rows = encrypt_bits(MINI, mini_keys.lwe_sk, bits, SeededRng(42))
    assert rows.shape == (200, MINI.n + 1)
    assert np.array_equal(decrypt_rows(mini_keys.lwe_sk, rows), bits.astype(np.uint8))


def test_fresh_phase_sits_at_message_levels(mini_keys):
    rows = encrypt_bits(MINI, mini_keys.lwe_sk, [1] * 50 + [0] * 50, SeededRng(43))
    ph = torus_signed(phase_rows(mini_keys.lwe_sk, rows)).astype(np.int64)
    assert np.all(np.abs(ph[:50] - MINI.mu) < 2 ** 14)
    assert np.all(np.abs(ph[50:] + MINI.mu) < 2 ** 14)


def test_encrypt_rejects_bad_bits(mini_keys):
    with pytest.raises(ValueError):
        encrypt_bits(MINI, mini_keys.lwe_sk, [0, 2], SeededRng(1))
    with pytest.raises(DimensionError):
        encrypt_bits(MINI, mini_keys.lwe_sk, [[0], [1]], SeededRng(1))


def test_trivial_samples_and_linear_combination(mini_keys):
    sk = mini_keys.lwe_sk
    assert decrypt_bit(sk, lwe_trivial(MINI, MINI.mu)) == 1
    assert decrypt_bit(sk, lwe_trivial(MINI, MINI.minus_mu)) == 0
    rng = SeededRng(44)
    cts = [encrypt_bit(MINI, sk, b, rng) for b in (0, 1, 1)]
    combo = lwe_linear([1, -2, 3], cts, 0x12345678)
    want = (sum(w * phase(sk, ct) for w, ct in zip([1, -2, 3], cts)) + 0x12345678) & 0xFFFFFFFF
    assert phase(sk, combo) == want


def test_gadget_digits_range_and_recompose():
    rng = np.random.default_rng(45)
    for _ in range(50):
        poly = rng.integers(0, 2 ** 32, MINI.N, dtype=np.uint32)
        d = cggi.gadget_decompose(poly, MINI)
        assert d.min() >= -256 and d.max() < 256
        err = torus_signed(poly - cggi.gadget_recompose(d, MINI)).astype(np.int64)
        assert np.all(np.abs(err) <= 1 << (32 - MINI.l * MINI.Bg_bits - 1))


def test_decompose_offset_matches_oracle():
    import oracle as O
    assert cggi.decompose_offset(9, 2) == O.decompose_offset(9, 2)


def test_gate_tables():
    assert cggi.BOOTSTRAPS_PER_GATE[GateKind.AND] == 1
    assert cggi.BOOTSTRAPS_PER_GATE[GateKind.MUX] == 2
    assert cggi.BOOTSTRAPS_PER_GATE[GateKind.NOT] == 0
    assert [k.value for k in GateKind] == ["AND", "OR", "NAND", "NOR", "XOR", "XNOR", "NOT",
                                           "MUX", "CONST0", "CONST1", "COPY"]


def test_gate_api_validates_before_touching_the_device(mini_keys):
    """DimensionError cases of the reference (tests/test_cggi.py:372-383) are
    raised host-side, so they hold with or without a GPU."""
    ek = mini_keys.eval_key()
    good = np.zeros((2, MINI.n + 1), np.uint32)
    with pytest.raises(DimensionError):
        cggi.eval_gate_batch(GateKind.AND, [good, np.zeros((2, MINI.n), np.uint32)], ek)
    with pytest.raises(DimensionError):
        cggi.eval_gate_batch(GateKind.AND, [good], ek)
    with pytest.raises(DimensionError):
        cggi.eval_gate_batch(GateKind.AND, [good, np.zeros((3, MINI.n + 1), np.uint32)], ek)
    with pytest.raises(DimensionError):
        cggi.eval_gate_batch(GateKind.CONST0, [], ek)


def test_engine_methods_are_serialised():
    """Every public method of the context wrappers holds the engine lock (a
    gw_ctx is single-submitter; the reference runtime calls from K threads)."""
    from paper_2306_11006_b200 import engine as E
    for cls, names in ((E.Engine, ("eval_gate_batch", "blind_rotate", "keyswitch", "wires_put",
                                   "wires_get", "plan_create", "sync", "upload_keys")),
                       (E.Plan, ("run", "run_timed", "close")),
                       (E.ExchangePlanHandle, ("pack", "unpack", "peer_rows", "enqueue", "close"))):
        for n in names:
            assert hasattr(getattr(cls, n), "__wrapped__"), f"{cls.__name__}.{n} is not serialised"


def test_api_golden_inputs_reproduced(mini_keys, p128_keys):
    """keygen + encrypt_bits reproduce the operands the reference encrypted
    for tests/golden/api.npz (so the GPU wrappers see identical bytes)."""
    import os
    from conftest import GOLDEN, MINI
    from paper_2306_11006_b200.cggi import PARAM_128, encrypt_bits
    from paper_2306_11006_b200.rng import SeededRng
    g = dict(np.load(os.path.join(GOLDEN, "api.npz")))
    for tag, ks, p, seed in (("mini", mini_keys, MINI, 2024), ("p128", p128_keys, PARAM_128, 7)):
        bits = np.random.default_rng(500 + seed).integers(0, 2, g[f"{tag}_bits"].shape)
        assert np.array_equal(bits, g[f"{tag}_bits"])
        rng = SeededRng(500 + seed)
        for k in range(3):
            assert np.array_equal(encrypt_bits(p, ks.lwe_sk, bits[k], rng), g[f"{tag}_ct{k}"])


def test_sample_extract_matches_reference_golden():
    import os
    from conftest import GOLDEN
    from paper_2306_11006_b200.cggi import TlweCiphertext, sample_extract
    g = dict(np.load(os.path.join(GOLDEN, "api.npz")))
    for tag in ("mini", "p128"):
        got = np.stack([sample_extract(TlweCiphertext(a)).vec for a in g[f"{tag}_blind_rotate"]])
        assert np.array_equal(got, g[f"{tag}_sample_extract"])
