"""Parity of the CUDA engine against the oracle and the reference's golden
vectors -- bit-exact ciphertexts (all arithmetic is exact integer mod 2^32).
Runs on a B200 through the C ABI."""
import numpy as np
import pytest

from conftest import MINI, digest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine_mod():
    from paper_2306_11006_b200 import engine
    if engine.device_count() < 1:
        pytest.fail("no CUDA device visible: the gpu tests need a B200")
    return engine


def _mini_eval_key(g):
    from paper_2306_11006_b200.cggi import EvalKey
    return EvalKey.build(MINI, g["bk_data"], g["ksk_data"])


def test_bk_fft_roundtrip_mini(engine_mod, golden_mini):
    """The device FFT-domain key inverts (numpy, same index map) to the
    balanced 16-bit halves of bootstrapping_key.data."""
    from tools_fft import native_inverse_poly
    ek = _mini_eval_key(golden_mini)
    eng = ek.engine()
    fft = eng.bk_fft()
    back = native_inverse_poly(fft, MINI.n, MINI.l, MINI.N)  # (n, 2l, 2, N) int64 lo + 2^16 hi
    assert np.array_equal((back & 0xFFFFFFFF).astype(np.uint32), golden_mini["bk_data"])


def test_blind_rotate_matches_reference_mini(engine_mod, golden_mini):
    ek = _mini_eval_key(golden_mini)
    acc = ek.engine().blind_rotate(golden_mini["br_lin"], golden_mini["br_tv"])
    assert np.array_equal(acc, golden_mini["br_acc"])


def test_keyswitch_matches_reference_mini(engine_mod, golden_mini):
    ek = _mini_eval_key(golden_mini)
    out = ek.engine().keyswitch(golden_mini["ks_in"])
    assert np.array_equal(out, golden_mini["ks_out"])


@pytest.mark.parametrize("kind", ["AND", "OR", "NAND", "NOR", "XOR", "XNOR", "NOT", "MUX",
                                  "CONST0", "CONST1", "COPY"])
def test_every_gate_kind_matches_reference_mini(engine_mod, golden_mini, kind):
    from paper_2306_11006_b200.cggi import GATE_ARITY, GateKind, OpCounter, eval_gate_batch
    ek = _mini_eval_key(golden_mini)
    k = GateKind(kind)
    ops = [golden_mini["op0"], golden_mini["op1"], golden_mini["op2"]][:GATE_ARITY[k]]
    ctr = OpCounter()
    out = eval_gate_batch(k, ops, ek, ctr, count=8)
    assert np.array_equal(out, golden_mini[f"gate_{kind}"])


def test_config1_first_gates_p128(engine_mod, golden_p128, p128_keys):
    """Raw blind-rotation accumulators of the first two config-1 gates."""
    from paper_2306_11006_b200.cggi import PARAM_128
    ek = p128_keys.eval_key()
    tv = np.zeros((2, PARAM_128.N), np.uint32)
    tv[1, :] = PARAM_128.mu
    acc = ek.engine().blind_rotate(golden_p128["lin2"], tv)
    assert np.array_equal(acc, golden_p128["acc2"])


def test_first_gates_p110(engine_mod, golden_p110, p110_keys):
    """PARAM_110 (n = 512): the reference's own accumulators and NAND outputs."""
    from paper_2306_11006_b200.cggi import PARAM_110, GateKind, eval_gate_batch
    ek = p110_keys.eval_key()
    tv = np.zeros((2, PARAM_110.N), np.uint32)
    tv[1, :] = PARAM_110.mu
    acc = ek.engine().blind_rotate(golden_p110["lin2"], tv)
    assert np.array_equal(acc, golden_p110["acc2"])
    out = eval_gate_batch(GateKind.NAND, [golden_p110["in_a_head"], golden_p110["in_b_head"]], ek)
    assert np.array_equal(out, golden_p110["out_head"])


def test_config1_digest_p128(engine_mod, golden_json, golden_p128, p128_keys):
    """256 NAND bootstraps, output sha256[:16] 6b796965e2579b67."""
    from paper_2306_11006_b200.cggi import PARAM_128, GateKind, OpCounter, decrypt_rows, \
        encrypt_bits, eval_gate_batch
    from paper_2306_11006_b200.rng import SeededRng
    g = golden_json["p128"]
    bits_a = np.random.default_rng(0).integers(0, 2, 256)
    bits_b = np.random.default_rng(1).integers(0, 2, 256)
    rng = SeededRng(1)
    A = encrypt_bits(PARAM_128, p128_keys.lwe_sk, bits_a, rng)
    B = encrypt_bits(PARAM_128, p128_keys.lwe_sk, bits_b, rng)
    assert digest(A) == g["in_a"] and digest(B) == g["in_b"]
    ctr = OpCounter()
    out = eval_gate_batch(GateKind.NAND, [A, B], p128_keys.eval_key(), ctr)
    assert np.array_equal(out[:8], golden_p128["out_head"])
    assert digest(out) == g["out_nand"] == "6b796965e2579b67"
    assert [ctr.ntt_forward, ctr.ntt_inverse, ctr.bootstraps] == g["counters"]
    assert np.array_equal(decrypt_rows(p128_keys.lwe_sk, out), (1 - (bits_a & bits_b)).astype(np.uint8))


@pytest.mark.parametrize("batch", [1, 150, 300, 592, 600])  # gates per CTA 1, 2, 3, 4, 3
def test_blind_rotate_batch_shapes_p128(engine_mod, p128_keys, batch):
    """Every CTA geometry (1, 2 or 4 gates per CTA, partial last CTA) against
    the oracle on sampled rows of random LWE samples and a random test vector."""
    import oracle as O
    from paper_2306_11006_b200.cggi import PARAM_128
    rng = np.random.default_rng(batch)
    lin = rng.integers(0, 2 ** 32, (batch, PARAM_128.n + 1), dtype=np.uint32)
    tv = rng.integers(0, 2 ** 32, (2, PARAM_128.N), dtype=np.uint32)
    acc = p128_keys.eval_key().engine().blind_rotate(lin, tv)
    rows = sorted({0, batch - 1, batch // 2, batch // 3, min(batch - 1, 149), min(batch - 1, 297)})
    okeys = O.Keys.from_params(PARAM_128, p128_keys.bootstrapping_key.data,
                               p128_keys.keyswitch_key.data)
    want = O.blind_rotate(lin[rows], tv, okeys.bk_ntt, PARAM_128.Bg_bits, PARAM_128.l)
    assert np.array_equal(acc[rows], want)


def test_two_kernel_variants_agree_p128(engine_mod, p128_keys):
    """The 2-warp kernel (GATEWAVE_BR_KERNEL=v1) and the TMEM kernel give the
    same accumulators (both must equal the reference; see the digest test)."""
    import os
    from paper_2306_11006_b200 import engine
    from paper_2306_11006_b200.cggi import PARAM_128
    rng = np.random.default_rng(5)
    lin = rng.integers(0, 2 ** 32, (40, PARAM_128.n + 1), dtype=np.uint32)
    tv = np.zeros((2, PARAM_128.N), np.uint32)
    tv[1] = PARAM_128.mu
    ks = p128_keys
    a = engine.Engine(*engine.params_tuple(PARAM_128))
    a.upload_keys(ks.bootstrapping_key.data, ks.keyswitch_key.data)
    os.environ["GATEWAVE_BR_KERNEL"] = "v1"
    try:
        b = engine.Engine(*engine.params_tuple(PARAM_128))
    finally:
        del os.environ["GATEWAVE_BR_KERNEL"]
    b.upload_keys(ks.bootstrapping_key.data, ks.keyswitch_key.data)
    assert np.array_equal(a.blind_rotate(lin, tv), b.blind_rotate(lin, tv))


@pytest.mark.parametrize("mode", [{"GATEWAVE_BR_GC": "1", "GATEWAVE_BR_GC1": "tma"},
                                  {"GATEWAVE_BR_GC": "2", "GATEWAVE_BR_LDR": "0"},
                                  {"GATEWAVE_BR_GC": "3", "GATEWAVE_BR_LDR": "0"},
                                  {"GATEWAVE_BR_GC": "4"},
                                  {"GATEWAVE_BR_KERNEL": "v2"}])
def test_blind_rotate_alternative_kernels_p128(engine_mod, p128_keys, mode, monkeypatch):
    """The non-default blind-rotation configurations (key staging through shared
    memory, key streaming by the compute warps, forced gates-per-CTA, the v2
    kernel) are bit-exact too; a fresh context reads the overrides."""
    import oracle as O
    from paper_2306_11006_b200.cggi import PARAM_128
    from paper_2306_11006_b200.engine import Engine, params_tuple
    for k, v in mode.items():
        monkeypatch.setenv(k, v)
    eng = Engine(*params_tuple(PARAM_128), device=0)
    eng.upload_keys(p128_keys.bootstrapping_key.data, None)
    rng = np.random.default_rng(7)
    lin = rng.integers(0, 2 ** 32, (200, PARAM_128.n + 1), dtype=np.uint32)
    tv = rng.integers(0, 2 ** 32, (2, PARAM_128.N), dtype=np.uint32)
    acc = eng.blind_rotate(lin, tv)
    okeys = O.Keys.from_params(PARAM_128, p128_keys.bootstrapping_key.data, p128_keys.keyswitch_key.data)
    rows = [0, 77, 199]
    want = O.blind_rotate(lin[rows], tv, okeys.bk_ntt, okeys.bg_bits, okeys.l, 8)
    assert np.array_equal(acc[rows], want)
