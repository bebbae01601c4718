"""Batches wider than CUDA's 65,535 grid.y limit: the reference
evaluates any batch size (cggi.py:785-854), so eval_gate_batch, the seam-1
keyswitch twin and the plan segments must too.  ~70,000-row NAND at
PARAM_128 (decrypt-exact, oracle-exact on a sample) and 70,000-row MUX /
keyswitch batches at MINI (every row against the oracle)."""
import numpy as np
import pytest

from conftest import MINI

pytestmark = pytest.mark.gpu

B_LARGE = 70_001


def test_nand_batch_wider_than_grid_y_p128(p128_keys):
    import oracle as O
    from paper_2306_11006_b200.cggi import PARAM_128, GateKind, OpCounter, decrypt_rows, encrypt_bits, eval_gate_batch
    from paper_2306_11006_b200.rng import SeededRng
    ks = p128_keys
    r = np.random.default_rng(70)
    a, b = r.integers(0, 2, B_LARGE), r.integers(0, 2, B_LARGE)
    rng = SeededRng(70)
    A = encrypt_bits(PARAM_128, ks.lwe_sk, a, rng)
    B = encrypt_bits(PARAM_128, ks.lwe_sk, b, rng)
    ctr = OpCounter()
    out = eval_gate_batch(GateKind.NAND, [A, B], ks, ctr)
    assert np.array_equal(decrypt_rows(ks.lwe_sk, out), (1 - (a & b)).astype(np.uint8))
    assert ctr.bootstraps == B_LARGE
    okeys = O.Keys.from_params(PARAM_128, ks.bootstrapping_key.data, ks.keyswitch_key.data)
    pick = np.sort(np.concatenate([r.choice(B_LARGE, 12, replace=False), [0, 65534, 65535, B_LARGE - 1]]))
    want = O.eval_gate_batch("NAND", [A[pick], B[pick]], okeys, threads=16)
    assert np.array_equal(out[pick], want)


def test_mux_and_keyswitch_batches_wider_than_grid_y_mini(mini_keys):
    import oracle as O
    from paper_2306_11006_b200.cggi import GateKind, decrypt_rows, encrypt_bits, eval_gate_batch, keyswitch_rows
    from paper_2306_11006_b200.rng import SeededRng
    ks = mini_keys
    r = np.random.default_rng(71)
    bits = r.integers(0, 2, (3, B_LARGE))
    rng = SeededRng(71)
    ops = [encrypt_bits(MINI, ks.lwe_sk, bits[k], rng) for k in range(3)]
    out = eval_gate_batch(GateKind.MUX, ops, ks)
    assert np.array_equal(decrypt_rows(ks.lwe_sk, out), np.where(bits[0] == 1, bits[1], bits[2]).astype(np.uint8))
    okeys = O.Keys.from_params(MINI, ks.bootstrapping_key.data, ks.keyswitch_key.data)
    assert np.array_equal(out, O.eval_gate_batch("MUX", ops, okeys, threads=16))
    ext = r.integers(0, 2 ** 32, (B_LARGE, MINI.N + 1), dtype=np.uint32)
    got = keyswitch_rows(ext, ks)
    assert np.array_equal(got, O.keyswitch(ext, okeys.ksk, MINI.ks_levels, MINI.ks_base_bits, 16))
