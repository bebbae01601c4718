"""Single-image blind rotation (v5, the default at PARAM_128 / PARAM_110) against
the split-key kernel (v3, exact mode) and the reference's golden vectors.

v5 holds ONE FFT image of the 32-bit bootstrapping-key words: every value its
inverse transforms round is an integer of magnitude up to 2^51, where the FP64
error is no longer provably < 1/2, so its exactness is measured:
the same outputs as the exact kernel, bit for bit, and the probe build's worst
|x - rint(x)| well inside 1/2."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _with_exact(eng, on, fn):
    prev = eng.exact()
    eng.set_exact(on)
    try:
        return fn()
    finally:
        eng.set_exact(prev)


def _probe(eng, fn):
    eng.set_margin_probe(True)
    try:
        out = fn()
        return out, eng.margin(reset=True)
    finally:
        eng.set_margin_probe(False)


def test_default_is_v5_and_exact_mode_switches(p128_keys):
    import os
    default = os.environ.get("GATEWAVE_BR_EXACT", "0") not in ("", "0")  # the suite can run forced-exact
    eng = p128_keys.eval_key().engine()
    assert eng.exact() is default
    assert _with_exact(eng, True, eng.exact) is True
    assert _with_exact(eng, False, eng.exact) is False
    assert eng.exact() is default


@pytest.mark.parametrize("G", [1, 148, 256, 296, 444, 600])
def test_v5_matches_exact_kernel_every_gc(p128_keys, G):
    """Batch sizes covering 1, 2 and 3 gates per SM (and a partial last wave):
    accumulators bit-identical between v5 and the split-key v3."""
    from paper_2306_11006_b200.cggi import PARAM_128
    ek = p128_keys.eval_key()
    eng = ek.engine()
    rng = np.random.default_rng(G)
    lin = rng.integers(0, 2 ** 32, (G, PARAM_128.n + 1), dtype=np.uint32)
    tv = rng.integers(0, 2 ** 32, (2, PARAM_128.N), dtype=np.uint32)
    fast, worst = _probe(eng, lambda: eng.blind_rotate(lin, tv))
    exact = _with_exact(eng, True, lambda: eng.blind_rotate(lin, tv))
    assert np.array_equal(fast, exact)
    print(f"G={G}: v5 worst |x - rint(x)| = {worst:.3e}")
    assert 0 < worst < 0.25


def test_v5_config1_digest_both_modes(p128_keys):
    from conftest import digest
    import bench
    from paper_2306_11006_b200.cggi import PARAM_128, GateKind, eval_gate_batch
    ek = p128_keys.eval_key()
    eng = ek.engine()
    ks, A, B, _, _ = bench._workload(PARAM_128, 0, 256)
    out, worst = _probe(eng, lambda: eval_gate_batch(GateKind.NAND, [A, B], ek))
    assert digest(out) == "6b796965e2579b67"
    out3, worst3 = _with_exact(eng, True, lambda: _probe(eng, lambda: eval_gate_batch(GateKind.NAND, [A, B], ek)))
    assert digest(out3) == "6b796965e2579b67"
    print(f"config 1: v5 margin {worst:.3e}, v3 (exact) margin {worst3:.3e}")
    assert worst < 0.25 and worst3 < 1e-4


def test_v5_p110_golden(golden_p110, p110_keys):
    from paper_2306_11006_b200.cggi import PARAM_110
    eng = p110_keys.eval_key().engine()
    tv = np.zeros((2, PARAM_110.N), np.uint32)
    tv[1, :] = PARAM_110.mu
    acc, worst = _probe(eng, lambda: eng.blind_rotate(golden_p110["lin2"], tv))
    assert np.array_equal(acc, golden_p110["acc2"])
    assert 0 < worst < 0.25


def test_adversarial_extreme_key_words_margin(p128_keys):
    """Worst-case-leaning inputs for v5: a test vector and LWE rows drawn so the
    digits hit the ends of their range often (rows of all-ones / all-zeros
    bits), against the exact kernel."""
    from paper_2306_11006_b200.cggi import PARAM_128
    eng = p128_keys.eval_key().engine()
    rng = np.random.default_rng(99)
    G = 148
    lin = rng.choice(np.array([0, 0xFFFFFFFF, 0x80000000, 0x7FFFFFFF], np.uint32), (G, PARAM_128.n + 1))
    tv = rng.choice(np.array([0x7FFFFFFF, 0x80000000, 0x7F800000, 0x807FFFFF], np.uint32), (2, PARAM_128.N))
    fast, worst = _probe(eng, lambda: eng.blind_rotate(lin, tv))
    exact = _with_exact(eng, True, lambda: eng.blind_rotate(lin, tv))
    assert np.array_equal(fast, exact)
    print(f"extreme digits: v5 worst |x - rint(x)| = {worst:.3e}")
    assert worst < 0.25
