"""Paper-scale netlists on the GPU (BASELINE configs 3 and 5, SURVEY.md §8(d)
parity protocol for big configs): every decrypted output against the
plaintext model, plus >= 16 sampled gates per level recomputed by the oracle's
eval_gate_batch from the GPU's own input ciphertexts and compared bit-exactly
with the GPU's output ciphertexts (the wire store keeps every wire: SSA)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SAMPLES_PER_LEVEL = 16


def _run_and_sample(c, seed, p128_keys, samples=SAMPLES_PER_LEVEL, margin=False):
    import oracle as O
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200.cggi import PARAM_128, decrypt_rows, encrypt_bits
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import evaluate
    from paper_2306_11006_b200.scheduler import build_schedule
    ks = p128_keys
    ek = ks.eval_key()
    rng = np.random.default_rng(seed)
    bits = {p.name: rng.integers(0, 2, p.width).astype(np.uint8) for p in c.inputs}
    srng = SeededRng(1000 * seed)
    inputs = {p.name: encrypt_bits(PARAM_128, ks.lwe_sk, bits[p.name], srng) for p in c.inputs}
    sched = build_schedule(c, 1)
    eng = ek.engine()
    if margin:
        eng.set_margin_probe(True)
    outs, met = evaluate(c, sched, inputs, ek, keep_wires=True)
    plain = C.simulate_plain_bits(c, {k: v[:, None] for k, v in bits.items()})
    for k in plain:
        assert np.array_equal(decrypt_rows(ks.lwe_sk, outs[k]), plain[k][:, 0]), k
    worst = None
    if margin:
        worst = eng.margin()
        eng.set_margin_probe(False)
    # sampled gates: oracle(GPU's operand rows) == GPU's output rows, bit for bit
    okeys = O.Keys.from_params(PARAM_128, ks.bootstrapping_key.data, ks.keyswitch_key.data)
    by_id = {g.id: g for g in c.gates}
    pick = np.random.default_rng(seed + 1)
    checked = 0
    for wave in sched.waves:
        for b in wave:
            ids = np.asarray(b.gate_ids)
            take = ids if samples is None else ids[pick.choice(len(ids), size=min(samples, len(ids)),
                                                                   replace=False)]
            gates = [by_id[int(g)] for g in take]
            ar = len(gates[0].operands)
            ops = [eng.wires_get(np.asarray([g.operands[k] for g in gates], np.int64)) for k in range(ar)]
            want = O.eval_gate_batch(b.opcode.value, ops, okeys, count=len(gates), threads=16)
            got = eng.wires_get(np.asarray(take, np.int64))
            assert np.array_equal(got, want), f"level gate batch {b.opcode} differs from the oracle"
            checked += len(gates)
    eng.wires_alloc(0)
    return met, checked, worst


def test_config3_dot_product_500(p128_keys):
    from paper_2306_11006_b200 import netlists as NL
    c = NL.gen_dot_product(500)
    met, checked, _ = _run_and_sample(c, 3, p128_keys)
    assert met.bootstrap_count == 767874 and checked >= 16 * 100


def test_config5_matmul_sigmoid(p128_keys):
    from paper_2306_11006_b200 import netlists as NL
    c = NL.gen_matmul_sigmoid(10)
    met, checked, _ = _run_and_sample(c, 5, p128_keys)
    assert met.total_gates == 1533002 and checked >= 16 * 90


def test_config2_multiplier8_every_gate(p128_keys):
    """Config 2's 8x8 multiplier (320 gates, 35 levels): EVERY gate's output
    ciphertext recomputed by the oracle from the GPU's operands, bit-exact."""
    from paper_2306_11006_b200 import netlists as NL
    c = NL.gen_multiplier(8)
    met, checked, _ = _run_and_sample(c, 80, p128_keys, samples=None)
    assert checked == len(c.gates) == 320 and met.bootstrap_count == 320


def test_config2_adder8_every_gate(p128_keys):
    from paper_2306_11006_b200 import circuit as C
    c = C.gen_adder(8)
    met, checked, _ = _run_and_sample(c, 81, p128_keys, samples=None)
    assert checked == len(c.gates) == 40 and met.bootstrap_count == 39


def test_config2_combined_netlist_every_gate(p128_keys):
    """Config 2's two circuits as ONE level-scheduled netlist (netlists.merge_circuits):
    35 levels, every gate recomputed by the oracle from the GPU's operands, bit-exact."""
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200 import netlists as NL
    c = NL.merge_circuits([("add", C.gen_adder(8)), ("mul", NL.gen_multiplier(8))])
    met, checked, _ = _run_and_sample(c, 82, p128_keys, samples=None)
    assert checked == len(c.gates) == 360 and met.bootstrap_count == 359


def test_config4_fc_layer_sampled_and_margin(p128_keys):
    """Config 4 (fc layer 256 -> 30, w[30][256]: 11.79M gates, 117 levels, the
    largest single-GPU workload): every decrypted output exact, 16 sampled
    gates of every level batch bit-exact against the oracle, and the FP64
    rounding margin over all 11.79M bootstraps measured by the probe build."""
    from paper_2306_11006_b200 import netlists as NL
    c = NL.gen_fc_layer(256, 30)
    met, checked, worst = _run_and_sample(c, 4, p128_keys, margin=True)
    assert met.total_gates == 11792041 and checked >= 16 * 110
    print(f"config 4 rounding margin: worst |x - rint(x)| = {worst:.3e}")
    assert worst < 0.1
