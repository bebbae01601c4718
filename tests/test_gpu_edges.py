"""Edge cases the reference's gate API accepts (cggi.py:785-854): empty
batches of every kind (and a zero CONST count), single-row batches, and a
netlist without a single bootstrap -- on the B200, against the oracle."""
import numpy as np
import pytest

from conftest import MINI

pytestmark = pytest.mark.gpu

KINDS = ["AND", "OR", "NAND", "NOR", "XOR", "XNOR", "NOT", "MUX", "CONST0", "CONST1", "COPY"]


@pytest.mark.parametrize("kind", KINDS)
def test_empty_batch_every_kind(kind, p128_keys):
    from paper_2306_11006_b200.cggi import GATE_ARITY, PARAM_128, GateKind, OpCounter, eval_gate_batch
    k = GateKind(kind)
    ops = [np.zeros((0, PARAM_128.n + 1), np.uint32)] * GATE_ARITY[k]
    ctr = OpCounter()
    out = eval_gate_batch(k, ops, p128_keys, ctr, count=0)
    assert out.shape == (0, PARAM_128.n + 1) and out.dtype == np.uint32
    assert (ctr.ntt_forward, ctr.ntt_inverse, ctr.bootstraps) == (0, 0, 0)


@pytest.mark.parametrize("kind", KINDS)
def test_single_row_every_kind_p128(kind, p128_keys):
    import oracle as O
    from paper_2306_11006_b200.cggi import GATE_ARITY, PARAM_128, GateKind, encrypt_bits, eval_gate_batch
    from paper_2306_11006_b200.rng import SeededRng
    ks = p128_keys
    k = GateKind(kind)
    rng = SeededRng(99)
    ops = [encrypt_bits(PARAM_128, ks.lwe_sk, np.array([j & 1], np.uint8), rng) for j in range(GATE_ARITY[k])]
    out = eval_gate_batch(k, ops, ks, count=1)
    okeys = O.Keys.from_params(PARAM_128, ks.bootstrapping_key.data, ks.keyswitch_key.data)
    assert np.array_equal(out, O.eval_gate_batch(kind, ops, okeys, count=1, threads=4))


def test_netlist_without_bootstraps(mini_keys):
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200.cggi import decrypt_rows, encrypt_bits
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import evaluate
    from paper_2306_11006_b200.scheduler import build_schedule
    c = C.gen_not_chain(9)
    x = encrypt_bits(MINI, mini_keys.lwe_sk, np.array([1], np.uint8), SeededRng(5))
    outs, met = evaluate(c, build_schedule(c, 2), {c.inputs[0].name: x}, mini_keys)
    assert met.bootstrap_count == 0 and met.ntt_forward_count == 0
    (name, rows), = outs.items()
    assert decrypt_rows(mini_keys.lwe_sk, rows)[0] == 0          # nine NOTs of 1
