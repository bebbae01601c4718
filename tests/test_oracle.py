"""The oracle (oracle/, a C restatement of the reference's algorithm) pinned
against golden vectors produced by the reference itself (make_golden.py)."""
import numpy as np
import pytest

import oracle as O
from conftest import MINI


def test_ntt_matches_reference_mini(golden_mini):
    assert np.array_equal(O.ntt_forward(golden_mini["ntt_in"]), golden_mini["ntt_fwd"])
    assert np.array_equal(O.ntt_inverse(golden_mini["ntt_in"]), golden_mini["ntt_inv"])


def test_ntt_tables_match_reference(golden_mini):
    t = O.tables(64)
    assert np.array_equal(t.psi_brv, golden_mini["psi_brv"])
    assert np.array_equal(t.ipsi_brv, golden_mini["ipsi_brv"])


def test_ntt_roundtrip_and_order_n1024(golden_p128):
    fwd = O.ntt_forward(golden_p128["ntt_in"])
    assert np.array_equal(fwd, golden_p128["ntt_fwd"])
    assert np.array_equal(O.ntt_inverse(fwd), golden_p128["ntt_in"])


def test_bk_ntt_matches_reference_mini(golden_mini):
    assert np.array_equal(O.bk_to_ntt(golden_mini["bk_data"]), golden_mini["bk_ntt"])


def test_bk_ntt_slab_matches_reference_p128(golden_p128, p128_keys):
    slab = O.bk_to_ntt(p128_keys.bootstrapping_key.data[:1])[0]
    assert np.array_equal(slab, golden_p128["bk_ntt_slab0"])


def test_blind_rotate_matches_reference_mini(golden_mini):
    acc = O.blind_rotate(golden_mini["br_lin"], golden_mini["br_tv"], golden_mini["bk_ntt"], 9, 2)
    assert np.array_equal(acc, golden_mini["br_acc"])


def test_extract_and_keyswitch_match_reference_mini(golden_mini):
    assert np.array_equal(O.extract(golden_mini["extract_in"]), golden_mini["extract_out"])
    assert np.array_equal(O.keyswitch(golden_mini["ks_in"], golden_mini["ksk_data"], 8, 2),
                          golden_mini["ks_out"])


@pytest.mark.parametrize("kind", sorted(O.GATE_ARITY))
def test_gate_batch_matches_reference_mini(golden_mini, kind):
    keys = O.Keys.from_params(MINI, golden_mini["bk_data"], golden_mini["ksk_data"])
    ops = [golden_mini["op0"], golden_mini["op1"], golden_mini["op2"]][:O.GATE_ARITY[kind]]
    assert np.array_equal(O.eval_gate_batch(kind, ops, keys, count=8), golden_mini[f"gate_{kind}"])


def test_first_config1_gates_match_reference_p128(golden_p128, p128_keys):
    """Two PARAM_128 bootstraps: raw accumulators and refreshed samples."""
    from paper_2306_11006_b200.cggi import PARAM_128
    keys = O.Keys.from_params(PARAM_128, p128_keys.bootstrapping_key.data,
                              p128_keys.keyswitch_key.data)
    acc = O.blind_rotate(golden_p128["lin2"], keys.test_vector(), keys.bk_ntt, 9, 2)
    assert np.array_equal(acc, golden_p128["acc2"])
    out = O.keyswitch(O.extract(acc), keys.ksk, 8, 2)
    assert np.array_equal(out, golden_p128["out_head"][:2])


def test_negacyclic_mul_naive_matches_reference(golden_mini):
    """The exact host product used by keygen equals the reference's schoolbook oracle."""
    from paper_2306_11006_b200.cggi import negacyclic_small_times_torus
    for p, q, want in zip(golden_mini["nm_p"], golden_mini["nm_q"], golden_mini["nm_out"]):
        assert np.array_equal(negacyclic_small_times_torus(p, q), want)
