"""The single-sample public entry points (cggi.py:730-777, 857-873 of the
reference) on the B200, against golden vectors the unmodified reference wrote
(tests/golden/make_golden_api.py): gate_bootstrap (the engine's BOOTSTRAP
opcode), blind_rotate, keyswitch and eval_gate for every gate kind, with the
exact counter tallies.  Bit-exact: all arithmetic is integer mod 2^32."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, MINI

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    with open(os.path.join(GOLDEN, "api.json")) as f:
        js = json.load(f)
    return dict(np.load(os.path.join(GOLDEN, "api.npz"))), js


def _keys(tag, mini_keys, p128_keys):
    return mini_keys if tag == "mini" else p128_keys


def _params(tag):
    from paper_2306_11006_b200.cggi import PARAM_128
    return MINI if tag == "mini" else PARAM_128


@pytest.mark.parametrize("tag", ["mini", "p128"])
def test_gate_bootstrap_matches_reference(api, tag, mini_keys, p128_keys):
    from paper_2306_11006_b200.cggi import LweCiphertext, OpCounter, gate_bootstrap
    g, js = api
    ks = _keys(tag, mini_keys, p128_keys)
    ctr = OpCounter()
    got = np.stack([gate_bootstrap(LweCiphertext(row), ks, ctr).vec for row in g[f"{tag}_ct0"]])
    assert np.array_equal(got, g[f"{tag}_gate_bootstrap"])
    assert [ctr.ntt_forward, ctr.ntt_inverse, ctr.bootstraps] == js[tag]["gate_bootstrap"]


@pytest.mark.parametrize("tag", ["mini", "p128"])
def test_blind_rotate_wrapper_matches_reference(api, tag, mini_keys, p128_keys):
    from paper_2306_11006_b200.cggi import (LweCiphertext, OpCounter, TlweCiphertext, blind_rotate,
                                            sample_extract)
    g, js = api
    ks = _keys(tag, mini_keys, p128_keys)
    p = _params(tag)
    ek = ks.eval_key()
    tv_mu = np.zeros((2, p.N), np.uint32)
    tv_mu[1, :] = p.mu
    ctr = OpCounter()
    got = []
    for row in g[f"{tag}_ct1"]:
        for tv in (tv_mu, g[f"{tag}_tv_rand"]):
            got.append(blind_rotate(TlweCiphertext(tv), LweCiphertext(row), ek.bk, ek.tables, ctr).data)
    got = np.stack(got)
    assert np.array_equal(got, g[f"{tag}_blind_rotate"])
    assert [ctr.ntt_forward, ctr.ntt_inverse] == js[tag]["blind_rotate"]
    ext = np.stack([sample_extract(TlweCiphertext(a)).vec for a in got])
    assert np.array_equal(ext, g[f"{tag}_sample_extract"])


@pytest.mark.parametrize("tag", ["mini", "p128"])
def test_keyswitch_wrapper_matches_reference(api, tag, mini_keys, p128_keys):
    from paper_2306_11006_b200.cggi import LweCiphertext, keyswitch
    g, _ = api
    ek = _keys(tag, mini_keys, p128_keys).eval_key()
    got = np.stack([keyswitch(LweCiphertext(e), ek.ksk).vec for e in g[f"{tag}_sample_extract"]])
    assert np.array_equal(got, g[f"{tag}_keyswitch"])


@pytest.mark.parametrize("tag", ["mini", "p128"])
@pytest.mark.parametrize("kind", ["AND", "OR", "NAND", "NOR", "XOR", "XNOR", "NOT", "MUX",
                                  "CONST0", "CONST1", "COPY"])
def test_eval_gate_every_kind_matches_reference(api, tag, kind, mini_keys, p128_keys):
    from paper_2306_11006_b200.cggi import GATE_ARITY, GateKind, LweCiphertext, OpCounter, eval_gate
    g, js = api
    ks = _keys(tag, mini_keys, p128_keys)
    k = GateKind(kind)
    ctr = OpCounter()
    out = eval_gate(k, [LweCiphertext(g[f"{tag}_ct{j}"][0]) for j in range(GATE_ARITY[k])], ks, ctr)
    assert np.array_equal(out.vec, g[f"{tag}_eval_gate_{kind}"])
    assert [ctr.ntt_forward, ctr.ntt_inverse, ctr.bootstraps] == js[tag][f"eval_gate_{kind}"]
