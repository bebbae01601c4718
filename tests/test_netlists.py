"""Netlist generators for configs 2-5: plaintext-correct (simulate_plain),
SSA-valid, and their level shapes."""
import numpy as np
import pytest

from paper_2306_11006_b200 import circuit as C
from paper_2306_11006_b200 import netlists as NL
from paper_2306_11006_b200.scheduler import partition_waves


def _bits_signed(v, w):
    return v & ((1 << w) - 1)


def test_multiplier_exhaustive_4bit_and_random_8bit():
    c4 = NL.gen_multiplier(4)
    for a in range(16):
        for b in range(16):
            assert C.simulate_plain(c4, {"a": a, "b": b})["p"] == a * b
    c8 = NL.gen_multiplier(8)
    rng = np.random.default_rng(1)
    for a, b in rng.integers(0, 256, (200, 2)):
        assert C.simulate_plain(c8, {"a": int(a), "b": int(b)})["p"] == int(a) * int(b)
    assert not C.validate(c8)


@pytest.mark.parametrize("n,w", [(1, 4), (3, 4), (7, 8), (20, 16)])
def test_dot_product_signed(n, w):
    c = NL.gen_dot_product(n, w)
    A = 2 * w + max(1, (n - 1).bit_length())
    rng = np.random.default_rng(n * 100 + w)
    for _ in range(20):
        a = rng.integers(-(1 << (w - 1)), 1 << (w - 1), n)
        b = rng.integers(-(1 << (w - 1)), 1 << (w - 1), n)
        asg = {f"a{i}": _bits_signed(int(a[i]), w) for i in range(n)}
        asg.update({f"b{i}": _bits_signed(int(b[i]), w) for i in range(n)})
        y = C.simulate_plain(c, asg)["y"]
        assert NL.to_signed(y, A) == int(np.dot(a.astype(object), b.astype(object)))
    # extremes: most negative values
    asg = {f"a{i}": 1 << (w - 1) for i in range(n)}
    asg.update({f"b{i}": 1 << (w - 1) for i in range(n)})
    assert NL.to_signed(C.simulate_plain(c, asg)["y"], A) == n * (1 << (2 * w - 2))


def test_fc_layer_small():
    n_in, n_out, w = 6, 3, 8
    c = NL.gen_fc_layer(n_in, n_out, w)
    A = 2 * w + max(1, (n_in - 1).bit_length())
    rng = np.random.default_rng(4)
    x = rng.integers(-128, 128, n_in)
    W = rng.integers(-128, 128, (n_out, n_in))
    asg = {f"x{i}": _bits_signed(int(x[i]), w) for i in range(n_in)}
    asg.update({f"w{o}_{i}": _bits_signed(int(W[o, i]), w) for o in range(n_out) for i in range(n_in)})
    out = C.simulate_plain(c, asg)
    for o in range(n_out):
        assert NL.to_signed(out[f"y{o}"], A) == int(W[o].astype(object) @ x.astype(object))


def test_matmul_sigmoid_small():
    n, w, frac = 3, 6, 6
    c = NL.gen_matmul_sigmoid(n, w, frac)
    A = 2 * w + max(1, (n - 1).bit_length())
    rng = np.random.default_rng(5)
    a = rng.integers(-32, 32, (n, n))
    b = rng.integers(-32, 32, (n, n))
    asg = {f"a{i}_{k}": _bits_signed(int(a[i, k]), w) for i in range(n) for k in range(n)}
    asg.update({f"b{k}_{j}": _bits_signed(int(b[k, j]), w) for k in range(n) for j in range(n)})
    out = C.simulate_plain(c, asg)
    cm = a @ b
    for i in range(n):
        for j in range(n):
            assert out[f"s{i}_{j}"] == NL.hard_sigmoid_plain(int(cm[i, j]), A, frac)


def test_generated_netlists_are_wide_and_shallow():
    c = NL.gen_dot_product(64, 16)
    w = partition_waves(c)
    assert len(c.gates) > 20000
    assert w.depth < 120
    assert max(len(x) for x in w.order) > 2000


def test_merge_circuits_side_by_side():
    """Two independent circuits in one netlist: same outputs as each alone, valid,
    text round trip, levels = the deeper circuit's."""
    from paper_2306_11006_b200.scheduler import build_schedule
    a, m = C.gen_adder(8), NL.gen_multiplier(8)
    mc = NL.merge_circuits([("add", a), ("mul", m)])
    assert not C.validate(mc)
    assert C.parse_circuit(C.serialize_circuit(mc)) == mc
    assert len(mc.gates) == len(a.gates) + len(m.gates)
    assert len(build_schedule(mc, 1).waves) == max(len(build_schedule(a, 1).waves), len(build_schedule(m, 1).waves))
    rng = np.random.default_rng(5)
    for _ in range(20):
        vals = {p.name: int(rng.integers(0, 1 << p.width)) for p in mc.inputs}
        out = C.simulate_plain(mc, vals)
        oa = C.simulate_plain(a, {k[4:]: v for k, v in vals.items() if k.startswith("add_")})
        om = C.simulate_plain(m, {k[4:]: v for k, v in vals.items() if k.startswith("mul_")})
        assert out == {**{"add_" + k: v for k, v in oa.items()}, **{"mul_" + k: v for k, v in om.items()}}
