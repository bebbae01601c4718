"""Circuit IR and the level partitioner: same semantics as the reference's
circuit.py / scheduler.py (tests modelled on tests/test_circuit.py and
tests/test_scheduler.py of the reference)."""
import numpy as np
import pytest

from paper_2306_11006_b200 import circuit as C
from paper_2306_11006_b200.cggi import GateKind
from paper_2306_11006_b200.runtime import EvaluateError, compile_plan
from paper_2306_11006_b200.scheduler import (SchedulerError, build_schedule, partition_waves,
                                             split_batches)


def test_parse_serialize_roundtrip():
    for c in (C.gen_adder(8), C.gen_mux_tree(3), C.gen_flat(10, GateKind.NOT), C.gen_not_chain(4)):
        assert C.parse_circuit(C.serialize_circuit(c)) == c


def test_parser_diagnostics_carry_line_numbers():
    bad = "input a 2\ngate 2 AND 0\ngate 3 FOO 0,1\noutput y 9\n"
    with pytest.raises(C.CircuitError) as e:
        C.parse_circuit(bad)
    msgs = [str(d) for d in e.value.diagnostics]
    assert any(m.startswith("line 2") for m in msgs)
    assert any("unknown opcode" in m for m in msgs)
    assert any("undefined wire 9" in m for m in msgs)


def test_adder8_shape_matches_reference():
    """tests/test_circuit.py:162-182 of the reference: 40 gates, 15 levels,
    16 XOR / 16 AND / 7 OR / 1 CONST0."""
    c = C.gen_adder(8)
    assert len(c.gates) == 40
    hist = {}
    for g in c.gates:
        hist[g.opcode] = hist.get(g.opcode, 0) + 1
    assert hist == {GateKind.XOR: 16, GateKind.AND: 16, GateKind.OR: 7, GateKind.CONST0: 1}
    assert partition_waves(c).depth == 15
    assert max(C.gate_levels(c).values()) + 1 == 15


def test_simulate_plain_adder():
    c = C.gen_adder(8)
    for a, b in ((0, 0), (255, 1), (77, 200), (128, 128)):
        assert C.simulate_plain(c, {"a": a, "b": b})["s"] == a + b


def test_diamond_waves():
    c = C.parse_circuit("input x 2\ngate 2 AND 0,1\ngate 3 OR 0,1\ngate 4 XOR 2,3\n"
                        "gate 5 NOT 4\noutput y 5\n")
    w = partition_waves(c)
    assert w.order == ((2, 3), (4,), (5,))


def test_wave_equals_gate_levels_on_random_dags():
    rng = np.random.default_rng(3)
    kinds = [GateKind.AND, GateKind.XOR, GateKind.NOT, GateKind.MUX, GateKind.CONST1]
    for _ in range(20):
        lines = ["input x 6"]
        nxt = 6
        for _ in range(int(rng.integers(5, 60))):
            k = kinds[int(rng.integers(len(kinds)))]
            ar = {GateKind.AND: 2, GateKind.XOR: 2, GateKind.NOT: 1, GateKind.MUX: 3,
                  GateKind.CONST1: 0}[k]
            ops = ",".join(str(int(rng.integers(0, nxt))) for _ in range(ar))
            lines.append(f"gate {nxt} {k.value} {ops}".rstrip())
            nxt += 1
        lines.append(f"output y {nxt - 1}")
        c = C.parse_circuit("\n".join(lines))
        lv = C.gate_levels(c)
        w = partition_waves(c)
        for gid, wave in w.wave_of.items():
            assert lv[gid] == wave


def test_split_is_contiguous_and_balanced():
    ids = list(range(23))
    b = split_batches({GateKind.AND: ids}, 4)
    sizes = [len(x.gate_ids) for x in b]
    assert sizes == [6, 6, 6, 5]
    assert [g for x in b for g in x.gate_ids] == ids
    with pytest.raises(SchedulerError):
        split_batches({GateKind.AND: ids}, 0)


def test_paper_wave_split():
    """Acceptance C6 of the reference: 2125 AND / 25000 OR / 16750 NOT on 2 workers."""
    groups = {GateKind.AND: list(range(2125)), GateKind.OR: list(range(25000)),
              GateKind.NOT: list(range(16750))}
    b = split_batches(groups, 2)
    sizes = {(x.opcode, x.worker): len(x.gate_ids) for x in b}
    assert sizes[(GateKind.AND, 0)] == 1063 and sizes[(GateKind.AND, 1)] == 1062
    assert sizes[(GateKind.OR, 0)] == 12500 and sizes[(GateKind.NOT, 1)] == 8375


def test_compile_plan_static_ssa_checks():
    c = C.gen_adder(3)
    plan = compile_plan(c, build_schedule(c, 2))
    assert plan.gates == len(c.gates)
    assert plan.bootstraps == sum(1 for g in c.gates if g.opcode not in (GateKind.CONST0,))
    other = build_schedule(C.gen_adder(4), 1)
    with pytest.raises(EvaluateError):
        compile_plan(c, other)
