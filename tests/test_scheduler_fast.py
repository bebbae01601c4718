"""The vectorised partitioner (native gw_levels + numpy grouping) against a
gate-by-gate restatement of the reference's rules (gatewave/scheduler.py:57-178):
levels by longest path, opcode groups in first-seen order per wave, contiguous
slices differing by at most one, earlier slices larger."""
import numpy as np
import pytest

from paper_2306_11006_b200 import circuit as C
from paper_2306_11006_b200 import netlists as NL
from paper_2306_11006_b200.cggi import GateKind
from paper_2306_11006_b200.scheduler import SchedulerError, build_schedule, wave_index


def _naive(c, workers):
    level = {}
    for g in c.gates:
        level[g.id] = 1 + max((level[w] for w in g.operands if w in level), default=-1)
    depth = max(level.values()) + 1
    waves = []
    for w in range(depth):
        groups = {}
        for g in c.gates:
            if level[g.id] == w:
                groups.setdefault(g.opcode, []).append(g.id)
        out = []
        for op, gids in groups.items():
            q, r = divmod(len(gids), workers)
            s = 0
            for k in range(workers):
                n = q + (1 if k < r else 0)
                if n == 0:
                    break
                out.append((op, tuple(gids[s:s + n]), k))
                s += n
        waves.append(out)
    return waves


def _random_circuit(seed, n_in=6, n_gates=120):
    rng = np.random.default_rng(seed)
    nb = NL.NetBuilder()
    wires = nb.add_input("x", n_in)
    kinds = [GateKind.AND, GateKind.OR, GateKind.XOR, GateKind.NAND, GateKind.NOT, GateKind.MUX,
             GateKind.COPY, GateKind.XNOR]
    for _ in range(n_gates):
        k = kinds[rng.integers(len(kinds))]
        ar = {GateKind.NOT: 1, GateKind.COPY: 1, GateKind.MUX: 3}.get(k, 2)
        ops = [wires[rng.integers(len(wires))] for _ in range(ar)]
        wires.append(nb.gate(k, *ops))
    nb.add_output("y", wires[-8:])
    return nb.build()


@pytest.mark.parametrize("workers", [1, 2, 3, 8])
@pytest.mark.parametrize("make", [lambda: C.gen_adder(8), lambda: NL.gen_multiplier(6),
                                  lambda: C.gen_mux_tree(4), lambda: _random_circuit(1),
                                  lambda: _random_circuit(2, 3, 300)])
def test_build_schedule_matches_reference_rules(make, workers):
    c = make()
    got = [[(b.opcode, b.gate_ids, b.worker) for b in w] for w in build_schedule(c, workers).waves]
    assert got == _naive(c, workers)


def test_wave_index_rejects_non_sequential():
    c = C.Circuit(inputs=(C.Port("a", (0,)),), outputs=(C.Port("y", (2,)),),
                  gates=(C.Gate(1, GateKind.NOT, (2,)), C.Gate(2, GateKind.NOT, (0,))))
    with pytest.raises(SchedulerError):
        wave_index(c)
