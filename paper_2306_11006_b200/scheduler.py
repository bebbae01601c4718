"""Level (wave) partitioning and per-opcode splitting -- the netlist partitioner.

Same schedule as gatewave/scheduler.py (reference): wave 0 holds gates fed only
by circuit inputs, wave w+1 the gates whose deepest gate operand sits in wave
w (FIFO topological order, scheduler.py:57-102); each wave is grouped by
opcode in first-seen order (:105-112) and every group is cut into at most K
contiguous slices whose sizes differ by at most one, earlier slices larger
(:133-157).  Here K counts GPUs: slice k of every opcode group runs on GPU k.

Levels are computed in one pass over the SSA gate list with array lookups
(gates are in execution order, so no work queue is needed).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np

from .cggi import BOOTSTRAPS_PER_GATE, GATE_ARITY, GateKind, as_kind
from .circuit import Circuit


class SchedulerError(ValueError):
    pass


@dataclass(frozen=True)
class Waves:
    order: tuple[tuple[int, ...], ...]
    wave_of: Mapping[int, int] = field(hash=False)

    @property
    def depth(self) -> int:
        return len(self.order)


@dataclass(frozen=True)
class Batch:
    opcode: GateKind
    gate_ids: tuple[int, ...]
    worker: int


@dataclass(frozen=True)
class Schedule:
    waves: tuple[tuple[Batch, ...], ...]
    workers: int

    @property
    def batch_count(self) -> int:
        return sum(len(w) for w in self.waves)


def gate_arrays(c: Circuit):
    """(ids, opcodes, operands (G,3) with -1 padding) as numpy arrays."""
    G = len(c.gates)
    ids = np.fromiter((g.id for g in c.gates), dtype=np.int64, count=G)
    codes = np.fromiter((_OPC[as_kind(g.opcode)] for g in c.gates), dtype=np.int32, count=G)
    opnd = np.full((G, 3), -1, dtype=np.int64)
    for k, g in enumerate(c.gates):
        for j, w in enumerate(g.operands):
            opnd[k, j] = w
    return ids, codes, opnd


_KINDS = list(GateKind)
_OPC = {k: i for i, k in enumerate(_KINDS)}


def wave_index(c: Circuit) -> np.ndarray:
    """Longest-path level of every gate (same rule as the reference's FIFO
    walk: level = 1 + max level of gate operands, 0 if only inputs feed it).

    Gates are in SSA execution order, so one pass in gate order suffices;
    operands that are not gate outputs (circuit inputs) contribute nothing.
    """
    ids, _, opnd = gate_arrays(c)
    if len(ids) == 0:
        return np.zeros(0, dtype=np.int64)
    top = int(max(ids.max(), opnd.max(), c.max_wire)) + 1
    level_of_wire = np.full(top + 1, -1, dtype=np.int64)  # -1: input / undefined
    pos_of_wire = np.full(top + 1, -1, dtype=np.int64)
    pos_of_wire[ids] = np.arange(len(ids))
    lv = np.zeros(len(ids), dtype=np.int64)
    # SSA order check: an operand defined by a LATER gate means not sequential
    for k in range(len(ids)):
        m = -1
        for w in opnd[k]:
            if w < 0:
                continue
            p = pos_of_wire[w]
            if p >= k:
                raise SchedulerError(
                    "circuit is not a valid sequential form: gate "
                    f"{int(ids[k])} reads wire {int(w)} defined later")
            if p >= 0 and level_of_wire[w] > m:
                m = level_of_wire[w]
        lv[k] = m + 1
        level_of_wire[ids[k]] = lv[k]
    return lv


def partition_waves(c: Circuit) -> Waves:
    lv = wave_index(c)
    depth = int(lv.max()) + 1 if lv.size else 0
    order: list[list[int]] = [[] for _ in range(depth)]
    wave_of = {}
    for g, w in zip(c.gates, lv.tolist()):
        order[w].append(g.id)
        wave_of[g.id] = w
    return Waves(order=tuple(tuple(o) for o in order), wave_of=wave_of)


def batch_by_opcode(wave_gates: Sequence[int], c: Circuit) -> dict[GateKind, list[int]]:
    by_id = {g.id: g for g in c.gates}
    groups: dict[GateKind, list[int]] = {}
    for gid in wave_gates:
        groups.setdefault(as_kind(by_id[gid].opcode), []).append(gid)
    return groups


def split_batches(groups: Mapping[GateKind, Sequence[int]], workers: int) -> list[Batch]:
    """Contiguous near-equal slices per opcode group, larger slices first."""
    if workers < 1:
        raise SchedulerError(f"worker count must be >= 1, got {workers}")
    out: list[Batch] = []
    for op, ids in groups.items():
        m = len(ids)
        q, r = divmod(m, workers)
        start = 0
        for w in range(workers):
            size = q + (1 if w < r else 0)
            if size == 0:
                break
            out.append(Batch(opcode=op, gate_ids=tuple(ids[start:start + size]), worker=w))
            start += size
    return out


def build_schedule(c: Circuit, workers: int) -> Schedule:
    if workers < 1:
        raise SchedulerError(f"worker count must be >= 1, got {workers}")
    waves = partition_waves(c)
    by_id = {g.id: g for g in c.gates}
    out = []
    for wg in waves.order:
        groups: dict[GateKind, list[int]] = {}
        for gid in wg:
            groups.setdefault(as_kind(by_id[gid].opcode), []).append(gid)
        out.append(tuple(split_batches(groups, workers)))
    return Schedule(waves=tuple(out), workers=workers)


def bootstraps_of(schedule: Schedule) -> int:
    return sum(len(b.gate_ids) * BOOTSTRAPS_PER_GATE[as_kind(b.opcode)]
               for w in schedule.waves for b in w)


def arity(kind) -> int:
    return GATE_ARITY[as_kind(kind)]
