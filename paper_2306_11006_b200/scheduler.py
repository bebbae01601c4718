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


def circuit_arrays(c: Circuit):
    """(ids, opcode codes, operands (G, 3) -1 padded, arity) in circuit order,
    built in one pass over the Gate objects and cached on the circuit."""
    cached = c.__dict__.get("_plan_arrays")
    if cached is not None:
        return cached
    G = len(c.gates)
    ids = np.fromiter((g.id for g in c.gates), dtype=np.int64, count=G)
    codes = np.fromiter((_OPC[as_kind(g.opcode)] for g in c.gates), dtype=np.int32, count=G)
    ar = np.fromiter((len(g.operands) for g in c.gates), dtype=np.int32, count=G)
    flat = np.fromiter((w for g in c.gates for w in (*g.operands, -1, -1, -1)[:3]), dtype=np.int64, count=3 * G)
    out = (ids, codes, flat.reshape(G, 3), ar)
    c.__dict__["_plan_arrays"] = out
    return out


def gate_arrays(c: Circuit):
    """(ids, opcodes, operands (G,3) with -1 padding) as numpy arrays."""
    ids, codes, opnd, _ = circuit_arrays(c)
    return ids, codes, opnd


_KINDS = list(GateKind)
_OPC = {k: i for i, k in enumerate(_KINDS)}


def _levels_native(pos: np.ndarray):
    """gw_levels from the engine library (host code, no GPU); None if unavailable."""
    try:
        import ctypes
        from .engine import load_library
        lib = load_library()
    except Exception:
        return None
    pos = np.ascontiguousarray(pos, dtype=np.int64)
    lv = np.empty(pos.shape[0], dtype=np.int32)
    rc = lib.gw_levels(pos.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), pos.shape[0],
                       lv.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)))
    return lv.astype(np.int64) if rc == 0 else None


def wave_index(c: Circuit) -> np.ndarray:
    """Longest-path level of every gate (same rule as the reference's FIFO
    walk: level = 1 + max level of gate operands, 0 if only inputs feed it).

    Gates are in SSA execution order, so one pass in gate order suffices
    (native `gw_levels` when the engine library is present); operands that are
    not gate outputs (circuit inputs) contribute nothing.
    """
    ids, _, opnd, _ = circuit_arrays(c)
    if len(ids) == 0:
        return np.zeros(0, dtype=np.int64)
    top = int(max(ids.max(), opnd.max(), c.max_wire)) + 1
    pos_of_wire = np.full(top + 1, -1, dtype=np.int64)
    pos_of_wire[ids] = np.arange(len(ids))
    pos = np.where(opnd >= 0, pos_of_wire[np.where(opnd >= 0, opnd, top)], -1)
    # SSA order check: an operand defined by a LATER gate means not sequential
    late = pos >= np.arange(len(ids))[:, None]
    if late.any():
        k = int(np.argwhere(late)[0][0])
        w = int(opnd[k][np.argmax(late[k])])
        raise SchedulerError("circuit is not a valid sequential form: gate "
                             f"{int(ids[k])} reads wire {w} defined later")
    lv = _levels_native(pos)
    if lv is not None:
        return lv
    lv = np.zeros(len(ids), dtype=np.int64)
    for k in range(len(ids)):
        m = -1
        for p in pos[k]:
            if p >= 0 and lv[p] > m:
                m = lv[p]
        lv[k] = m + 1
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
    """Waves -> opcode groups in first-seen order -> <= `workers` contiguous
    slices per group (scheduler.py:170-178), vectorised over the circuit arrays."""
    if workers < 1:
        raise SchedulerError(f"worker count must be >= 1, got {workers}")
    ids, codes, _, _ = circuit_arrays(c)
    G = len(ids)
    if G == 0:
        return Schedule(waves=(), workers=workers)
    lv = wave_index(c)
    depth = int(lv.max()) + 1
    nk = len(_KINDS)
    key = lv * nk + codes
    first = np.full(depth * nk, G, dtype=np.int64)
    np.minimum.at(first, key, np.arange(G, dtype=np.int64))
    # stable order: wave, then the opcode's first appearance in the wave, then position
    order = np.lexsort((np.arange(G), first[key], lv))
    ks = key[order]
    starts = np.concatenate(([0], np.flatnonzero(np.diff(ks)) + 1, [G]))
    gid_sorted = ids[order]
    waves: list[list[Batch]] = [[] for _ in range(depth)]
    for a, b in zip(starts[:-1].tolist(), starts[1:].tolist()):
        w, op = divmod(int(ks[a]), nk)
        m = b - a
        q, r = divmod(m, workers)
        s0 = a
        for wk in range(workers):
            size = q + (1 if wk < r else 0)
            if size == 0:
                break
            waves[w].append(Batch(opcode=_KINDS[op], gate_ids=tuple(gid_sorted[s0:s0 + size].tolist()),
                                  worker=wk))
            s0 += size
    return Schedule(waves=tuple(tuple(w) for w in waves), workers=workers)


def bootstraps_of(schedule: Schedule) -> int:
    return sum(len(b.gate_ids) * BOOTSTRAPS_PER_GATE[as_kind(b.opcode)]
               for w in schedule.waves for b in w)


def arity(kind) -> int:
    return GATE_ARITY[as_kind(kind)]
