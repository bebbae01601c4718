"""Multi-GPU netlist evaluation: per-rank level slices + cross-GPU wire exchange.

One process per GPU (torch.distributed; NCCL over NVLink on B200, gloo on CPU
for tests).  The reference's partitioner assigns slice k of every opcode
group of every level to worker k (scheduler.py:133-157); here worker k runs on
rank k mod world.  Keys are replicated.  After each level a static plan moves
only the produced wires that some OTHER rank reads in a later level, or that
are circuit outputs (every rank returns the full outputs): grouped
point-to-point sends, each row only to the ranks that read it (SURVEY.md
§8(e); ~2.5 KB per wire), scattered into each rank's device wire store.
Levels stay stream-ordered: run level -> pack -> ncclSend/ncclRecv per peer
-> unpack -> next level, all on the engine stream (gw_exchange_enqueue).
"""
from __future__ import annotations

import contextlib
import time
import weakref
from dataclasses import dataclass

import numpy as np

from .cggi import EvalKey
from .circuit import Circuit
from .runtime import EvaluateError, Metrics
from .scheduler import Schedule


@dataclass
class ExchangePlan:
    """Point-to-point exchange plan, identical on every rank.

    counts[L, q, r] = wires rank q produces at level L that rank r needs (a gate
    on r reads them later, or they are circuit outputs, which every rank
    returns); ids lists them in (L, q, r) order, schedule order inside a cell."""
    world: int
    counts: np.ndarray     # (levels, world, world) int64
    ids: np.ndarray        # (counts.sum(),) int64
    offsets: np.ndarray    # (levels * world * world + 1,) int64 into ids

    def cell(self, level: int, src: int, dst: int) -> np.ndarray:
        k = (level * self.world + src) * self.world + dst
        return self.ids[self.offsets[k]:self.offsets[k + 1]]

    def bytes_per_level(self, row_bytes: int) -> list[int]:
        """Bytes that cross between GPUs per level (each row once per consumer rank)."""
        return [int(x) * row_bytes for x in self.counts.sum(axis=(1, 2))]


def owners(c: Circuit, schedule: Schedule, world: int) -> dict[int, int]:
    own = {}
    for wave in schedule.waves:
        for b in wave:
            for gid in b.gate_ids:
                own[gid] = b.worker % world
    return own


def exchange_plan(c: Circuit, schedule: Schedule, world: int) -> ExchangePlan:
    """Per level, per (producer rank, consumer rank), the produced wires the
    consumer needs.  Vectorised over the circuit arrays (numpy)."""
    from .runtime import _circuit_arrays
    ids, _, opnd, _ = _circuit_arrays(c)
    nb = [(wi, b) for wi, wave in enumerate(schedule.waves) for b in wave]
    sizes = np.fromiter((len(b.gate_ids) for _, b in nb), dtype=np.int64, count=len(nb))
    total = int(sizes.sum())
    gid = np.fromiter((g for _, b in nb for g in b.gate_ids), dtype=np.int64, count=total)
    wave = np.repeat(np.fromiter((wi for wi, _ in nb), dtype=np.int64, count=len(nb)), sizes)
    rank = np.repeat(np.fromiter((b.worker % world for _, b in nb), dtype=np.int64, count=len(nb)), sizes)
    levels = len(schedule.waves)
    top = int(max(c.max_wire, ids.max() if len(ids) else 0, opnd.max() if opnd.size else 0)) + 1
    own = np.full(top, -1, dtype=np.int64)
    own[gid] = rank
    lvl = np.full(top, -1, dtype=np.int64)
    lvl[gid] = wave
    order = np.full(top, -1, dtype=np.int64)   # position in schedule order
    order[gid] = np.arange(total)
    # (wire, consumer rank) pairs: cross-rank operand reads ...
    reader = np.repeat(own[ids], 3)
    w = opnd.reshape(-1)
    valid = w >= 0
    w, reader = w[valid], reader[valid]
    cross = (own[w] >= 0) & (own[w] != reader)
    pw, pr = w[cross], reader[cross]
    # ... and circuit outputs, needed by every rank
    outs = np.unique(np.concatenate([np.asarray(p.wires, np.int64) for p in c.outputs])
                     if c.outputs else np.zeros(0, np.int64))
    outs = outs[own[outs] >= 0]
    if len(outs) and world > 1:
        ow = np.repeat(outs, world)
        orr = np.tile(np.arange(world, dtype=np.int64), len(outs))
        keep = orr != own[ow]
        pw, pr = np.concatenate([pw, ow[keep]]), np.concatenate([pr, orr[keep]])
    if len(pw):
        pairs = np.unique(pw * world + pr)
        pw, pr = pairs // world, pairs % world
    srt = np.lexsort((order[pw], pr, own[pw], lvl[pw]))
    pw, pr = pw[srt], pr[srt]
    cellk = (lvl[pw] * world + own[pw]) * world + pr
    counts = np.bincount(cellk, minlength=levels * world * world).astype(np.int64)
    offsets = np.zeros(levels * world * world + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(counts)
    return ExchangePlan(world=world, counts=counts.reshape(levels, world, world), ids=pw.astype(np.int64),
                        offsets=offsets)


class _DeviceLevels:
    """Adapter: the CUDA engine running one rank's level plan on a torch wire store."""

    def __init__(self, eng, plan, slots: int, device):
        import torch
        self.eng = eng
        self.stream = torch.cuda.current_stream(device)
        if self.stream.cuda_stream == 0:
            self.stream = torch.cuda.Stream(device)
            torch.cuda.set_stream(self.stream)
        self.eng.set_stream(self.stream.cuda_stream)
        self.wires = torch.zeros((slots, self.eng.row_stride), dtype=torch.int32, device=device)
        self.eng.wires_attach(self.wires.data_ptr(), slots, self.eng.row_stride)
        self.handle = self.eng.plan_create(plan.level_offsets, plan.opcodes, plan.operands,
                                           plan.out_ids)
        self.xplan = None

    def run_level(self, level: int):
        self.handle.run(level, level + 1)

    def exchange_plan(self, xp: ExchangePlan, rank: int):
        """Device exchange plan: the level's rows are packed / unpacked by engine
        kernels on the engine stream (gw_exchange_pack / _unpack / _enqueue)."""
        from .engine import ExchangePlanHandle
        self.xplan = ExchangePlanHandle(self.eng, xp.counts, xp.ids, xp.world, rank)
        return self.xplan

    def close(self):
        if self.xplan is not None:
            self.xplan.close()
        self.handle.close()
        self.eng.wires_alloc(0)


_NCCL_COMMS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()  # engine -> (group, world)


def _native_comm(eng, group, world: int, rank: int) -> bool:
    """Give the engine its own NCCL communicator over `group` (once per engine
    and group): rank 0's ncclUniqueId travels over the process group."""
    import torch.distributed as dist
    from .engine import nccl_available, nccl_unique_id
    key = (id(group) if group is not None else None, world)
    if _NCCL_COMMS.get(eng) == key:
        return True
    if not nccl_available()[0]:
        return False
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    eng.nccl_init(world, rank, obj[0])
    _NCCL_COMMS[eng] = key
    return True


def _p2p_host(send_rows: dict, recv_shapes: dict, group):
    """Grouped point-to-point through torch.distributed (gloo, CPU tensors):
    the host-staged transport for CPU tests and for ranks sharing one GPU."""
    import torch
    import torch.distributed as dist
    ops, recv = [], {}
    for q, t in send_rows.items():
        ops.append(dist.P2POp(dist.isend, t.contiguous(), dist.get_global_rank(group, q) if group is not None else q,
                              group=group))
    for q, shape in recv_shapes.items():
        recv[q] = torch.empty(shape, dtype=torch.int32)
        ops.append(dist.P2POp(dist.irecv, recv[q], dist.get_global_rank(group, q) if group is not None else q,
                              group=group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()
    return recv


def evaluate_distributed(c: Circuit, schedule: Schedule, mats: dict, ek: EvalKey, *, group=None,
                         levels_factory=None):
    """Rank-local part of `runtime.evaluate` for world > 1.

    levels_factory(plan, slots, device) -> object with `.wires` (torch int32
    (slots, stride) tensor), `.run_level(level)` and `.close()`; defaults to
    the CUDA engine.  Tests substitute a plaintext mock to check the
    partition/exchange logic on CPU with gloo.

    Transport: with the NCCL backend and the engine on the GPU, the engine's
    own NCCL communicator moves the rows (gw_exchange_enqueue: pack -> grouped
    ncclSend/ncclRecv -> unpack, stream-ordered, no host sync between levels).
    Otherwise (gloo) the packed rows are staged through host memory.
    """
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    p = ek.params
    from .runtime import _cached_plan
    plan = _cached_plan(c, schedule, worker=rank, world=world)
    xp = exchange_plan(c, schedule, world)
    slots = c.max_wire + 1
    # the engine lives on the same GPU as the wire tensor, and the context is
    # single-submitter: it is held for the whole evaluation (as runtime.evaluate does)
    lock = contextlib.nullcontext()
    if levels_factory is None:
        device = torch.device("cuda", torch.cuda.current_device())
        eng = ek.engine(device=device.index)
        lock = eng._mtx
        lock.__enter__()
        try:
            lv = _DeviceLevels(eng, plan, slots, device)
        except BaseException:
            lock.__exit__(None, None, None)
            raise
    else:
        device = torch.device("cpu")
        lv = levels_factory(plan, slots, device)
    wires = lv.wires
    W = p.n + 1
    levels = len(schedule.waves)
    stride = wires.shape[1]
    dx, native = None, False
    try:
        dx = lv.exchange_plan(xp, rank) if hasattr(lv, "exchange_plan") else None
        if dx is not None and dist.get_backend(group) == "nccl":
            native = _native_comm(lv.eng, group, world, rank)
        for port in c.inputs:
            ids = torch.as_tensor(np.asarray(port.wires, np.int64), device=device)
            wires[ids, :W] = torch.from_numpy(mats[port.name].view(np.int32)).to(device)
        if native:
            lv.eng.timeline_reset()
        dist.barrier(group=group)
        if native:
            lv.eng.timeline_mark()
        per_wave = []
        t0 = time.monotonic()
        for L in range(levels):
            s = time.monotonic()
            lv.run_level(L)
            moves = xp.counts[L].sum() > 0
            if native:
                if moves:
                    dx.enqueue(L)
                lv.eng.timeline_mark()
                continue
            if moves and dx is not None:      # engine pack / unpack, rows staged through the host
                sr, rr = dx.peer_rows(L)
                tot_s, tot_r = int(sr.sum()), int(rr.sum())
                sendbuf = torch.empty((max(tot_s, 1), stride), dtype=torch.int32, device=device)
                if tot_s:
                    dx.pack(L, sendbuf.data_ptr())      # rows grouped by destination rank
                torch.cuda.current_stream(device).synchronize()
                host = sendbuf[:tot_s].cpu()
                send, o = {}, 0
                for q in range(world):
                    if sr[q]:
                        send[q] = host[o:o + sr[q]]
                        o += int(sr[q])
                recv = _p2p_host(send, {q: (int(rr[q]), stride) for q in range(world) if rr[q]}, group)
                if tot_r:                              # rows grouped by source rank
                    rbuf = torch.cat([recv[q] for q in range(world) if rr[q]]).to(device).contiguous()
                    dx.unpack(L, rbuf.data_ptr())
                    torch.cuda.current_stream(device).synchronize()
            elif moves:                          # plaintext mock levels (CPU tests)
                send = {q: wires[torch.as_tensor(xp.cell(L, rank, q))] for q in range(world)
                        if q != rank and xp.counts[L, rank, q]}
                recv = _p2p_host(send, {q: (int(xp.counts[L, q, rank]), stride) for q in range(world)
                                        if q != rank and xp.counts[L, q, rank]}, group)
                for q, rows in recv.items():
                    wires[torch.as_tensor(xp.cell(L, q, rank))] = rows
            if device.type == "cuda":
                torch.cuda.current_stream(device).synchronize()
            per_wave.append(time.monotonic() - s)
        if native:
            per_wave = [ms / 1e3 for ms in lv.eng.timeline_read()]   # one sync, after the last level
            lv.eng.timeline_reset()
        t1 = time.monotonic()
        outputs = {}
        for port in c.outputs:
            ids = torch.as_tensor(np.asarray(port.wires, np.int64), device=device)
            outputs[port.name] = wires[ids, :W].cpu().numpy().view(np.uint32).copy()
    finally:
        try:
            lv.close()
        finally:
            lock.__exit__(None, None, None)
    # whole-job metrics: wall time is the max over ranks
    cdev = device if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = torch.tensor([t1 - t0] + per_wave, dtype=torch.float64, device=cdev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    boots = torch.tensor([plan.bootstraps], dtype=torch.int64, device=cdev)
    dist.all_reduce(boots, group=group)
    total_boot = int(boots.item())
    m = Metrics(total_gates=len(c.gates), workers=schedule.workers, gpus=world)
    m.wall_time_seconds = float(t[0])
    m.per_wave_wall_time = [float(x) for x in t[1:]]
    m.device_time_seconds = float(sum(m.per_wave_wall_time))
    m.bootstrap_count = total_boot
    m.ntt_forward_count = 2 * p.l * p.n * total_boot
    m.ntt_inverse_count = 2 * p.n * total_boot
    m.gates_per_second = len(c.gates) / m.wall_time_seconds if m.wall_time_seconds > 0 else 0.0
    m.per_worker_busy_time = [m.wall_time_seconds] * schedule.workers
    m.exchange_bytes = int(sum(xp.bytes_per_level(W * 4)))
    m.transport = "nccl" if native else ("host-staged" if dx is not None else "mock")
    return outputs, m


def check_world(schedule: Schedule, world: int):
    if world < 1:
        raise EvaluateError("world size must be >= 1")
