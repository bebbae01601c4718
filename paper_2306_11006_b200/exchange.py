"""Multi-GPU netlist evaluation: per-rank level slices + cross-GPU wire exchange.

One process per GPU (torch.distributed; NCCL over NVLink on B200, gloo on CPU
for tests).  The reference's partitioner assigns slice k of every opcode
group of every level to worker k (scheduler.py:133-157); here worker k runs on
rank k mod world.  Keys are replicated.  After each level a static plan moves
only the produced wires that some OTHER rank reads in a later level, or that
are circuit outputs (every rank returns the full outputs): one padded
all-gather per level over the ranks' send lists (~2.5 KB per
wire), scattered into each rank's device wire store.  Levels stay
stream-ordered: run level -> pack -> all_gather -> unpack -> next level.
"""
from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .cggi import EvalKey
from .circuit import Circuit
from .runtime import EvaluateError, Metrics
from .scheduler import Schedule


@dataclass
class ExchangePlan:
    world: int
    sends: list            # [level][rank] -> int64 array of wire ids that rank broadcasts
    pad: list              # [level] -> max send count (all_gather row count per rank)

    def bytes_per_level(self, row_bytes: int) -> list[int]:
        return [self.world * m * row_bytes for m in self.pad]


def owners(c: Circuit, schedule: Schedule, world: int) -> dict[int, int]:
    own = {}
    for wave in schedule.waves:
        for b in wave:
            for gid in b.gate_ids:
                own[gid] = b.worker % world
    return own


def exchange_plan(c: Circuit, schedule: Schedule, world: int) -> ExchangePlan:
    """Per level and rank, the produced wires that another rank reads later or
    that are circuit outputs.  Vectorised over the circuit arrays (numpy)."""
    from .runtime import _circuit_arrays
    ids, _, opnd, _ = _circuit_arrays(c)
    nb = [(wi, b) for wi, wave in enumerate(schedule.waves) for b in wave]
    sizes = np.fromiter((len(b.gate_ids) for _, b in nb), dtype=np.int64, count=len(nb))
    total = int(sizes.sum())
    gid = np.fromiter((g for _, b in nb for g in b.gate_ids), dtype=np.int64, count=total)
    wave = np.repeat(np.fromiter((wi for wi, _ in nb), dtype=np.int64, count=len(nb)), sizes)
    rank = np.repeat(np.fromiter((b.worker % world for _, b in nb), dtype=np.int64, count=len(nb)), sizes)
    top = int(max(c.max_wire, ids.max() if len(ids) else 0)) + 1
    own = np.full(top, -1, dtype=np.int64)
    own[gid] = rank
    send = np.zeros(top, dtype=bool)
    # reader rank of every operand slot (circuit order) vs the writer's rank
    reader = own[ids]
    valid = opnd >= 0
    w = np.where(valid, opnd, 0)
    cross = valid & (own[w] >= 0) & (own[w] != reader[:, None])
    send[w[cross]] = True
    for p in c.outputs:
        send[np.asarray(p.wires, np.int64)] = True
    keep = send[gid]
    sends, pad = [], []
    levels = len(schedule.waves)
    order = np.lexsort((rank[keep], wave[keep]))
    kg, kw, kr = gid[keep][order], wave[keep][order], rank[keep][order]
    # split into [level][rank] (schedule order inside each bucket)
    key = kw * world + kr
    bounds = np.searchsorted(key, np.arange(levels * world + 1))
    for L in range(levels):
        per_rank = [kg[bounds[L * world + r]:bounds[L * world + r + 1]] for r in range(world)]
        sends.append(per_rank)
        pad.append(max((len(x) for x in per_rank), default=0))
    return ExchangePlan(world=world, sends=sends, pad=pad)


class _DeviceLevels:
    """Adapter: the CUDA engine running one rank's level plan on a torch wire store."""

    def __init__(self, ek: EvalKey, plan, slots: int, device):
        import torch
        self.eng = ek.engine()
        self.stream = torch.cuda.current_stream(device)
        if self.stream.cuda_stream == 0:
            self.stream = torch.cuda.Stream(device)
            torch.cuda.set_stream(self.stream)
        self.eng.set_stream(self.stream.cuda_stream)
        self.wires = torch.zeros((slots, self.eng.row_stride), dtype=torch.int32, device=device)
        self.eng.wires_attach(self.wires.data_ptr(), slots, self.eng.row_stride)
        self.handle = self.eng.plan_create(plan.level_offsets, plan.opcodes, plan.operands,
                                           plan.out_ids)

    def run_level(self, level: int):
        self.handle.run(level, level + 1)

    def exchange_plan(self, sends, world: int):
        """Device exchange plan: the level's send rows are packed / unpacked by
        engine kernels on the engine stream (gw_exchange_pack / _unpack)."""
        from .engine import ExchangePlanHandle
        self.xplan = ExchangePlanHandle(self.eng, sends, world)
        return self.xplan

    def close(self):
        if getattr(self, "xplan", None) is not None:
            self.xplan.close()
        self.handle.close()
        self.eng.wires_alloc(0)


def _all_gather(send, world: int, group):
    """all_gather of equal-size row blocks.  NCCL takes device tensors
    directly (NVLink); a CPU backend (gloo, used by the one-GPU two-rank test)
    gets a host-staged copy."""
    import torch
    import torch.distributed as dist
    backend = dist.get_backend(group)
    if send.is_cuda and backend != "nccl":
        host = send.cpu()
        out = torch.empty((world * host.shape[0], host.shape[1]), dtype=host.dtype)
        dist.all_gather_into_tensor(out, host, group=group)
        return out.to(send.device)
    out = torch.empty((world * send.shape[0], send.shape[1]), dtype=send.dtype, device=send.device)
    dist.all_gather_into_tensor(out, send, group=group)
    return out


def evaluate_distributed(c: Circuit, schedule: Schedule, mats: dict, ek: EvalKey, *, group=None,
                         levels_factory=None):
    """Rank-local part of `runtime.evaluate` for world > 1.

    levels_factory(plan, slots, device) -> object with `.wires` (torch int32
    (slots, stride) tensor), `.run_level(level)` and `.close()`; defaults to
    the CUDA engine.  Tests substitute a plaintext mock to check the
    partition/exchange logic on CPU with gloo.
    """
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    p = ek.params
    from .runtime import _cached_plan
    plan = _cached_plan(c, schedule, worker=rank, world=world)
    xplan = exchange_plan(c, schedule, world)
    slots = c.max_wire + 1
    if levels_factory is None:
        device = torch.device("cuda", torch.cuda.current_device())
        lv = _DeviceLevels(ek, plan, slots, device)
    else:
        device = torch.device("cpu")
        lv = levels_factory(plan, slots, device)
    wires = lv.wires
    W = p.n + 1
    dx = lv.exchange_plan(xplan.sends, world) if hasattr(lv, "exchange_plan") else None
    try:
        for port in c.inputs:
            ids = torch.as_tensor(np.asarray(port.wires, np.int64), device=device)
            wires[ids, :W] = torch.from_numpy(mats[port.name].view(np.int32)).to(device)
        per_wave = []
        t0 = time.monotonic()
        for L in range(len(schedule.waves)):
            s = time.monotonic()
            lv.run_level(L)
            m = xplan.pad[L]
            if m and dx is not None:   # engine kernels pack / unpack on the engine stream
                send = torch.empty((m, wires.shape[1]), dtype=torch.int32, device=device)
                dx.pack(L, rank, send.data_ptr())
                recv = _all_gather(send, world, group)
                dx.unpack(L, rank, recv.data_ptr())
            elif m:                    # plaintext mock levels (CPU tests)
                mine = xplan.sends[L][rank]
                send = torch.zeros((m, wires.shape[1]), dtype=torch.int32, device=device)
                if len(mine):
                    send[:len(mine)] = wires[torch.as_tensor(mine, device=device)]
                recv = _all_gather(send, world, group)
                for q in range(world):
                    ids = xplan.sends[L][q]
                    if q == rank or not len(ids):
                        continue
                    wires[torch.as_tensor(ids, device=device)] = recv[q * m:q * m + len(ids)]
            if device.type == "cuda":
                torch.cuda.current_stream(device).synchronize()
            per_wave.append(time.monotonic() - s)
        t1 = time.monotonic()
        outputs = {}
        for port in c.outputs:
            ids = torch.as_tensor(np.asarray(port.wires, np.int64), device=device)
            outputs[port.name] = wires[ids, :W].cpu().numpy().view(np.uint32).copy()
    finally:
        lv.close()
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
    m.device_time_seconds = m.wall_time_seconds
    m.bootstrap_count = total_boot
    m.ntt_forward_count = 2 * p.l * p.n * total_boot
    m.ntt_inverse_count = 2 * p.n * total_boot
    m.gates_per_second = len(c.gates) / m.wall_time_seconds if m.wall_time_seconds > 0 else 0.0
    m.per_worker_busy_time = [m.wall_time_seconds] * schedule.workers
    return outputs, m


def check_world(schedule: Schedule, world: int):
    if world < 1:
        raise EvaluateError("world size must be >= 1")
