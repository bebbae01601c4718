"""Two ranks on one B200 (gloo process group, host-staged exchange): the real
CUDA engine runs each rank's level slices and the cross-rank wire exchange
must reproduce the single-process ciphertexts bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import MINI

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200 import netlists as NL
    from paper_2306_11006_b200.cggi import encrypt_bits, keygen
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import evaluate
    from paper_2306_11006_b200.scheduler import build_schedule
    ks = keygen(MINI, 2024)
    res = []
    for c in (C.gen_adder(4), NL.gen_multiplier(4), C.gen_mux_tree(2)):
        rng = np.random.default_rng(3)
        srng = SeededRng(11)
        inputs = {p.name: encrypt_bits(MINI, ks.lwe_sk, rng.integers(0, 2, p.width), srng) for p in c.inputs}
        outs, met = evaluate(c, build_schedule(c, world), inputs, ks)
        res.append({k: v.tobytes() for k, v in outs.items()})
    q.put((rank, res))
    dist.destroy_process_group()


def _single():
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200 import netlists as NL
    from paper_2306_11006_b200.cggi import encrypt_bits, keygen
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import evaluate
    from paper_2306_11006_b200.scheduler import build_schedule
    ks = keygen(MINI, 2024)
    res = []
    for c in (C.gen_adder(4), NL.gen_multiplier(4), C.gen_mux_tree(2)):
        rng = np.random.default_rng(3)
        srng = SeededRng(11)
        inputs = {p.name: encrypt_bits(MINI, ks.lwe_sk, rng.integers(0, 2, p.width), srng) for p in c.inputs}
        outs, _ = evaluate(c, build_schedule(c, 1), inputs, ks)
        res.append({k: v.tobytes() for k, v in outs.items()})
    return res


def test_two_ranks_one_gpu_match_single_process():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    try:
        got = dict(q.get(timeout=300) for _ in procs)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():  # never leave a rank behind to disturb later runs on this box
                p.kill()
                p.join()
    want = _single()
    assert got[0] == want and got[1] == want


def _nccl_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200 import netlists as NL
    from paper_2306_11006_b200.cggi import encrypt_bits, keygen
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import evaluate
    from paper_2306_11006_b200.scheduler import build_schedule
    ks = keygen(MINI, 2024)
    res, transports = [], []
    for c in (C.gen_adder(4), NL.gen_multiplier(4), C.gen_mux_tree(2)):
        rng = np.random.default_rng(3)
        srng = SeededRng(11)
        inputs = {p.name: encrypt_bits(MINI, ks.lwe_sk, rng.integers(0, 2, p.width), srng) for p in c.inputs}
        outs, met = evaluate(c, build_schedule(c, world), inputs, ks)
        res.append({k: v.tobytes() for k, v in outs.items()})
        transports.append(met.transport)
    q.put((rank, res, transports))
    dist.destroy_process_group()


def test_two_gpus_native_nccl_exchange_matches_single_process():
    """NCCL over NVLink between two GPUs: the engine's own communicator moves
    the rows (gw_exchange_enqueue, grouped ncclSend / ncclRecv).  NCCL cannot
    put two ranks on one GPU, so this needs two visible GPUs."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip(f"needs 2 GPUs for a 2-rank NCCL communicator, {torch.cuda.device_count()} visible")
    from paper_2306_11006_b200.engine import nccl_available
    ver, why = nccl_available()
    assert ver > 0, why
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in procs:
            rank, res, tr = q.get(timeout=300)
            got[rank] = res
            assert tr == ["nccl"] * 3
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():  # never leave a rank behind to disturb later runs on this box
                p.kill()
                p.join()
    want = _single()
    assert got[0] == want and got[1] == want


def test_nccl_library_binds():
    """The engine binds libnccl at run time (no link-time dependency)."""
    from paper_2306_11006_b200.engine import nccl_available, nccl_unique_id
    ver, why = nccl_available()
    assert ver >= 22700, why
    assert len(nccl_unique_id()) == 128


def test_nccl_communicator_on_this_gpu():
    """gw_nccl_init builds a real NCCL communicator on the device through the
    run-time-bound library (world 1: the most one GPU allows), and a world-1
    exchange plan enqueues as a no-op on it."""
    import numpy as np
    from paper_2306_11006_b200 import engine
    from paper_2306_11006_b200.cggi import PARAM_128
    ver, why = engine.nccl_available()
    assert ver >= 22700, why
    eng = engine.Engine(*engine.params_tuple(PARAM_128))
    eng.nccl_init(1, 0, engine.nccl_unique_id())
    xp = engine.ExchangePlanHandle(eng, np.zeros((2, 1, 1), np.int64), np.zeros(0, np.int64), 1, 0)
    try:
        xp.enqueue(0)
        xp.enqueue(1)
    finally:
        xp.close()
    eng.close()
