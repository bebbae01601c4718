"""Netlist evaluation on the GPU (seam 3): device wire store + level plans.
Ciphertext outputs must equal the reference runtime's (golden adder4) and the
oracle evaluated gate batch by gate batch; decrypted outputs equal
simulate_plain; results are identical for every worker count."""
import numpy as np
import pytest

from conftest import MINI

pytestmark = pytest.mark.gpu


def _oracle_evaluate(c, sched, inputs, okeys, n):
    """Reference semantics (runtime.py:122-222) with the oracle's gate batches."""
    import oracle as O
    rows = {}
    for p in c.inputs:
        for k, w in enumerate(p.wires):
            rows[w] = inputs[p.name][k]
    by_id = {g.id: g for g in c.gates}
    for wave in sched.waves:
        for b in wave:
            gates = [by_id[gid] for gid in b.gate_ids]
            ar = len(gates[0].operands)
            ops = [np.stack([rows[g.operands[k]] for g in gates]) for k in range(ar)]
            out = O.eval_gate_batch(b.opcode.value, ops, okeys, count=len(gates))
            for g, r in zip(gates, out):
                rows[g.id] = r
    return {p.name: np.stack([rows[w] for w in p.wires]) for p in c.outputs}


def test_adder4_matches_reference_runtime_mini(golden_mini, golden_json):
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200.cggi import EvalKey
    from paper_2306_11006_b200.runtime import evaluate
    from paper_2306_11006_b200.scheduler import build_schedule
    ek = EvalKey.build(MINI, golden_mini["bk_data"], golden_mini["ksk_data"])
    c = C.gen_adder(4)
    outs, met = evaluate(c, build_schedule(c, 2), {"a": golden_mini["adder_a"],
                                                   "b": golden_mini["adder_b"]}, ek)
    assert np.array_equal(outs["s"], golden_mini["adder_s"])
    g = golden_json["mini_adder4"]
    assert (met.bootstrap_count, met.ntt_forward_count, met.ntt_inverse_count,
            met.total_gates) == (g["bootstraps"], g["fwd"], g["inv"], g["total_gates"])
    assert len(met.per_wave_wall_time) == len(g["waves"])


@pytest.mark.parametrize("name", ["adder8", "mux3", "flat40_xor", "not_chain"])
def test_netlists_match_oracle_and_plaintext_p128(p128_keys, name):
    import oracle as O
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200.cggi import PARAM_128, GateKind, decrypt_rows, encrypt_bits
    from paper_2306_11006_b200.rng import SeededRng
    from paper_2306_11006_b200.runtime import evaluate
    from paper_2306_11006_b200.scheduler import build_schedule
    c = {"adder8": lambda: C.gen_adder(8), "mux3": lambda: C.gen_mux_tree(3),
         "flat40_xor": lambda: C.gen_flat(40, GateKind.XOR),
         "not_chain": lambda: C.gen_not_chain(6)}[name]()
    rng = np.random.default_rng(80)
    vals = {p.name: int(rng.integers(0, 1 << p.width)) for p in c.inputs}
    srng = SeededRng(8000)
    inputs = {p.name: encrypt_bits(PARAM_128, p128_keys.lwe_sk, C.value_to_bits(vals[p.name], p.width), srng)
              for p in c.inputs}
    ek = p128_keys.eval_key()
    outs = {}
    for K in (1, 2, 4):
        o, met = evaluate(c, build_schedule(c, K), inputs, ek)
        outs[K] = o
    for K in (2, 4):
        for k in outs[1]:
            assert np.array_equal(outs[1][k], outs[K][k])
    okeys = O.Keys.from_params(PARAM_128, p128_keys.bootstrapping_key.data,
                               p128_keys.keyswitch_key.data)
    want = _oracle_evaluate(c, build_schedule(c, 1), inputs, okeys, PARAM_128.n)
    plain = C.simulate_plain(c, vals)
    for k, rows in outs[1].items():
        assert np.array_equal(rows, want[k])
        assert C.bits_to_value(decrypt_rows(p128_keys.lwe_sk, rows)) == plain[k]


def test_evaluate_errors(mini_keys):
    from paper_2306_11006_b200 import circuit as C
    from paper_2306_11006_b200.cggi import DimensionError
    from paper_2306_11006_b200.runtime import EvaluateError, evaluate
    from paper_2306_11006_b200.scheduler import build_schedule
    c = C.gen_adder(2)
    s = build_schedule(c, 1)
    good = np.zeros((2, MINI.n + 1), np.uint32)
    with pytest.raises(EvaluateError):
        evaluate(c, s, {"a": good}, mini_keys)
    with pytest.raises(EvaluateError):
        evaluate(c, s, {"a": good, "b": good, "zz": good}, mini_keys)
    with pytest.raises(EvaluateError):
        evaluate(c, s, {"a": good, "b": np.zeros((3, MINI.n + 1), np.uint32)}, mini_keys)
    with pytest.raises(DimensionError):
        evaluate(c, s, {"a": good, "b": np.zeros((2, MINI.n), np.uint32)}, mini_keys)
    with pytest.raises(EvaluateError):
        evaluate(c, build_schedule(C.gen_adder(3), 1), {"a": good, "b": good}, mini_keys)


def test_exchange_pack_unpack_kernels(p128_keys):
    """gw_exchange_pack / _unpack move exactly the planned wire rows, grouped by
    destination (pack) and by source (unpack)."""
    import torch
    from paper_2306_11006_b200.cggi import PARAM_128
    from paper_2306_11006_b200.engine import Engine, ExchangePlanHandle, params_tuple
    eng = Engine(*params_tuple(PARAM_128), device=0)
    slots, W = 64, PARAM_128.n + 1
    eng.wires_alloc(slots)
    rows = np.random.default_rng(5).integers(0, 2 ** 32, (slots, W), dtype=np.uint32)
    eng.wires_put(np.arange(slots), rows)
    # 3 ranks, 2 levels; this is rank 0.  counts[L][src][dst]
    counts = np.zeros((2, 3, 3), np.int64)
    cells = {(0, 0, 1): [3, 7], (0, 0, 2): [9], (0, 1, 0): [20, 21], (0, 2, 0): [30],
             (0, 1, 2): [22], (1, 2, 0): [40]}
    ids = []
    for L in range(2):
        for q in range(3):
            for r in range(3):
                cell = cells.get((L, q, r), [])
                counts[L, q, r] = len(cell)
                ids += cell
    x = ExchangePlanHandle(eng, counts, np.array(ids, np.int64), 3, 0)
    sr, rr = x.peer_rows(0)
    assert sr.tolist() == [0, 2, 1] and rr.tolist() == [0, 2, 1]
    stride = eng.row_stride
    send = torch.zeros((3, stride), dtype=torch.int32, device="cuda")
    x.pack(0, send.data_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(send[:, :W].cpu().numpy().view(np.uint32), rows[[3, 7, 9]])
    recv = torch.zeros((3, stride), dtype=torch.int32, device="cuda")
    new = np.random.default_rng(6).integers(0, 2 ** 32, (3, W), dtype=np.uint32)
    recv[:, :W] = torch.from_numpy(new.view(np.int32)).cuda()
    x.unpack(0, recv.data_ptr())        # rank 1's wires 20, 21 then rank 2's wire 30
    torch.cuda.synchronize()
    got = eng.wires_get(np.arange(slots))
    want = rows.copy()
    want[[20, 21, 30]] = new
    assert np.array_equal(got, want)
    # plan-owned staging buffers
    ds, dr = x.buffers()
    assert ds and dr
    x.close()


def test_concurrent_gate_batches_from_pool_threads(p128_keys):
    """The reference runtime submits eval_gate_batch from K pool threads at once
    (runtime.py:184); with the drop-in patched in, every thread shares one cached
    engine.  Results must equal the sequential ones bit for bit."""
    from concurrent.futures import ThreadPoolExecutor
    from paper_2306_11006_b200.cggi import GATE_ARITY, PARAM_128, GateKind, encrypt_bits, eval_gate_batch
    from paper_2306_11006_b200.rng import SeededRng
    ks = p128_keys
    ek = ks.eval_key()
    rng = np.random.default_rng(17)
    kinds = [GateKind.NAND, GateKind.XOR, GateKind.AND, GateKind.MUX, GateKind.OR, GateKind.NOT,
             GateKind.XNOR, GateKind.NOR]
    jobs = []
    for j, kind in enumerate(kinds):
        ar = GATE_ARITY[kind]
        B = 24 + 8 * j
        ops = [encrypt_bits(PARAM_128, ks.lwe_sk, rng.integers(0, 2, B).astype(np.uint8), SeededRng(100 * j + k))
               for k in range(ar)]
        jobs.append((kind, ops))
    want = [eval_gate_batch(kind, ops, ek) for kind, ops in jobs]
    with ThreadPoolExecutor(max_workers=8) as pool:
        for _ in range(2):
            got = list(pool.map(lambda job: eval_gate_batch(job[0], job[1], ek), jobs))
            for g, w in zip(got, want):
                assert np.array_equal(g, w)


def test_eval_key_file_feeds_the_device(p128_keys, tmp_path):
    """An ARFX evaluation key (reference format) loads straight onto the GPU and
    gives the same gate outputs as the in-memory keys."""
    from paper_2306_11006_b200 import serial as S
    from paper_2306_11006_b200.cggi import PARAM_128, GateKind, encrypt_bits, eval_gate_batch
    from paper_2306_11006_b200.rng import SeededRng
    path = str(tmp_path / "p128.ek")
    S.write_eval_key(path, p128_keys)
    ek = S.read_eval_key(path, upload=True)
    rng = np.random.default_rng(5)
    a = encrypt_bits(PARAM_128, p128_keys.lwe_sk, rng.integers(0, 2, 40).astype(np.uint8), SeededRng(1))
    b = encrypt_bits(PARAM_128, p128_keys.lwe_sk, rng.integers(0, 2, 40).astype(np.uint8), SeededRng(2))
    assert np.array_equal(eval_gate_batch(GateKind.XOR, [a, b], ek),
                          eval_gate_batch(GateKind.XOR, [a, b], p128_keys.eval_key()))


def test_wires_attach_rejects_non_device_memory():
    """gw_wires_attach takes only device memory on the context's own GPU: a host
    (pinned) pointer is rejected before any kernel could dereference it; a
    device tensor is accepted and evaluated into (foreign pointers)."""
    import torch
    from paper_2306_11006_b200.cggi import PARAM_128
    from paper_2306_11006_b200.engine import Engine, params_tuple
    eng = Engine(*params_tuple(PARAM_128), device=0)
    stride = eng.row_stride
    host = torch.zeros((8, stride), dtype=torch.int32, pin_memory=True)
    with pytest.raises(ValueError, match="device memory"):
        eng.wires_attach(host.data_ptr(), 8, stride)
    plain = np.zeros((8, stride), np.int32)
    with pytest.raises(ValueError):
        eng.wires_attach(plain.ctypes.data, 8, stride)
    dev = torch.zeros((8, stride), dtype=torch.int32, device="cuda:0")
    eng.wires_attach(dev.data_ptr(), 8, stride)
    rows = np.random.default_rng(2).integers(0, 2 ** 32, (3, PARAM_128.n + 1), dtype=np.uint32)
    eng.wires_put(np.array([1, 4, 6]), rows)
    assert np.array_equal(eng.wires_get(np.array([1, 4, 6])), rows)
    eng.wires_attach(None, 0, stride)
    eng.close()
