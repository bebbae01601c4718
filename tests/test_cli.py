"""The drop-in command line (paper_2306_11006_b200/cli.py; reference cli.py:
199-241 cmd_run, :314-387 main): arguments, printed fields, exit codes
(0 ok, 1 usage, 2 circuit, 3 crypto/params, 4 I/O), ARFX files, and the
GPU `run` (marked gpu).  The reference's own tests/test_cli.py also runs
against this CLI through tools/ref_suite (GW_SEAM=3)."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, MINI
from paper_2306_11006_b200.cli import main

MINI_JSON = dict(n=MINI.n, N=MINI.N, lwe_noise_std=MINI.lwe_noise_std, rlwe_noise_std=MINI.rlwe_noise_std,
                 Bg_bits=MINI.Bg_bits, l=MINI.l, ks_base_bits=MINI.ks_base_bits, ks_levels=MINI.ks_levels)


@pytest.fixture()
def wd(tmp_path):
    (tmp_path / "mini.json").write_text(json.dumps(MINI_JSON))
    return tmp_path


def _keys(d, seed="00ff"):
    assert main(["keygen", "--params", str(d / "mini.json"), "--seed", seed,
                 "--out-secret", str(d / "sk.bin"), "--out-eval", str(d / "ek.bin")]) == 0


def _adder(d, width=4):
    assert main(["gen", "--fixture", "adder", "--width", str(width), "--out", str(d / "adder.cir")]) == 0


def _encrypt(d, a=9, b=8, seed="01"):
    assert main(["encrypt", "--secret", str(d / "sk.bin"), "--circuit", str(d / "adder.cir"),
                 "--assign", f"a={a}", "--assign", f"b={b}", "--seed", seed, "--out", str(d / "in.bin")]) == 0


def test_keygen_prints_parameters_and_writes_reference_files(wd, capsys):
    _keys(wd)
    out = capsys.readouterr().out
    assert f"n = {MINI.n}" in out and f"N = {MINI.N}" in out
    # MINI, keygen seed 2024 (int) vs hex seeds: the files for the int seed are the
    # reference's own (tests/golden/arfx); here only the sizes are fixed by the format
    assert f"secret_key_bytes = {os.path.getsize(os.path.join(GOLDEN, 'arfx', 'mini.sk'))}" in out
    assert f"eval_key_bytes = {os.path.getsize(os.path.join(GOLDEN, 'arfx', 'mini.ek'))}" in out


def test_same_seed_same_key_bytes(wd, tmp_path_factory):
    _keys(wd)
    other = tmp_path_factory.mktemp("o")
    (other / "mini.json").write_text(json.dumps(MINI_JSON))
    _keys(other)
    assert (wd / "sk.bin").read_bytes() == (other / "sk.bin").read_bytes()
    assert (wd / "ek.bin").read_bytes() == (other / "ek.bin").read_bytes()


def test_unknown_param_set_is_usage_error(tmp_path, capsys):
    assert main(["keygen", "--params", "nope", "--out-secret", str(tmp_path / "a"),
                 "--out-eval", str(tmp_path / "b")]) == 1
    err = capsys.readouterr().err
    assert "110" in err and "128" in err


def test_analyze_and_gen(wd, capsys):
    _adder(wd, 8)
    assert main(["analyze", "--circuit", str(wd / "adder.cir"), "--workers", "2",
                 "--csv", str(wd / "lv.csv"), "--schedule-csv", str(wd / "s.csv")]) == 0
    out = capsys.readouterr().out
    assert "total_gates = 40" in out and "levels = 15" in out and "XOR = 16" in out
    assert "workers = 2" in out and "cost_units = 39937" in out     # 39 bootstraps x 1024 + CONST0 (1)
    assert (wd / "lv.csv").read_text().splitlines()[0] == "level,width"
    assert len((wd / "lv.csv").read_text().splitlines()) == 16
    assert (wd / "s.csv").read_text().splitlines()[0] == "wave,opcode,worker,count,cost_units"
    for args, gates in ((["--fixture", "mux-tree", "--depth", "2"], 3),
                        (["--fixture", "not-chain", "--length", "7"], 7),
                        (["--fixture", "flat", "--gates", "12", "--op", "XNOR"], 12)):
        assert main(["gen", *args, "--out", str(wd / "f.cir")]) == 0
        from paper_2306_11006_b200.circuit import parse_circuit
        assert len(parse_circuit((wd / "f.cir").read_text()).gates) == gates


def test_workers_from_environment(wd, capsys, monkeypatch):
    _adder(wd)
    monkeypatch.setenv("ARCTYREX_THREADS", "3")
    assert main(["analyze", "--circuit", str(wd / "adder.cir")]) == 0
    assert "workers = 3" in capsys.readouterr().out
    monkeypatch.setenv("ARCTYREX_THREADS", "zebra")
    assert main(["analyze", "--circuit", str(wd / "adder.cir")]) == 1


def test_exit_codes(wd, capsys):
    _keys(wd)
    _adder(wd)
    # 1: usage
    assert main(["gen", "--fixture", "flat", "--op", "WIBBLE", "--out", str(wd / "x.cir")]) == 1
    assert main(["encrypt", "--secret", str(wd / "sk.bin"), "--circuit", str(wd / "adder.cir"),
                 "--assign", "a=1", "--out", str(wd / "in.bin")]) == 1          # missing b
    assert main(["encrypt", "--secret", str(wd / "sk.bin"), "--circuit", str(wd / "adder.cir"),
                 "--assign", "a=1", "--assign", "b=99", "--out", str(wd / "in.bin")]) == 1  # does not fit
    # 2: circuit parse error
    (wd / "bad.cir").write_text("this is not a circuit\n")
    assert main(["analyze", "--circuit", str(wd / "bad.cir")]) == 2
    # 3: bad parameters
    (wd / "bad.json").write_text(json.dumps({**MINI_JSON, "N": 63}))
    assert main(["keygen", "--params", str(wd / "bad.json"), "--out-secret", str(wd / "s2"),
                 "--out-eval", str(wd / "e2")]) == 3
    # 4: I/O and format
    assert main(["decrypt", "--secret", str(wd / "missing.bin"), "--circuit", str(wd / "adder.cir"),
                 "--in", str(wd / "in.bin")]) == 4
    (wd / "junk.bin").write_bytes(b"JUNKJUNKJUNK")
    assert main(["decrypt", "--secret", str(wd / "junk.bin"), "--circuit", str(wd / "adder.cir"),
                 "--in", str(wd / "in.bin")]) == 4
    capsys.readouterr()


def test_run_reports_failing_stage(wd, capsys):
    _adder(wd)
    rc = main(["run", "--eval", str(wd / "nope.bin"), "--circuit", str(wd / "adder.cir"),
               "--in", str(wd / "in.bin"), "--out", str(wd / "out.bin")])
    assert rc == 4 and "[keys]" in capsys.readouterr().err


@pytest.mark.gpu
def test_full_pipeline_on_gpu(wd, capsys):
    """keygen -> encrypt -> run (B200) -> decrypt: adder4 9 + 8 = 17, 20 gates,
    19 bootstraps, metrics JSON in the reference's shape (runtime.py:62-73)."""
    _keys(wd)
    _adder(wd)
    _encrypt(wd)
    assert main(["run", "--eval", str(wd / "ek.bin"), "--circuit", str(wd / "adder.cir"),
                 "--in", str(wd / "in.bin"), "--out", str(wd / "out.bin"),
                 "--metrics", str(wd / "m.json")]) == 0
    out = capsys.readouterr().out
    assert "gates = 20" in out and "bootstraps = 19" in out
    m = json.loads((wd / "m.json").read_text())
    assert m["bootstrap_count"] == 19 and m["ntt_forward_count"] == 19 * 4 * MINI.n
    assert set(m) == {"total_gates", "workers", "bootstrap_count", "ntt_forward_count", "ntt_inverse_count",
                      "wall_time_seconds", "gates_per_second", "per_wave_wall_time", "per_worker_busy_time"}
    assert main(["decrypt", "--secret", str(wd / "sk.bin"), "--circuit", str(wd / "adder.cir"),
                 "--in", str(wd / "out.bin")]) == 0
    assert "s = 17" in capsys.readouterr().out


@pytest.mark.gpu
def test_worker_count_does_not_change_output_bytes(wd, capsys):
    _keys(wd)
    _adder(wd)
    _encrypt(wd, 5, 6)
    blobs = []
    for k in ("1", "2", "4"):
        assert main(["run", "--eval", str(wd / "ek.bin"), "--circuit", str(wd / "adder.cir"),
                     "--in", str(wd / "in.bin"), "--out", str(wd / f"o{k}.bin"), "--workers", k]) == 0
        blobs.append((wd / f"o{k}.bin").read_bytes())
    assert blobs[0] == blobs[1] == blobs[2]
    capsys.readouterr()
