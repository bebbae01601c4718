"""ARFX files: byte-compatible with the reference's
serial.py.  tests/golden/arfx holds files the unmodified reference wrote
(tests/golden/make_arfx.py); these tests read them, rewrite them bit for bit,
and check every FormatError / ParamsMismatchError path the reference has
(serial.py:60-179; its tests/test_serial.py covers the same cases)."""
import hashlib
import json
import os
import shutil

import numpy as np
import pytest

from conftest import MINI

GOLD = os.path.join(os.path.dirname(__file__), "golden", "arfx")
DIG = json.load(open(os.path.join(GOLD, "digests.json")))
WIRES = [9, 3, 41, 0, 7]
BITS = np.array([1, 0, 1, 1, 0], np.uint8)


def _sha(path):
    return hashlib.sha256(open(path, "rb").read()).hexdigest()


@pytest.fixture(scope="module")
def keys():
    from paper_2306_11006_b200.cggi import keygen
    return keygen(MINI, seed=2024)


def test_params_block_and_digest():
    from paper_2306_11006_b200 import serial as S
    from paper_2306_11006_b200.cggi import PARAM_128
    raw = open(os.path.join(GOLD, "p128.params"), "rb").read()
    assert S.params_to_bytes(PARAM_128) == raw and len(raw) == 44
    assert S.params_from_bytes(raw) == PARAM_128
    assert S.params_digest(PARAM_128).hex() == DIG["p128_params_digest"]
    with pytest.raises(S.FormatError):
        S.params_from_bytes(raw[:-1])


def test_reads_reference_files(keys):
    from paper_2306_11006_b200 import serial as S
    from paper_2306_11006_b200.cggi import decrypt_rows
    sk = S.read_secret_key(os.path.join(GOLD, "mini.sk"))
    assert sk.params == MINI
    assert np.array_equal(sk.lwe_sk, keys.lwe_sk) and np.array_equal(sk.rlwe_sk, keys.rlwe_sk)
    ek = S.read_eval_key(os.path.join(GOLD, "mini.ek"))
    assert ek.params == MINI
    assert np.array_equal(ek.bk.data, keys.bootstrapping_key.data)
    assert np.array_equal(ek.ksk.data, keys.keyswitch_key.data)
    b = S.read_bundle(os.path.join(GOLD, "mini.bundle"), MINI)
    assert sorted(b) == sorted(WIRES)
    got = decrypt_rows(sk.lwe_sk, np.stack([b[w] for w in WIRES]))
    assert np.array_equal(got, BITS)


def test_writes_reference_bytes(keys, tmp_path):
    from paper_2306_11006_b200 import serial as S
    from paper_2306_11006_b200.cggi import encrypt_bits
    from paper_2306_11006_b200.rng import SeededRng
    S.write_secret_key(str(tmp_path / "k.sk"), keys)
    S.write_eval_key(str(tmp_path / "k.ek"), keys)
    rows = encrypt_bits(MINI, keys.lwe_sk, BITS, SeededRng(77))
    S.write_bundle(str(tmp_path / "c.bundle"), MINI, {w: rows[k] for k, w in enumerate(WIRES)})
    assert _sha(tmp_path / "k.sk") == DIG["mini.sk"]
    assert _sha(tmp_path / "k.ek") == DIG["mini.ek"]
    assert _sha(tmp_path / "c.bundle") == DIG["mini.bundle"]
    # EvalKey and SecretKey objects write the same bytes as the KeySet
    S.write_eval_key(str(tmp_path / "e.ek"), keys.eval_key())
    S.write_secret_key(str(tmp_path / "s.sk"), keys.secret_key())
    assert _sha(tmp_path / "e.ek") == DIG["mini.ek"] and _sha(tmp_path / "s.sk") == DIG["mini.sk"]


def _corrupt(tmp_path, name, edit):
    dst = tmp_path / name
    shutil.copy(os.path.join(GOLD, name), dst)
    raw = bytearray(open(dst, "rb").read())
    raw = edit(raw)
    open(dst, "wb").write(bytes(raw))
    return str(dst)


@pytest.mark.parametrize("reader", ["sk", "ek", "bundle"])
def test_format_errors(tmp_path, reader):
    from paper_2306_11006_b200 import serial as S
    name = {"sk": "mini.sk", "ek": "mini.ek", "bundle": "mini.bundle"}[reader]

    def read(p):
        if reader == "sk":
            return S.read_secret_key(p)
        if reader == "ek":
            return S.read_eval_key(p)
        return S.read_bundle(p, MINI)

    def set_bytes(off, val):
        def f(raw):
            raw[off:off + len(val)] = val
            return raw
        return f

    cases = {
        "magic": set_bytes(0, b"ARFY"),
        "version": set_bytes(4, (2).to_bytes(2, "little")),
        "kind": set_bytes(6, (3 if reader != "bundle" else 1).to_bytes(2, "little")),
        "truncated": lambda raw: raw[:-3],
        "trailing": lambda raw: raw + b"\0",
        "empty": lambda raw: raw[:0],
    }
    for what, edit in cases.items():
        with pytest.raises(S.FormatError):
            read(_corrupt(tmp_path, name, edit))


def test_bundle_param_mismatch_and_duplicates(tmp_path):
    from paper_2306_11006_b200 import serial as S
    from paper_2306_11006_b200.cggi import ParamSet
    other = ParamSet(n=16, N=64, lwe_noise_std=2.0 ** -20, rlwe_noise_std=1e-9, Bg_bits=9, l=2,
                     ks_base_bits=2, ks_levels=8, mu=1 << 28)
    with pytest.raises(S.ParamsMismatchError):
        S.read_bundle(os.path.join(GOLD, "mini.bundle"), other)
    # second record's wire id rewritten to equal the first's
    rec = 4 + 4 * (MINI.n + 1)
    first = 8 + 8 + 4

    def dup(raw):
        raw[first + rec:first + rec + 4] = raw[first:first + 4]
        return raw
    with pytest.raises(S.FormatError, match="duplicate"):
        S.read_bundle(_corrupt(tmp_path, "mini.bundle", dup), MINI)
    with pytest.raises(S.FormatError):
        S.write_bundle(str(tmp_path / "x.bundle"), MINI, {1: np.zeros(MINI.n, np.uint32)})
    S.write_bundle(str(tmp_path / "empty.bundle"), MINI, {})
    assert S.read_bundle(str(tmp_path / "empty.bundle"), MINI) == {}
