"""ctypes front-end of oracle/gw_oracle.c plus the numpy glue of the reference's
gate layer -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every function restates a reference function; citations are to
/root/reference/pkg/src/gatewave/.  Parity of this restatement with the
reference itself is pinned by tests/test_oracle.py against
tests/golden/*.npz, which make_golden.py produced by running the reference.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

Q = 0xFFFFFFFF_00000001
_U32P = ctypes.POINTER(ctypes.c_uint32)
_U64P = ctypes.POINTER(ctypes.c_uint64)


def build() -> str:
    """Compile gw_oracle.c (gcc) into oracle/liboracle.so."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def use_native() -> str:
    """Rebuild for THIS host's CPU (-march=native: AVX-512 vectorises the
    transform loops, ~2x) and load that copy.  For the CPU-baseline timings,
    which run on the GPU box's host; the portable build stays the test copy."""
    global _lib, _LIB_PATH
    out = os.path.join(_HERE, "liboracle_native.so")
    subprocess.run(["gcc", "-O3", "-march=native", "-pthread", "-fPIC", "-std=c11", "-shared", "-o", out,
                    os.path.join(_HERE, "gw_oracle.c")], check=True)
    _LIB_PATH = out
    _lib = None
    lib()
    return out


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
                os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "gw_oracle.c"))):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_build_tables.argtypes = [ctypes.c_int, _U64P, _U64P, _U64P]
        L.orc_ntt_forward.argtypes = [_U64P, ctypes.c_int64, ctypes.c_int, _U64P]
        L.orc_ntt_inverse.argtypes = [_U64P, ctypes.c_int64, ctypes.c_int, _U64P, ctypes.c_uint64]
        L.orc_bk_to_ntt.argtypes = [_U32P, ctypes.c_int64, ctypes.c_int, _U64P, _U64P]
        L.orc_decompose_offset.argtypes = [ctypes.c_int, ctypes.c_int]
        L.orc_decompose_offset.restype = ctypes.c_uint32
        L.orc_blind_rotate.argtypes = [_U32P, ctypes.c_int64, ctypes.c_int, _U32P, ctypes.c_int,
                                       _U64P, ctypes.c_int, ctypes.c_int, _U64P, _U64P,
                                       ctypes.c_uint64, _U32P, ctypes.c_int]
        L.orc_extract.argtypes = [_U32P, ctypes.c_int64, ctypes.c_int, _U32P]
        L.orc_keyswitch.argtypes = [_U32P, ctypes.c_int64, ctypes.c_int, _U32P, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, _U32P, ctypes.c_int]
        _lib = L
    return _lib


def _p32(a):
    return a.ctypes.data_as(_U32P)


def _p64(a):
    return a.ctypes.data_as(_U64P)


def default_threads() -> int:
    return os.cpu_count() or 1


class Tables:
    """torus.py:219-270 (NttTables / build_ntt_tables)."""

    def __init__(self, n: int):
        self.n = n
        self.log_n = n.bit_length() - 1
        self.psi_brv = np.empty(n, np.uint64)
        self.ipsi_brv = np.empty(n, np.uint64)
        ninv = np.zeros(1, np.uint64)
        if lib().orc_build_tables(n, _p64(self.psi_brv), _p64(self.ipsi_brv), _p64(ninv)):
            raise ValueError(f"bad transform size {n}")
        self.n_inv = int(ninv[0])


_TABLES: dict[int, Tables] = {}


def tables(n: int) -> Tables:
    if n not in _TABLES:
        _TABLES[n] = Tables(n)
    return _TABLES[n]


def ntt_forward(rows: np.ndarray) -> np.ndarray:
    """torus.py:282-294"""
    a = np.array(rows, dtype=np.uint64, copy=True, order="C")
    n = a.shape[-1]
    lib().orc_ntt_forward(_p64(a), a.size // n, n, _p64(tables(n).psi_brv))
    return a


def ntt_inverse(rows: np.ndarray) -> np.ndarray:
    """torus.py:297-304"""
    a = np.array(rows, dtype=np.uint64, copy=True, order="C")
    n = a.shape[-1]
    t = tables(n)
    lib().orc_ntt_inverse(_p64(a), a.size // n, n, _p64(t.ipsi_brv), t.n_inv)
    return a


def bk_to_ntt(bk_data: np.ndarray) -> np.ndarray:
    """cggi.py:283-285: NTT-domain copy of the bootstrapping key."""
    bk = np.ascontiguousarray(bk_data, dtype=np.uint32)
    N = bk.shape[-1]
    out = np.empty(bk.shape, np.uint64)
    lib().orc_bk_to_ntt(_p32(bk), bk.size // N, N, _p64(tables(N).psi_brv), _p64(out))
    return out


def decompose_offset(bg_bits: int, levels: int) -> int:
    """cggi.py:516-522"""
    return int(lib().orc_decompose_offset(bg_bits, levels))


def blind_rotate(lin: np.ndarray, tv: np.ndarray, bk_ntt: np.ndarray, bg_bits: int, levels: int,
                 threads: int | None = None) -> np.ndarray:
    """cggi.py:592-667 (_blind_rotate_kernel): (B, n+1) u32 -> (B, 2, N) u32."""
    lin = np.ascontiguousarray(lin, dtype=np.uint32)
    tv = np.ascontiguousarray(tv, dtype=np.uint32)
    bk_ntt = np.ascontiguousarray(bk_ntt, dtype=np.uint64)
    B, W = lin.shape
    N = tv.shape[1]
    t = tables(N)
    acc = np.empty((B, 2, N), np.uint32)
    rc = lib().orc_blind_rotate(_p32(lin), B, W - 1, _p32(tv), N, _p64(bk_ntt), bg_bits, levels,
                                _p64(t.psi_brv), _p64(t.ipsi_brv), t.n_inv, _p32(acc),
                                threads or default_threads())
    if rc:
        raise RuntimeError(f"oracle blind_rotate failed ({rc})")
    return acc


def extract(acc: np.ndarray) -> np.ndarray:
    """cggi.py:695-704 (_extract_rows)"""
    acc = np.ascontiguousarray(acc, dtype=np.uint32)
    B, _, N = acc.shape
    out = np.empty((B, N + 1), np.uint32)
    lib().orc_extract(_p32(acc), B, N, _p32(out))
    return out


def keyswitch(exts: np.ndarray, ksk: np.ndarray, levels: int, gamma: int,
              threads: int | None = None) -> np.ndarray:
    """cggi.py:670-692 (_keyswitch_kernel)"""
    exts = np.ascontiguousarray(exts, dtype=np.uint32)
    ksk = np.ascontiguousarray(ksk, dtype=np.uint32)
    B = exts.shape[0]
    N = ksk.shape[0]
    width = ksk.shape[3]
    out = np.empty((B, width), np.uint32)
    lib().orc_keyswitch(_p32(exts), B, N, _p32(ksk), levels, gamma, width, _p32(out),
                        threads or default_threads())
    return out


# cggi.py:177-184 (_GATE_COMBO): (constant, w1, w2) in units of mu
GATE_COMBO = {"AND": (-1, 1, 1), "OR": (1, 1, 1), "NAND": (1, -1, -1), "NOR": (-1, -1, -1),
              "XOR": (2, 2, 2), "XNOR": (-2, -2, -2)}
GATE_ARITY = {"AND": 2, "OR": 2, "NAND": 2, "NOR": 2, "XOR": 2, "XNOR": 2, "NOT": 1, "MUX": 3,
              "CONST0": 0, "CONST1": 0, "COPY": 1}


class Keys:
    """Plain container of what the oracle needs from an eval key."""

    def __init__(self, n, N, bg_bits, l, ks_base_bits, ks_levels, mu, bk_data, ksk_data,
                 bk_ntt=None):
        self.n, self.N, self.bg_bits, self.l = n, N, bg_bits, l
        self.ks_base_bits, self.ks_levels, self.mu = ks_base_bits, ks_levels, mu
        self.ksk = np.ascontiguousarray(ksk_data, dtype=np.uint32)
        self.bk_ntt = bk_to_ntt(bk_data) if bk_ntt is None else bk_ntt

    @classmethod
    def from_params(cls, params, bk_data, ksk_data, bk_ntt=None):
        return cls(params.n, params.N, params.Bg_bits, params.l, params.ks_base_bits,
                   params.ks_levels, params.mu, bk_data, ksk_data, bk_ntt)

    def test_vector(self):
        tv = np.zeros((2, self.N), np.uint32)
        tv[1, :] = np.uint32(self.mu)
        return tv


def bootstrap_rows(lin, keys: Keys, threads=None):
    """cggi.py:707-727 (_bootstrap_rows)"""
    acc = blind_rotate(lin, keys.test_vector(), keys.bk_ntt, keys.bg_bits, keys.l, threads)
    return keyswitch(extract(acc), keys.ksk, keys.ks_levels, keys.ks_base_bits, threads)


def eval_gate_batch(kind: str, operands, keys: Keys, count=None, threads=None) -> np.ndarray:
    """cggi.py:785-854 (eval_gate_batch), kind given by its GateKind value."""
    mats = [np.ascontiguousarray(m, dtype=np.uint32) for m in operands]
    mu = keys.mu
    if kind in ("CONST0", "CONST1"):
        out = np.zeros((count, keys.n + 1), np.uint32)
        out[:, -1] = np.uint32(mu if kind == "CONST1" else (1 << 32) - mu)
        return out
    if kind == "COPY":
        return mats[0].copy()
    if kind == "NOT":
        return np.uint32(0) - mats[0]
    if kind in GATE_COMBO:
        c_mu, w1, w2 = GATE_COMBO[kind]
        lin = mats[0].astype(np.int64) * w1 + mats[1].astype(np.int64) * w2
        lin[:, -1] += c_mu * mu
        return bootstrap_rows((lin & 0xFFFFFFFF).astype(np.uint32), keys, threads)
    if kind == "MUX":
        sel, a, b = (m.astype(np.int64) for m in mats)
        lin1 = sel + a
        lin2 = b - sel
        lin1[:, -1] -= mu
        lin2[:, -1] -= mu
        both = (np.concatenate([lin1, lin2], axis=0) & 0xFFFFFFFF).astype(np.uint32)
        acc = blind_rotate(both, keys.test_vector(), keys.bk_ntt, keys.bg_bits, keys.l, threads)
        exts = extract(acc)
        B = mats[0].shape[0]
        pre = exts[:B] + exts[B:]
        pre[:, -1] += np.uint32(mu)
        return keyswitch(pre, keys.ksk, keys.ks_levels, keys.ks_base_bits, threads)
    raise ValueError(f"unhandled gate kind {kind!r}")
