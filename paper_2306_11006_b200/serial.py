"""ARFX key and ciphertext-bundle files, byte-compatible with the reference
(gatewave/serial.py:1-179), so one set of key bytes feeds both the CPU
reference and this engine.

Layout (little-endian throughout; serial.py:26-35):

    header   "ARFX" | u16 version = 1 | u16 kind (1 secret, 2 eval, 3 bundle)
    secret   params block | lwe_sk u8[n] | rlwe_sk u8[N]
    eval     params block | bk u32[n, 2l, 2, N] | ksk u32[N, t, 2^gamma - 1, n+1]
    bundle   sha256(params block)[:8] | u32 count | count x (u32 wire, u32[n+1])
             records in ascending wire order

    params block = u32 n, N, Bg_bits, l, ks_base_bits, ks_levels, mu
                   | f64 lwe_noise_std, rlwe_noise_std                (44 bytes)

The bootstrapping key is stored in the coefficient domain.  The reference
transforms it into its NTT domain on the host when it loads an evaluation key
(serial.py:134-136 -> EvalKey.build).  Here `read_eval_key(..., upload=True)`
hands the coefficient-domain key straight to the device, which builds its
transform-domain image on the GPU (gw_upload_keys).

Errors mirror the reference's: FormatError for a structurally bad file
(magic, version, kind, truncation, trailing bytes, duplicate or mis-shaped
wires), ParamsMismatchError for a bundle made under other parameters.  Both
are ValueErrors.
"""
from __future__ import annotations

import hashlib
from typing import BinaryIO, Mapping

import numpy as np

from .cggi import EvalKey, KeySet, ParamSet, SecretKey  # noqa: F401  (KeySet: annotations)

MAGIC = b"ARFX"
FORMAT_VERSION = 1
KIND_SECRET, KIND_EVAL, KIND_BUNDLE = 1, 2, 3
_KIND_NAMES = {KIND_SECRET: "secret-key", KIND_EVAL: "evaluation-key", KIND_BUNDLE: "ciphertext-bundle"}

# one record dtype per fixed-size block: decoding is a single np.frombuffer
_HEADER = np.dtype([("magic", "S4"), ("version", "<u2"), ("kind", "<u2")])
_PARAMS = np.dtype([("n", "<u4"), ("N", "<u4"), ("Bg_bits", "<u4"), ("l", "<u4"),
                    ("ks_base_bits", "<u4"), ("ks_levels", "<u4"), ("mu", "<u4"),
                    ("lwe_noise_std", "<f8"), ("rlwe_noise_std", "<f8")])
_INT_FIELDS = ("n", "N", "Bg_bits", "l", "ks_base_bits", "ks_levels", "mu")


class FormatError(ValueError):
    """Structurally bad key/bundle file."""


class ParamsMismatchError(ValueError):
    """File was produced under different scheme parameters."""


# -- parameter block ----------------------------------------------------------

def params_to_bytes(p: ParamSet) -> bytes:
    rec = np.zeros((), _PARAMS)
    for name in _INT_FIELDS:
        rec[name] = getattr(p, name)
    rec["lwe_noise_std"], rec["rlwe_noise_std"] = p.lwe_noise_std, p.rlwe_noise_std
    return rec.tobytes()


def params_from_bytes(buf: bytes) -> ParamSet:
    if len(buf) != _PARAMS.itemsize:
        raise FormatError(f"parameter block is {len(buf)} bytes, expected {_PARAMS.itemsize}")
    rec = np.frombuffer(buf, _PARAMS)[0]
    ints = {name: int(rec[name]) for name in _INT_FIELDS}
    return ParamSet(lwe_noise_std=float(rec["lwe_noise_std"]),
                    rlwe_noise_std=float(rec["rlwe_noise_std"]), **ints)


def params_digest(p: ParamSet) -> bytes:
    """First 8 bytes of sha256(params block): the bundle's parameter check."""
    return hashlib.sha256(params_to_bytes(p)).digest()[:8]


# -- low-level reading --------------------------------------------------------

class _Reader:
    """Sequential reads that fail with FormatError instead of returning short."""

    def __init__(self, f: BinaryIO):
        self.f = f

    def take(self, nbytes: int, what: str) -> bytes:
        buf = self.f.read(nbytes)
        if len(buf) != nbytes:
            raise FormatError(f"truncated file while reading {what}")
        return buf

    def array(self, dtype, shape, what: str) -> np.ndarray:
        dt = np.dtype(dtype)
        count = int(np.prod(shape, dtype=np.int64))
        return np.frombuffer(self.take(count * dt.itemsize, what), dt).reshape(shape)

    def header(self, kind: int) -> None:
        h = np.frombuffer(self.take(_HEADER.itemsize, "header"), _HEADER)[0]
        what = _KIND_NAMES[kind]
        if bytes(h["magic"]) != MAGIC:
            raise FormatError(f"not a {what} file (bad magic)")
        if int(h["version"]) != FORMAT_VERSION:
            raise FormatError(f"unsupported format version {int(h['version'])}")
        if int(h["kind"]) != kind:
            raise FormatError(f"expected {what} data, found kind {int(h['kind'])}")

    def params(self) -> ParamSet:
        return params_from_bytes(self.take(_PARAMS.itemsize, "parameters"))

    def end(self, what: str) -> None:
        if self.f.read(1):
            raise FormatError(f"trailing data after {what}")


def _header_bytes(kind: int) -> bytes:
    h = np.zeros((), _HEADER)
    h["magic"], h["version"], h["kind"] = MAGIC, FORMAT_VERSION, kind
    return h.tobytes()


def _le(arr, dtype: str) -> bytes:
    return np.ascontiguousarray(np.asarray(arr).astype(dtype, copy=False)).tobytes()


def _write(path: str, chunks) -> None:
    with open(path, "wb") as f:
        for c in chunks:
            f.write(c)


# -- secret keys --------------------------------------------------------------

def write_secret_key(path: str, key: SecretKey | KeySet) -> None:
    sk = key.secret_key() if hasattr(key, "secret_key") else key  # KeySet (ours or the reference's)
    _write(path, (_header_bytes(KIND_SECRET), params_to_bytes(sk.params),
                  _le(sk.lwe_sk, "u1"), _le(sk.rlwe_sk, "u1")))


def read_secret_key(path: str) -> SecretKey:
    with open(path, "rb") as f:
        r = _Reader(f)
        r.header(KIND_SECRET)
        p = r.params()
        lwe = r.array("u1", (p.n,), "LWE secret")
        rlwe = r.array("u1", (p.N,), "ring secret")
        r.end("secret key")
    return SecretKey(params=p, lwe_sk=lwe.astype(np.uint32), rlwe_sk=rlwe.astype(np.uint32))


# -- evaluation keys ----------------------------------------------------------

def _key_shapes(p: ParamSet):
    return (p.n, 2 * p.l, 2, p.N), (p.N, p.ks_levels, (1 << p.ks_base_bits) - 1, p.n + 1)


def write_eval_key(path: str, keys: KeySet | EvalKey) -> None:
    ek = keys.eval_key() if hasattr(keys, "eval_key") else keys
    _write(path, (_header_bytes(KIND_EVAL), params_to_bytes(ek.params),
                  _le(ek.bk.data, "<u4"), _le(ek.ksk.data, "<u4")))


def read_eval_key(path: str, upload: bool = False) -> EvalKey:
    """Evaluation key from an ARFX file.  upload=True also places it on the
    GPU now (device-side transform), instead of at the first gate."""
    with open(path, "rb") as f:
        r = _Reader(f)
        r.header(KIND_EVAL)
        p = r.params()
        bk_shape, ks_shape = _key_shapes(p)
        bk = r.array("<u4", bk_shape, "bootstrapping key")
        ksk = r.array("<u4", ks_shape, "keyswitch key")
        r.end("evaluation key")
    ek = EvalKey.build(p, bk.astype(np.uint32), ksk.astype(np.uint32))
    if upload:
        ek.engine()
    return ek


# -- ciphertext bundles -------------------------------------------------------

def write_bundle(path: str, params: ParamSet, wires: Mapping[int, np.ndarray]) -> None:
    """Wire-id-sorted (id, sample) records; every sample must be (n+1,)."""
    width = params.n + 1
    ids = sorted(wires)
    rec = np.dtype([("wire", "<u4"), ("row", "<u4", (width,))])
    body = np.empty(len(ids), rec)
    for k, w in enumerate(ids):
        row = np.asarray(wires[w], dtype=np.uint32)
        if row.shape != (width,):
            raise FormatError(f"wire {w}: sample has shape {row.shape}, expected ({width},)")
        body[k] = (w, row)
    _write(path, (_header_bytes(KIND_BUNDLE), params_digest(params),
                  np.uint32(len(ids)).astype("<u4").tobytes(), body.tobytes()))


def read_bundle(path: str, params: ParamSet) -> dict[int, np.ndarray]:
    width = params.n + 1
    with open(path, "rb") as f:
        r = _Reader(f)
        r.header(KIND_BUNDLE)
        if r.take(8, "parameter digest") != params_digest(params):
            raise ParamsMismatchError("bundle was produced under a different parameter set")
        count = int(r.array("<u4", (1,), "record count")[0])
        out: dict[int, np.ndarray] = {}
        for _ in range(count):
            w = int(r.array("<u4", (1,), "wire id")[0])
            if w in out:
                raise FormatError(f"duplicate wire {w} in bundle")
            out[w] = r.array("<u4", (width,), f"wire {w} sample").astype(np.uint32)
        r.end("bundle records")
    return out


__all__ = ["MAGIC", "FORMAT_VERSION", "KIND_SECRET", "KIND_EVAL", "KIND_BUNDLE", "FormatError",
           "ParamsMismatchError", "params_to_bytes", "params_from_bytes", "params_digest",
           "write_secret_key", "read_secret_key", "write_eval_key", "read_eval_key",
           "write_bundle", "read_bundle"]
