"""Reader/writer for the reference's ``.cplx`` container
(``include/shlr/io.hpp:24-28``, ``src/io.cpp:35-103``):

    "CPLX0001" | u8 precision (0 = 32-bit, 1 = 64-bit) | u32 ndim |
    ndim x u64 dims | interleaved (re, im) scalars, little-endian, row-major.

Masks use the same container (0/1 real values) plus a ``.meta`` key=value
sidecar (``src/sampling.cpp:196-236``).
"""
from __future__ import annotations

import struct
from typing import Dict, Tuple

import numpy as np

MAGIC = b"CPLX0001"


def write_cplx(arr: np.ndarray, path: str, precision: int = 64) -> None:
    if precision not in (32, 64):
        raise ValueError("precision must be 32 or 64")
    a = np.asarray(arr)
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<B", 0 if precision == 32 else 1))
        f.write(struct.pack("<I", a.ndim))
        for d in a.shape:
            f.write(struct.pack("<Q", d))
        dt = np.complex64 if precision == 32 else np.complex128
        f.write(np.ascontiguousarray(a, dtype=dt).tobytes())


def read_cplx(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    if data[:8] != MAGIC:
        raise ValueError(f"bad magic in {path}")
    prec = data[8]
    ndim = struct.unpack_from("<I", data, 9)[0]
    dims = struct.unpack_from("<" + "Q" * ndim, data, 13)
    off = 13 + 8 * ndim
    dt = np.complex64 if prec == 0 else np.complex128
    n = int(np.prod(dims)) if ndim else 0
    arr = np.frombuffer(data, dtype=dt, count=n, offset=off).reshape(dims)
    return arr.astype(np.complex128)


def write_mask(bits: np.ndarray, path: str, meta: Dict[str, object] | None = None) -> None:
    b = np.asarray(bits)
    if b.ndim == 1:
        b = b.reshape(1, -1)
    write_cplx(b.astype(np.float64).astype(np.complex128), path)
    meta = dict(meta or {})
    with open(path + ".meta", "w") as f:
        for k in ("generator", "seed", "rate", "acs", "pf"):
            f.write(f"{k}={meta.get(k, '' if k == 'generator' else (1 if k == 'pf' else 0))}\n")


def read_mask(path: str) -> Tuple[np.ndarray, Dict[str, str]]:
    t = read_cplx(path)
    if t.ndim != 2:
        raise ValueError("mask file must be rank 2")
    bits = (t.real > 0.5).astype(np.uint8)
    meta: Dict[str, str] = {}
    try:
        with open(path + ".meta") as f:
            for line in f:
                if "=" in line:
                    k, v = line.rstrip("\n").split("=", 1)
                    meta[k] = v
    except FileNotFoundError:
        pass
    return bits, meta
