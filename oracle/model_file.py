"""Oracle-side writer/reader of the ``model.mdnm`` v1 file -- TEST INFRASTRUCTURE ONLY.

The byte layout is the documented contract in ``include/maddness.h``
(section "model.mdnm v1"); the library has its own independent parser.
All fields little-endian:

  "MDNM" | u32 ver=1 | u32 C | u32 D | u32 K=16 | u32 flags (bit0 = ridge,
                                                            bit1 = PQ model)
  f64 lambda | u64 n_train | u64 seed
  C x { u32 sub_begin | u32 sub_end | u16 dim[4] | f32 thr[15] }
  f32 P[16C][D]
  u64 fingerprint = FNV-1a 64 of every preceding byte
"""
from __future__ import annotations

import struct

import numpy as np

from .maddness import K, Model

MAGIC = b"MDNM"
VERSION = 1


def write_model(model: Model) -> bytes:
    out = bytearray()
    out += MAGIC
    flags = (1 if model.ridge else 0) | (2 if getattr(model, "pq", False) else 0)
    out += struct.pack("<5I", VERSION, model.C, model.D, K, flags)
    out += struct.pack("<dQQ", float(model.lam), int(model.n_train), int(model.seed))
    for c in range(model.C):
        b, e = model.sub[c]
        out += struct.pack("<2I", b, e)
        out += struct.pack("<4H", *[int(x) for x in model.dims[c]])
        out += np.asarray(model.thr[c], "<f4").tobytes()
    out += np.ascontiguousarray(model.P, "<f4").tobytes()
    out += struct.pack("<Q", fnv1a64(bytes(out)))
    return bytes(out)


def fnv1a64(data: bytes) -> int:
    """FNV-1a 64, byte-serial definition, in plain Python ints."""
    h = 0xCBF29CE484222325
    for b in data:
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def read_model(buf: bytes) -> Model:
    if len(buf) < 48 or buf[:4] != MAGIC:
        raise ValueError("bad magic / truncated header")
    ver, C, D, k, flags = struct.unpack_from("<5I", buf, 4)
    if ver != VERSION:
        raise ValueError(f"unsupported version {ver}")
    if k != K:
        raise ValueError("K must be 16")
    lam, n_train, seed = struct.unpack_from("<dQQ", buf, 24)
    off = 48
    need = off + C * 76 + 4 * K * C * D + 8
    if len(buf) < need:
        raise ValueError(f"truncated at {len(buf)} (need {need})")
    sub, dims, thr = [], np.zeros((C, 4), np.int64), np.zeros((C, 15), np.float32)
    for c in range(C):
        b, e = struct.unpack_from("<2I", buf, off)
        sub.append((b, e))
        dims[c] = struct.unpack_from("<4H", buf, off + 8)
        thr[c] = np.frombuffer(buf, "<f4", 15, off + 16)
        off += 76
    P = np.frombuffer(buf, "<f4", K * C * D, off).reshape(K * C, D).astype(np.float32)
    off += 4 * K * C * D
    (fp,) = struct.unpack_from("<Q", buf, off)
    if fp != fnv1a64(buf[:off]):
        raise ValueError("fingerprint mismatch")
    return Model(C=C, D=D, sub=sub, dims=dims, thr=thr, P=P, lam=lam,
                 n_train=n_train, seed=seed, ridge=bool(flags & 1), pq=bool(flags & 2))
