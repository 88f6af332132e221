"""Model file round trip and error rules (format: include/maddness.h)."""
import struct

import numpy as np
import pytest

import oracle as O


def _small_model():
    rng = np.random.default_rng(21)
    A = np.maximum(rng.standard_normal((300, 12)), 0).astype(np.float32)
    return O.train(A, 3)


def test_roundtrip_bit_exact():
    m = _small_model()
    blob = O.write_model(m)
    m2 = O.read_model(blob)
    assert O.write_model(m2) == blob
    assert (m2.dims == m.dims).all() and m2.thr.tobytes() == m.thr.tobytes()
    assert m2.P.tobytes() == m.P.tobytes() and m2.sub == m.sub
    assert len(blob) == 48 + 76 * m.C + 4 * 16 * m.C * m.D + 8


def test_errors():
    blob = O.write_model(_small_model())
    with pytest.raises(ValueError):
        O.read_model(blob[:-9])                          # truncated
    with pytest.raises(ValueError):
        O.read_model(b"XXXX" + blob[4:])                 # bad magic
    with pytest.raises(ValueError):
        O.read_model(blob[:4] + struct.pack("<I", 2) + blob[8:])   # version
    bad = bytearray(blob)
    bad[60] ^= 1
    with pytest.raises(ValueError):
        O.read_model(bytes(bad))                         # fingerprint


def test_fnv_reference_values():
    # FNV-1a 64 published test vectors (empty string, "a")
    from oracle.model_file import fnv1a64
    assert fnv1a64(b"") == 0xCBF29CE484222325
    assert fnv1a64(b"a") == 0xAF63DC4C8601EC8C
