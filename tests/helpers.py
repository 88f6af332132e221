"""Test helpers: artifact loading, the luts.mdnl parser used to compare library
bytes with the oracle, and device availability."""
import os
import struct

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARTIFACTS = os.path.join(ROOT, "artifacts")


def model_bytes(name: str) -> bytes:
    with open(os.path.join(ARTIFACTS, f"{name}.mdnm"), "rb") as f:
        return f.read()


def parse_luts(blob: bytes) -> dict:
    """Parse luts.mdnl v1 (include/maddness.h) independently of the library."""
    assert blob[:4] == b"MDNL"
    ver, C, M, K, mode, U = struct.unpack_from("<6I", blob, 4)
    l, alpha, beta, mfp = struct.unpack_from("<iffQ", blob, 28)
    off = 48
    delta = np.frombuffer(blob, "<f8", C, off)
    off += 8 * C
    Tq = np.frombuffer(blob, np.uint8, C * K * M, off).reshape(C, K, M)
    off += C * K * M
    (fp,) = struct.unpack_from("<Q", blob, off)
    assert off + 8 == len(blob)
    return dict(ver=ver, C=C, M=M, K=K, mode=mode, U=U, l=l, alpha=np.float32(alpha),
                beta32=np.float32(beta), model_fp=mfp, delta=delta, Tq=Tq, fp=fp)


def cuda_ok() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
