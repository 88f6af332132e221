"""CPU checks of the C-ABI library: it builds for sm_100a, loads, exports every
symbol include/maddness.h declares, and rejects malformed inputs before any
device work (no compute calls without a GPU)."""
import ctypes as ct
import os
import re
import struct

import pytest

from helpers import ROOT, model_bytes


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    path = __graft_entry__._builder().build()
    return ct.CDLL(path)


def _declared():
    src = open(os.path.join(ROOT, "include", "maddness.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mdn_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    names = _declared()
    assert len(names) >= 17
    for n in names:
        assert hasattr(lib, n), n


def test_binding_exposes_same_names():
    import paper_2106_10860_b200 as mdn
    for n in _declared():
        assert n in mdn.EXPORTED
    for n in ("mdn_model_load", "mdn_build_luts", "mdn_luts_serialize", "mdn_luts_load",
              "mdn_encode", "mdn_scan", "mdn_amm", "mdn_exec_create", "mdn_amm_host"):
        assert callable(getattr(mdn, n))


def test_sm100a_cubin_present():
    """The library carries sm_100a SASS (nvcc -gencode arch=compute_100a,code=sm_100a)."""
    import subprocess
    from paper_2106_10860_b200 import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(lib):
    lib.mdn_status_str.restype = ct.c_char_p
    assert lib.mdn_status_str(0) == b"ok"
    assert b"stream" in lib.mdn_status_str(-3)
    assert lib.mdn_abi_version() == 1


def _load(lib, blob):
    h, off = ct.c_void_p(), ct.c_size_t(0)
    lib.mdn_model_load.argtypes = [ct.c_void_p, ct.c_size_t, ct.c_int, ct.POINTER(ct.c_void_p),
                                   ct.POINTER(ct.c_size_t)]
    st = lib.mdn_model_load(blob, len(blob), 0, ct.byref(h), ct.byref(off))
    return st, off.value


def test_model_parser_errors(lib):
    blob = model_bytes("tiny")
    assert _load(lib, b"XXXX" + blob[4:]) == (-3, 0)
    st, off = _load(lib, blob[:100])
    assert st == -3 and off > 0
    assert _load(lib, blob[:4] + struct.pack("<I", 7) + blob[8:])[0] == -4
    bad = bytearray(blob)
    bad[-100] ^= 0xFF                               # inside P: only the fingerprint sees it
    st, off = _load(lib, bytes(bad))
    assert st == -3 and off == len(blob) - 8
    bad = bytearray(blob)
    bad[48 + 2 * 76] ^= 0xFF                        # codebook 2 sub_begin > sub_end
    assert _load(lib, bytes(bad)) == (-3, 48 + 2 * 76)
    bad = bytearray(blob)
    struct.pack_into("<H", bad, 48 + 8, 9999)       # split dim >= D
    assert _load(lib, bytes(bad))[0] in (-1, -3)


def test_model_nan_threshold_rejected(lib):
    """A NaN threshold has no meaning in Alg. 1 (and no 8-bit split value):
    MDN_EINVAL at its byte offset, before any device work."""
    import numpy as np
    import oracle as O
    om = O.read_model(model_bytes("tiny"))
    om.thr[2, 5] = np.nan
    st, off = _load(lib, O.write_model(om))
    assert st == -1 and off == 48 + 2 * 76 + 16 + 4 * 5


def test_luts_parser_errors(lib):
    h, off = ct.c_void_p(), ct.c_size_t(0)
    lib.mdn_luts_load.argtypes = [ct.c_void_p, ct.c_size_t, ct.c_int, ct.POINTER(ct.c_void_p),
                                  ct.POINTER(ct.c_size_t)]
    assert lib.mdn_luts_load(b"MDNX" + b"\0" * 60, 64, 0, ct.byref(h), ct.byref(off)) == -3
    hdr = b"MDNL" + struct.pack("<6I", 2, 4, 4, 16, 0, 1) + b"\0" * 40
    assert lib.mdn_luts_load(hdr, len(hdr), 0, ct.byref(h), ct.byref(off)) == -4
    hdr = b"MDNL" + struct.pack("<6I", 1, 4, 4, 16, 1, 3) + b"\0" * 40   # U not pow2
    assert lib.mdn_luts_load(hdr, len(hdr), 0, ct.byref(h), ct.byref(off)) == -1
    # U above the averaging-stack bound (mdn_build_luts caps U at 64): a crafted
    # blob must not reach the generic kernels' fixed-depth halves-recursion stack
    hdr = b"MDNL" + struct.pack("<6I", 1, 256, 4, 16, 1, 256) + b"\0" * 40
    assert lib.mdn_luts_load(hdr, len(hdr), 0, ct.byref(h), ct.byref(off)) == -1
    hdr = b"MDNL" + struct.pack("<6I", 1, 128, 4, 16, 1, 128) + b"\0" * 40
    assert lib.mdn_luts_load(hdr, len(hdr), 0, ct.byref(h), ct.byref(off)) == -1
    hdr = b"MDNL" + struct.pack("<6I", 1, 8, 4, 16, 0, 2) + b"\0" * 40    # exact mode, U != 1
    assert lib.mdn_luts_load(hdr, len(hdr), 0, ct.byref(h), ct.byref(off)) == -1


def test_null_and_shape_guards(lib):
    lib.mdn_encode.argtypes = [ct.c_void_p, ct.c_void_p, ct.c_int64, ct.c_int64, ct.c_void_p,
                               ct.c_void_p]
    assert lib.mdn_encode(None, None, 1, 1, None, None) == -1
    lib.mdn_amm.argtypes = [ct.c_void_p] * 3 + [ct.c_int64] * 2 + [ct.c_void_p, ct.c_int64,
                                                                   ct.c_void_p]
    assert lib.mdn_amm(None, None, None, 1, 1, None, 1, None) == -1


def test_binding_rejects_host_tensors():
    import numpy as np
    import torch

    import paper_2106_10860_b200 as mdn

    class Fake:
        C, D, _h = 4, 32, None
    with pytest.raises(TypeError):
        mdn.mdn_encode(Fake(), torch.zeros(4, 32), torch.zeros(4, 2, dtype=torch.uint8))
    with pytest.raises(TypeError):
        mdn._host_ptr(np.zeros((2, 2), np.float64), "A_host")


def test_no_unresolved_symbols(lib):
    """Every undefined dynamic symbol of the .so is a versioned system symbol
    (catches C/C++ linkage slips that only fail when a call is made)."""
    import subprocess
    from paper_2106_10860_b200 import LIB_PATH
    out = subprocess.run(["nm", "-D", "--undefined-only", LIB_PATH], capture_output=True,
                         text=True).stdout.split("\n")
    bad = [l for l in out if l.strip().startswith("U ") and "@" not in l]
    assert not bad, bad


def test_train_size_query_and_argument_errors(lib):
    """mdn_train's size query (buf == NULL) needs no device; bad shapes fail
    before any device work."""
    n = ct.c_size_t(0)
    lib.mdn_train.argtypes = [ct.c_void_p, ct.c_int64, ct.c_int64, ct.c_int, ct.c_int, ct.c_double,
                              ct.c_int, ct.c_void_p, ct.POINTER(ct.c_size_t)]
    assert lib.mdn_train(None, 0, 0, 512, 32, 1.0, 0, None, ct.byref(n)) == 0
    assert n.value == 48 + 76 * 32 + 64 * 32 * 512 + 8          # == len(cls100.mdnm)
    assert n.value == len(model_bytes("cls100"))
    assert lib.mdn_train(None, 0, 0, 8, 9, 1.0, 0, None, ct.byref(n)) == -1      # C > D
    assert lib.mdn_train(None, 0, 0, 8, 4, -1.0, 0, None, ct.byref(n)) == -1     # lambda < 0
    buf = ct.create_string_buffer(16)
    n = ct.c_size_t(16)
    assert lib.mdn_train(None, 10, 8, 8, 4, 1.0, 0, buf, ct.byref(n)) == -1      # capacity too small


def test_bench_split_dims_parser():
    """bench.py's independent model-header parser agrees with the oracle's reader."""
    import bench
    import oracle as O
    for name in ("tiny", "cls100", "scale"):
        blob = model_bytes(name)
        assert bench.split_dims(blob) == sorted(set(O.read_model(blob).dims.reshape(-1).tolist()))


def test_null_handle_guards_every_hot_path_call(lib):
    """Every device entry point rejects a NULL handle with MDN_EINVAL before
    touching a device (widened rows N1-N4 included)."""
    P, I = ct.c_void_p, ct.c_int64
    calls = {
        "mdn_encode_u8": ([P, P, I, I, P, P], (None, None, 1, 1, None, None)),
        "mdn_amm_u8": ([P, P, P, I, I, P, I, P], (None, None, None, 1, 1, None, 1, None)),
        "mdn_encode_cm": ([P, P, I, I, P, P], (None, None, 1, 1, None, None)),
        "mdn_amm_cm": ([P, P, P, I, I, P, I, P], (None, None, None, 1, 1, None, 1, None)),
        "mdn_encode_pq": ([P, P, I, I, P, P], (None, None, 1, 1, None, None)),
        "mdn_scan": ([P, P, I, P, P, I, P], (None, None, 1, None, None, 1, None)),
        "mdn_amm_host": ([P, P, I, I, P, I], (None, None, 1, 1, None, 1)),
        "mdn_amm_host_u8": ([P, P, I, I, P, I], (None, None, 1, 1, None, 1)),
        "mdn_encode_host": ([P, P, I, I, P], (None, None, 1, 1, None)),
        "mdn_encode_host_u8": ([P, P, I, I, P], (None, None, 1, 1, None)),
        "mdn_scan_host": ([P, P, I, P, I], (None, None, 1, None, 1)),
        "mdn_amm_cm_host": ([P, P, I, I, P, I], (None, None, 1, 1, None, 1)),
        "mdn_encode_cm_host": ([P, P, I, I, P], (None, None, 1, 1, None)),
        "mdn_encode_pq_host": ([P, P, I, I, P], (None, None, 1, 1, None)),
        "mdn_amm_pq_host": ([P, P, I, I, P, I], (None, None, 1, 1, None, 1)),
    }
    for name, (argtypes, args) in calls.items():
        f = getattr(lib, name)
        f.argtypes = argtypes
        assert f(*args) == -1, name
    # negative N is rejected too
    lib.mdn_encode.argtypes = [P, P, I, I, P, P]
    assert lib.mdn_encode(None, None, -1, 1, None, None) == -1


def test_package_without_library_fails_loudly(tmp_path):
    """The product path has no CPU fallback: importing the binding from a copy
    of the package that lacks libmaddness.so raises ImportError."""
    import shutil
    import subprocess
    import sys
    pkg = os.path.join(ROOT, "paper_2106_10860_b200")
    dst = tmp_path / "paper_2106_10860_b200"
    dst.mkdir()
    for name in os.listdir(pkg):
        if name.endswith(".py"):
            shutil.copy(os.path.join(pkg, name), dst / name)
    r = subprocess.run([sys.executable, "-c", "import paper_2106_10860_b200"], cwd=tmp_path,
                       env=dict(os.environ, PYTHONPATH=str(tmp_path)), capture_output=True,
                       text=True, timeout=120)
    assert r.returncode != 0
    assert "ImportError" in r.stderr and "no CPU fallback" in r.stderr
