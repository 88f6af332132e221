"""Host-parser hardening: mdn_model_load / mdn_luts_load
built with -fsanitize=address,undefined and fed 10,000 seeded mutants
(truncations, bit flips, byte and extreme-field overwrites, half of them with
a recomputed FNV-1a trailer so the field checks behind the checksum are
reached) of every model file in artifacts/ and of LUT streams of two shapes.
Every mutant must come back MDN_EFORMAT / MDN_EVERSION / MDN_EINVAL (or, if
still a valid stream, MDN_ECUDA at the first device call: no GPU here) with an
error offset inside the stream, and the sanitizers must report nothing.
Runs on the CPU box (tests/fuzz/parsers_fuzz.cpp)."""
import glob
import json
import os
import struct
import subprocess

import numpy as np
import pytest

from helpers import ARTIFACTS, ROOT, model_bytes

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
# one -Xcompiler per flag: nvcc splits a -Xcompiler value at commas
SAN = [x for f in ("-fsanitize=address", "-fsanitize=undefined", "-fno-sanitize-recover=undefined",
                   "-fno-omit-frame-pointer") for x in ("-Xcompiler", f)]


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    import __graft_entry__
    __graft_entry__._builder().build()                  # the library's other objects
    obj_dir = os.path.join(ROOT, "build", "obj")
    out = tmp_path_factory.mktemp("fuzz")
    host_o = str(out / "mdn_host_asan.o")
    inc = ["-I", os.path.join(ROOT, "include")]
    arch = ["-gencode", "arch=compute_100a,code=sm_100a"]
    subprocess.run([NVCC, *arch, "-std=c++17", "-O1", "-g", *SAN, *inc, "-c",
                    os.path.join(ROOT, "paper_2106_10860_b200", "csrc", "mdn_host.cpp"), "-o", host_o],
                   check=True, capture_output=True)
    objs = [o for o in sorted(glob.glob(os.path.join(obj_dir, "*.o")))
            if not o.endswith("mdn_host.cpp.o")]
    exe = str(out / "parsers_fuzz")
    subprocess.run([NVCC, *arch, "-std=c++17", "-O1", "-g", *SAN, *inc,
                    os.path.join(ROOT, "tests", "fuzz", "parsers_fuzz.cpp"), host_o, *objs,
                    "-Xlinker", "-rpath,/usr/local/cuda/lib64", "-L/usr/local/cuda/lib64",
                    "-Xlinker", "--as-needed", "-lcusolver", *SAN, "-o", exe],
                   check=True, capture_output=True)
    return exe, out


def _luts_blob(C, M, mode, U, seed):
    """A valid luts.mdnl v1 stream (include/maddness.h), fields from the oracle."""
    import oracle as O
    rng = np.random.default_rng(seed)
    T = rng.standard_normal((C, 16, M))
    Tq, delta, l, alpha = O.quantize_tables(T)
    beta = O.beta32(delta, alpha, O.debias_constant(C, U, mode))
    out = bytearray(b"MDNL")
    out += struct.pack("<6I", 1, C, M, 16, 0 if mode == "exact" else 1, 1 if mode == "exact" else U)
    out += struct.pack("<iffQ", int(l), float(alpha), float(beta), 0x1234)
    out += np.asarray(delta, "<f8").tobytes()
    out += np.ascontiguousarray(Tq, np.uint8).tobytes()
    h = 0xCBF29CE484222325
    for b in bytes(out):
        h = ((h ^ b) * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    out += struct.pack("<Q", h)
    return bytes(out)


def _run(harness, kind, blob, name, n=10000, seed=1):
    exe, out = harness
    path = out / f"{name}.bin"
    path.write_bytes(blob)
    env = dict(os.environ, ASAN_OPTIONS="detect_leaks=1:abort_on_error=0:halt_on_error=1:"
                                        "protect_shadow_gap=0",
               UBSAN_OPTIONS="halt_on_error=1:print_stacktrace=1")
    p = subprocess.run([exe, kind, str(path), str(n), str(seed)], capture_output=True, text=True,
                       env=env, timeout=600)
    assert p.returncode == 0, (p.stdout + p.stderr)[-4000:]
    assert "runtime error" not in p.stderr and "AddressSanitizer" not in p.stderr, p.stderr[-4000:]
    res = json.loads(p.stdout.strip().splitlines()[-1])
    assert res["mutants"] == n
    assert res["EFORMAT"] > 0.3 * n
    return res


@pytest.mark.parametrize("name", sorted(os.path.basename(f)[:-5]
                                        for f in glob.glob(os.path.join(ARTIFACTS, "*.mdnm"))
                                        if os.path.getsize(f) < 1_100_000))
def test_fuzz_model_parser(harness, name):
    blob = model_bytes(name)
    res = _run(harness, "model", blob, name, n=10000 if len(blob) < 300_000 else 2000)
    print(name, res)
    assert res["EINVAL"] + res["EVERSION"] > 0           # the field checks were reached


@pytest.mark.parametrize("C,M,mode,U", [(4, 4, "avg", 4), (32, 100, "exact", 1)])
def test_fuzz_luts_parser(harness, C, M, mode, U):
    res = _run(harness, "luts", _luts_blob(C, M, mode, U, seed=C + M), f"luts_{C}_{M}")
    assert res["EINVAL"] + res["EVERSION"] > 0


def test_unmutated_streams_reach_the_device_call(harness):
    """Sanity: the unmutated streams pass every parser check (so the mutants
    above are rejected for their mutation, not for the base stream)."""
    exe, out = harness
    for kind, blob, name in (("model", model_bytes("tiny"), "base_model"),
                             ("luts", _luts_blob(4, 4, "avg", 4, 3), "base_luts")):
        path = out / f"{name}.bin"
        path.write_bytes(blob)
        p = subprocess.run([exe, kind, str(path), "0", "1"], capture_output=True, text=True,
                           env=dict(os.environ, ASAN_OPTIONS="protect_shadow_gap=0"), timeout=120)
        assert p.returncode == 0, p.stderr
        st = json.loads(p.stdout.strip().splitlines()[-1])["status"]
        # MDN_ECUDA: parsed, then the first device call fails (no GPU here);
        # MDN_OK where a GPU is visible
        assert st in (-6, 0), st
