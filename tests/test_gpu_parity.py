"""GPU parity: the CUDA path through the C-ABI vs the oracle, element by element.

Bar: codes, integer sums and LUT bytes bit-exact;
fp32 outputs bit-exact by construction (one rounding of alpha*S + beta32 on
both sides), asserted against the north_star contract of 1e-5 relative too.
"""
import numpy as np
import pytest

import oracle as O
from datagen.synth import CONFIGS, make_config_data, relu_W, relu_lowrank_torch
from helpers import model_bytes, parse_luts

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REL_TOL = 1e-5  # north_star: dequantised fp32 outputs within 1e-5 relative


@pytest.fixture(scope="module")
def mdn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as m
    return m


_cache = {}


def _setup(mdn, name, n_test=None):
    key = (name, n_test)
    if key not in _cache:
        blob = model_bytes(name)
        om = O.read_model(blob)
        A, B = _data(name, n_test)
        _cache[key] = (blob, om, A, B)
    blob, om, A, B = _cache[key]
    return mdn.mdn_model_load(blob, 0), om, A, B


def _data(name, n_test):
    spec = CONFIGS[name]
    if spec.kind == "relu":
        if name == "scale":
            _, A, B = make_config_data(name, n_test=n_test or 4096)
        else:
            _, A, B = make_config_data(name, n_test=n_test)
    else:
        _, A, B = make_config_data(name, n_test=n_test or 300_000, n_train=0)
    return A, B


def _assert_out(got, want):
    got = np.asarray(got)
    assert got.dtype == np.float32 and want.dtype == np.float32
    rel = np.abs(got.astype(np.float64) - want) / np.maximum(np.abs(want.astype(np.float64)), 1e-30)
    assert (rel <= REL_TOL).all(), f"max rel {rel.max()}"
    assert (got.view(np.uint32) == want.view(np.uint32)).all(), "fp32 outputs not bit-identical"


CFGS = ["tiny", "cls10_c16", "cls10_c32", "cls10_c64", "cls100", "image", "scale"]
MODES = [("exact", 0), ("avg", 1)]


@pytest.mark.parametrize("name", CFGS)
@pytest.mark.parametrize("mode", MODES, ids=["exact", "avg"])
def test_luts_bit_exact(mdn, name, mode):
    model, om, A, B = _setup(mdn, name)
    spec = CONFIGS[name]
    luts = mdn.mdn_build_luts(model, B, mode[1], spec.U)
    got = parse_luts(mdn.mdn_luts_serialize(luts))
    want = O.make_luts(om, B, mode[0], spec.U)
    assert got["l"] == want.l
    assert got["alpha"] == want.alpha
    assert got["beta32"].view(np.uint32) == want.beta32.view(np.uint32)
    assert got["delta"].tobytes() == np.asarray(want.delta, np.float64).tobytes()
    assert (got["Tq"] == want.Tq).all()
    assert got["model_fp"] == model.fingerprint


@pytest.mark.parametrize("name", CFGS)
def test_encode_bit_exact(mdn, name):
    model, om, A, B = _setup(mdn, name)
    dA = torch.from_numpy(A).cuda()
    codes = torch.empty((A.shape[0], (om.C + 1) // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode(model, dA, codes)
    want = O.pack_codes(O.encode(A, om))
    got = codes.cpu().numpy()
    assert (got == want).all(), f"{(got != want).sum()} code bytes differ"


@pytest.mark.parametrize("name", CFGS)
@pytest.mark.parametrize("mode", MODES, ids=["exact", "avg"])
def test_scan_and_amm_bit_exact(mdn, name, mode):
    model, om, A, B = _setup(mdn, name)
    spec = CONFIGS[name]
    luts = mdn.mdn_build_luts(model, B, mode[1], spec.U)
    oluts = O.make_luts(om, B, mode[0], spec.U)
    codes_o, S_o, out_o = O.amm(A, om, oluts)
    N = A.shape[0]
    codes = torch.from_numpy(O.pack_codes(codes_o)).cuda()       # oracle codes as input
    sums = torch.empty((N, spec.M), dtype=torch.int32, device="cuda")
    out = torch.empty((N, spec.M), dtype=torch.float32, device="cuda")
    mdn.mdn_scan(luts, codes, sums=sums, out=out)
    assert (sums.cpu().numpy() == S_o).all()
    _assert_out(out.cpu().numpy(), out_o)
    out2 = torch.full((N, spec.M), float("nan"), device="cuda")
    mdn.mdn_amm(model, luts, torch.from_numpy(A).cuda(), out2)
    _assert_out(out2.cpu().numpy(), out_o)


@pytest.mark.parametrize("N", [0, 1, 31, 33, 257, 1000, 4099])
def test_ragged_and_tiny_N(mdn, N):
    model, om, A, B = _setup(mdn, "cls100")
    luts = mdn.mdn_build_luts(model, B, 0)
    oluts = O.make_luts(om, B, "exact")
    A = A[:N]
    out = torch.zeros((N, 100), device="cuda")
    mdn.mdn_amm(model, luts, torch.from_numpy(np.ascontiguousarray(A)).cuda(), out)
    if N:
        _assert_out(out.cpu().numpy(), O.amm(A, om, oluts)[2])


def test_strided_and_misaligned_inputs(mdn):
    """lda > D, ldo > M, and an A base pointer not 16-B aligned (generic path)."""
    model, om, A, B = _setup(mdn, "cls10_c16")
    luts = mdn.mdn_build_luts(model, B, 1, 16)
    oluts = O.make_luts(om, B, "avg", 16)
    A = A[:3001]
    want = O.amm(A, om, oluts)[2]
    big = torch.zeros((A.shape[0], 512 + 7), device="cuda")
    big[:, 3:515] = torch.from_numpy(A).cuda()
    view = big[:, 3:515]                                  # lda = 519, offset 12 B
    outbig = torch.zeros((A.shape[0], 13), device="cuda")
    out = outbig[:, :10]                                  # ldo = 13
    mdn.mdn_amm(model, luts, view, out)
    _assert_out(out.cpu().numpy(), want)
    codes = torch.empty((A.shape[0], 8), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode(model, view, codes)
    assert (codes.cpu().numpy() == O.pack_codes(O.encode(A, om))).all()


def test_luts_serialize_load_roundtrip(mdn):
    model, om, A, B = _setup(mdn, "cls100")
    luts = mdn.mdn_build_luts(model, B, 1, 16)
    blob = mdn.mdn_luts_serialize(luts)
    luts2 = mdn.mdn_luts_load(blob, 0)
    assert mdn.mdn_luts_serialize(luts2) == blob
    dA = torch.from_numpy(A[:2000]).cuda()
    o1 = torch.empty((2000, 100), device="cuda")
    o2 = torch.empty((2000, 100), device="cuda")
    mdn.mdn_amm(model, luts, dA, o1)
    mdn.mdn_amm(model, luts2, dA, o2)
    assert torch.equal(o1, o2)


def test_state_errors(mdn):
    m1, _, A, B = _setup(mdn, "cls10_c32")
    m2, _, _, B2 = _setup(mdn, "cls10_c16")
    l2 = mdn.mdn_build_luts(m2, B2, 0)
    dA = torch.from_numpy(A[:10]).cuda()
    out = torch.empty((10, 10), device="cuda")
    with pytest.raises(mdn.MdnError) as e:
        mdn.mdn_amm(m1, l2, dA, out)
    assert e.value.status == -2          # C mismatch
    # cls100 and cls10_c32 were trained on the same A~ with the same C: identical
    # model bytes, identical fingerprint -> luts are interchangeable.
    m3, _, _, _ = _setup(mdn, "cls100")
    l1 = mdn.mdn_build_luts(m1, B, 0)
    assert mdn.mdn_amm(m3, l1, dA, out) is out
    with pytest.raises(mdn.MdnError):
        mdn.mdn_build_luts(m1, B, 1, 3)  # U not a power of two


def test_e2e_host_executor(mdn):
    model, om, A, B = _setup(mdn, "cls100")
    luts = mdn.mdn_build_luts(model, B, 0)
    want = O.amm(A, om, O.make_luts(om, B, "exact"))[2]
    ex = mdn.mdn_exec_create(model, luts, chunk_rows=1536, n_slots=3)
    A_h = torch.from_numpy(A).pin_memory()
    out_h = torch.empty((A.shape[0], 100)).pin_memory()
    mdn.mdn_amm_host(ex, A_h, out_h)
    _assert_out(out_h.numpy(), want)


@pytest.mark.parametrize("name,n_rows", [("cls100", 1 << 21), ("scale", 1 << 24)])
def test_bench_size_sampled_parity(mdn, name, n_rows):
    """Full bench-size A in HBM, launched exactly as bench.py does; 65536
    sampled rows (plus the last rows) checked against the oracle."""
    spec = CONFIGS[name]
    model, om, _, B = _setup(mdn, name)
    A = relu_lowrank_torch(relu_W(name), n_rows, 0, "cuda")
    rng = np.random.default_rng(123)
    rows = np.unique(np.concatenate([rng.integers(0, n_rows, 65536), np.arange(n_rows - 300, n_rows)]))
    for mode, mi in MODES:
        luts = mdn.mdn_build_luts(model, B, mi, spec.U)
        out = torch.empty((n_rows, spec.M), device="cuda")
        mdn.mdn_amm(model, luts, A, out)
        torch.cuda.synchronize()
        idx = torch.from_numpy(rows).cuda()
        As = A.index_select(0, idx).cpu().numpy()
        got = out.index_select(0, idx).cpu().numpy()
        _assert_out(got, O.amm(As, om, O.make_luts(om, B, mode, spec.U))[2])
        del out
    # the unfused halves at the same size, as bench.py --op encode / --op scan
    codes = torch.empty((n_rows, (spec.C + 1) // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode(model, A, codes)
    luts = mdn.mdn_build_luts(model, B, 0)
    out = torch.empty((n_rows, spec.M), device="cuda")
    mdn.mdn_scan(luts, codes, out=out)
    torch.cuda.synchronize()
    idx = torch.from_numpy(rows).cuda()
    codes_o, _, want = O.amm(A.index_select(0, idx).cpu().numpy(), om, O.make_luts(om, B, "exact"))
    assert (codes.index_select(0, idx).cpu().numpy() == O.pack_codes(codes_o)).all()
    _assert_out(out.index_select(0, idx).cpu().numpy(), want)
    del A, codes, out
    torch.cuda.empty_cache()


def test_row_chunking_subprocess():
    """Calls above 2^30 rows run as consecutive chunk launches; MDN_ROW_CHUNK
    shrinks the chunk so a 4099-row call crosses 4 chunk boundaries (run in a
    subprocess: the library reads the knob once)."""
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, oracle as O, paper_2106_10860_b200 as mdn
from datagen.synth import make_config_data
from helpers import model_bytes
for name, C, M, U in (("cls10_c16", 16, 10, 16), ("tiny", 4, 4, 4)):
    blob = model_bytes(name); om = O.read_model(blob)
    _, A, B = make_config_data(name, n_test=4099)
    A = A[:4099]
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, 1, U)
    codes_o, S_o, want = O.amm(A, om, O.make_luts(om, B, "avg", U))
    dA = torch.from_numpy(A).cuda()
    out = torch.empty((4099, M), device="cuda"); mdn.mdn_amm(model, luts, dA, out)
    codes = torch.empty((4099, (C + 1) // 2), dtype=torch.uint8, device="cuda"); mdn.mdn_encode(model, dA, codes)
    sums = torch.empty((4099, M), dtype=torch.int32, device="cuda"); mdn.mdn_scan(luts, codes, sums=sums)
    outc = torch.empty((4099, M), device="cuda"); mdn.mdn_amm_cm(model, luts, dA.t().contiguous(), outc)
    assert (out.cpu().numpy().view(np.uint32) == want.view(np.uint32)).all(), name
    assert (outc.cpu().numpy().view(np.uint32) == want.view(np.uint32)).all(), name
    assert (codes.cpu().numpy() == O.pack_codes(codes_o)).all(), name
    assert (sums.cpu().numpy() == S_o).all(), name
print("chunked ok")
'''
    import os
    env = dict(os.environ, MDN_ROW_CHUNK="1024")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env["PYTHONPATH"] = os.pathsep.join([root, os.path.join(root, "tests")])
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "chunked ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("mix", ["0", "3"])
def test_scan_pipe_mix_subprocess(mix):
    """mdn_scan's exact accumulate with every add on the ALU pipe (0) and with
    two in three words' adds as IMADs on the FMA pipe (3), forced for every C:
    sums and outputs bit-exact either way (the default picks per C)."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, oracle as O, paper_2106_10860_b200 as mdn
from datagen.synth import make_config_data
from helpers import model_bytes
for name, C, M in (("cls100", 32, 100), ("cls10_c16", 16, 10), ("scale", 32, 16), ("tiny", 4, 4)):
    blob = model_bytes(name); om = O.read_model(blob)
    _, A, B = make_config_data(name, n_test=3001)
    A = A[:3001]
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, 0)
    codes_o, S_o, want = O.amm(A, om, O.make_luts(om, B, "exact"))
    codes = torch.from_numpy(O.pack_codes(codes_o)).cuda()
    sums = torch.empty((3001, M), dtype=torch.int32, device="cuda")
    out = torch.empty((3001, M), device="cuda")
    mdn.mdn_scan(luts, codes, sums=sums, out=out)
    assert (sums.cpu().numpy() == S_o).all(), name
    assert (out.cpu().numpy().view(np.uint32) == want.view(np.uint32)).all(), name
print("mix ok")
'''
    env = dict(os.environ, MDN_SCAN_MIX=mix)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env["PYTHONPATH"] = os.pathsep.join([root, os.path.join(root, "tests")])
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and "mix ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("name", ["cls10_c16", "scale", "tiny"])
@pytest.mark.parametrize("layout", ["odd_ldo", "even_ldo", "misaligned"])
def test_scan_strided_out(mdn, name, layout):
    """mdn_scan's dequantised store with row stride ldo != M: 8-byte pair
    stores only when M and ldo are even and out is 8-byte aligned, scalar
    stores otherwise; nothing written outside the N x M window."""
    model, om, A, B = _setup(mdn, name)
    A = A[:2053]
    n = A.shape[0]                     # tiny's test split has 2048 rows
    spec = CONFIGS[name]
    M = spec.M
    luts = mdn.mdn_build_luts(model, B, 0)
    codes_o, _, want = O.amm(A, om, O.make_luts(om, B, "exact"))
    codes = torch.from_numpy(O.pack_codes(codes_o)).cuda()
    ldo = {"odd_ldo": M + 1, "even_ldo": M + 2, "misaligned": M + 2}[layout]
    off = 1 if layout == "misaligned" else 0
    raw = torch.full((n * ldo + 2,), float("nan"), device="cuda")
    out = raw[off:off + n * ldo].view(n, ldo)[:, :M]
    mdn.mdn_scan(luts, codes, out=out)
    _assert_out(out.cpu().numpy(), want)
    rest = raw.clone()
    rest[off:off + n * ldo].view(n, ldo)[:, :M] = 0
    assert torch.isnan(rest[rest != 0]).all()


@pytest.mark.parametrize("name,chunk", [("cls100", 1536), ("tiny", 1000), ("image", 4096)])
def test_host_encode_and_scan(mdn, name, chunk):
    """mdn_encode_host / mdn_scan_host: the unfused halves through the
    pipelined host-buffer executor, ragged last chunk, strided host rows."""
    model, om, A, B = _setup(mdn, name)
    A = A[:5003]
    N = A.shape[0]
    spec = CONFIGS[name]
    luts = mdn.mdn_build_luts(model, B, 0)
    codes_o, _, want = O.amm(A, om, O.make_luts(om, B, "exact"))
    ex = mdn.mdn_exec_create(model, luts, chunk_rows=chunk, n_slots=3)
    A_h = torch.zeros((N, spec.D + 4)).pin_memory()
    A_h[:, :spec.D] = torch.from_numpy(A)
    c_h = torch.empty((N, (spec.C + 1) // 2), dtype=torch.uint8).pin_memory()
    mdn.mdn_encode_host(ex, A_h[:, :spec.D], c_h)
    assert (c_h.numpy() == O.pack_codes(codes_o)).all()
    out_h = torch.full((N, spec.M + 1), float("nan")).pin_memory()
    mdn.mdn_scan_host(ex, torch.from_numpy(O.pack_codes(codes_o)), out_h[:, :spec.M])
    ex.close()
    _assert_out(out_h[:, :spec.M].numpy(), want)
    assert torch.isnan(out_h[:, spec.M:]).all()
