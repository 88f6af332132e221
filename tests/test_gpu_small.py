"""GPU parity of the register-tree kernel (mdn_small.cu, k_amm_rt) beyond the
BASELINE configs: C in {4, 8} x M in {1..4} (16-bit-lane tables with W2 = 1, 2;
vector and scalar stores), exact and averaging sums, ragged N, strided A and
out, and the 8-bit path with and without byte-sized split values (q = 256
forces the integer select-tree variant). All bit-exact to the oracle."""
import numpy as np
import pytest

import oracle as O
from datagen.synth import _relu_rows, make_config_data
from helpers import model_bytes

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mdn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as m
    return m


_models = {}


def _model(C):
    if C not in _models:
        rng = np.random.default_rng([7, C])
        W = rng.standard_normal((8, 32))
        om = O.train(_relu_rows(rng, 3000, W), C)
        _models[C] = (om, O.write_model(om), _relu_rows(rng, 70_001, W))
    return _models[C]


def _bits(a):
    return np.asarray(a).view(np.uint32)


@pytest.mark.parametrize("C", [4, 8])
@pytest.mark.parametrize("M", [1, 2, 3, 4])
@pytest.mark.parametrize("mode", [("exact", 0), ("avg", 1)], ids=["exact", "avg"])
def test_rt_shapes(mdn, C, M, mode):
    om, blob, A = _model(C)
    B = np.random.default_rng([8, C, M]).standard_normal((32, M)).astype(np.float32)
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, mode[1], C)
    assert mdn.mdn_amm_variant(model, luts, 32).startswith("rt")
    want = O.amm(A, om, O.make_luts(om, B, mode[0], C))[2]
    out = torch.full((A.shape[0], M), float("nan"), device="cuda")
    mdn.mdn_amm(model, luts, torch.from_numpy(A).cuda(), out)
    assert (_bits(out.cpu().numpy()) == _bits(want)).all()


@pytest.mark.parametrize("N", [1, 31, 255, 256, 257, 4097])
def test_rt_ragged_strided(mdn, N):
    """lda = 36 (16-B aligned rows, TMA path), ldo = 7 (scalar stores)."""
    om, blob, A = _model(8)
    A = A[:N]
    B = np.random.default_rng(9).standard_normal((32, 2)).astype(np.float32)
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, 1, 8)
    want = O.amm(A, om, O.make_luts(om, B, "avg", 8))[2]
    big = torch.zeros((N, 36), device="cuda")
    big[:, :32] = torch.from_numpy(A).cuda()
    outbig = torch.full((N, 7), float("nan"), device="cuda")
    mdn.mdn_amm(model, luts, big[:, :32], outbig[:, :2])
    assert (_bits(outbig[:, :2].cpu().numpy()) == _bits(want)).all()
    assert torch.isnan(outbig[:, 2:]).all()              # nothing written past M


def _u8_data():
    _, A, B = make_config_data("image_u8", n_test=100_003, n_train=0)
    return A, B


@pytest.mark.parametrize("M", [1, 2, 4])
def test_u8_byte_thresholds_shapes(mdn, M):
    """The byte-threshold encoder (every q <= 255) with W2 = 1, 2 tables."""
    blob = model_bytes("image_u8")
    om = O.read_model(blob)
    A, _ = _u8_data()
    B = np.random.default_rng([10, M]).standard_normal((32, M)).astype(np.float32)
    model = mdn.mdn_model_load(blob, 0)
    for mode, mi in (("exact", 0), ("avg", 1)):
        luts = mdn.mdn_build_luts(model, B, mi, 8)
        want = O.amm_u8(A, om, O.make_luts(om, B, mode, 8))[2]
        out = torch.empty((A.shape[0], M), device="cuda")
        mdn.mdn_amm_u8(model, luts, torch.from_numpy(A).cuda(), out)
        assert (_bits(out.cpu().numpy()) == _bits(want)).all()


def test_u8_split_value_256_uses_integer_tree(mdn):
    """A split value above 255 (q = 256: no byte goes right) cannot be packed
    into a byte table; the model falls back to the integer select tree and
    must still match the oracle bit for bit, including rows at that node."""
    om = O.read_model(model_bytes("image_u8"))
    om.thr = om.thr.copy()
    om.thr[3, 0] = np.float32(300.0)       # level-0 split of codebook 3: every row goes left
    om.thr[5, 9] = np.float32(255.5)       # q = 256 at a level-3 node
    blob = O.write_model(om)
    A, B = _u8_data()
    model = mdn.mdn_model_load(blob, 0)
    for mode, mi in (("exact", 0), ("avg", 1)):
        luts = mdn.mdn_build_luts(model, B, mi, 8)
        codes_o, _, want = O.amm_u8(A, om, O.make_luts(om, B, mode, 8))
        assert (codes_o[:, 3] < 8).all()   # the node really sends everything left
        out = torch.empty((A.shape[0], 2), device="cuda")
        mdn.mdn_amm_u8(model, luts, torch.from_numpy(A).cuda(), out)
        assert (_bits(out.cpu().numpy()) == _bits(want)).all()


@pytest.mark.parametrize("name", ["tiny", "image", "image_u8"])
def test_bench_size_sampled_parity(mdn, name):
    """The register-tree kernels at the bench size, built exactly as bench.py
    builds them (tiny: 2^25 generated rows; image / image_u8: the 4M test
    patches tiled x8 = 32M rows); 65536 sampled rows + the tail vs the oracle."""
    import bench
    from datagen.synth import CONFIGS
    spec = CONFIGS[name]
    blob = model_bytes(name)
    om = O.read_model(blob)
    model = mdn.mdn_model_load(blob, 0)
    B = bench._config_B(name)
    A = bench._bench_rows(name, 0, 1, "cuda")
    n = A.shape[0]
    rng = np.random.default_rng(77)
    rows = np.unique(np.concatenate([rng.integers(0, n, 65536), np.arange(n - 300, n)]))
    idx = torch.from_numpy(rows).cuda()
    As = A.index_select(0, idx).cpu().numpy()
    u8 = A.dtype == torch.uint8
    for mode, mi in (("exact", 0), ("avg", 1)):
        luts = mdn.mdn_build_luts(model, B, mi, spec.U)
        out = torch.empty((n, spec.M), device="cuda")
        (mdn.mdn_amm_u8 if u8 else mdn.mdn_amm)(model, luts, A, out)
        torch.cuda.synchronize()
        got = out.index_select(0, idx).cpu().numpy()
        want = (O.amm_u8 if u8 else O.amm)(As, om, O.make_luts(om, B, mode, spec.U))[2]
        assert (_bits(got) == _bits(want)).all()
        del out
    # encode-only register-tree kernel + mdn_scan at the same size
    codes = torch.empty((n, spec.C // 2), dtype=torch.uint8, device="cuda")
    (mdn.mdn_encode_u8 if u8 else mdn.mdn_encode)(model, A, codes)
    luts = mdn.mdn_build_luts(model, B, 0)
    out = torch.empty((n, spec.M), device="cuda")
    mdn.mdn_scan(luts, codes, out=out)
    torch.cuda.synchronize()
    codes_o, _, want = (O.amm_u8 if u8 else O.amm)(As, om, O.make_luts(om, B, "exact"))
    assert (codes.index_select(0, idx).cpu().numpy() == O.pack_codes(codes_o)).all()
    assert (_bits(out.index_select(0, idx).cpu().numpy()) == _bits(want)).all()
    del A, codes, out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("C", [4, 8])
@pytest.mark.parametrize("N", [1, 31, 255, 257, 4097, 70_001])
def test_rt_encode_ragged(mdn, C, N):
    """Encode-only register-tree kernel (mdn_encode, C in {4, 8}, D = 32): packed
    codes bit-exact, strided A (lda = 36), nothing written past row N."""
    om, blob, A = _model(C)
    A = A[:N]
    model = mdn.mdn_model_load(blob, 0)
    big = torch.zeros((N, 36), device="cuda")
    big[:, :32] = torch.from_numpy(A).cuda()
    codes = torch.full((N + 3, C // 2), 0xAB, dtype=torch.uint8, device="cuda")
    mdn.mdn_encode(model, big[:, :32], codes[:N])
    got = codes.cpu().numpy()
    assert (got[:N] == O.pack_codes(O.encode(A, om))).all()
    assert (got[N:] == 0xAB).all()


@pytest.mark.parametrize("q256", [False, True], ids=["byte_tree", "int_tree"])
def test_rt_encode_u8(mdn, q256):
    """mdn_encode_u8 through the register-tree encoder: byte-threshold trees and
    (a split value of 256) the integer select tree."""
    om = O.read_model(model_bytes("image_u8"))
    if q256:
        om.thr = om.thr.copy()
        om.thr[5, 9] = np.float32(255.5)
    A, _ = _u8_data()
    model = mdn.mdn_model_load(O.write_model(om), 0)
    for n in (A.shape[0], 257, 1):
        codes = torch.empty((n, 4), dtype=torch.uint8, device="cuda")
        mdn.mdn_encode_u8(model, torch.from_numpy(A[:n]).cuda(), codes)
        assert (codes.cpu().numpy() == O.pack_codes(O.encode_u8(A[:n], om))).all()


def test_rt_encode_unaligned_codes_falls_back(mdn):
    """Codes at an odd byte offset (C = 8 wants 4-byte rows): the general
    encoder takes over and still matches."""
    om, blob, A = _model(8)
    A = A[:1000]
    model = mdn.mdn_model_load(blob, 0)
    raw = torch.zeros(1000 * 4 + 1, dtype=torch.uint8, device="cuda")
    codes = raw[1:].view(1000, 4)
    mdn.mdn_encode(model, torch.from_numpy(A).cuda(), codes)
    assert (codes.cpu().numpy() == O.pack_codes(O.encode(A, om))).all()
