"""GPU parity over shapes the BASELINE configs do not reach: odd C, D not a
multiple of 4 (generic encode), C up to MAX_C = 256, M from 1 to 1000 (W up
to 250: generic scan, tables beyond shared memory),
every averaging block U, non-contiguous outputs. Models are trained on the fly
by the oracle on small relu low-rank data."""
import numpy as np
import pytest

import oracle as O
from datagen.synth import _relu_rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mdn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as m
    return m


_models = {}


def _model(C, D, seed=0):
    key = (C, D, seed)
    if key not in _models:
        rng = np.random.default_rng([seed, C, D])
        W = rng.standard_normal((min(8, D), D))
        Atr = _relu_rows(rng, 1500, W)
        Ate = _relu_rows(rng, 1777, W)        # ragged: not a multiple of any tile
        om = O.train(Atr, C)
        _models[key] = (om, O.write_model(om), Ate)
    return _models[key]


def _check(got, want):
    assert (np.asarray(got).view(np.uint32) == want.view(np.uint32)).all()


SHAPES = [  # (C, D, M)
    (1, 8, 3), (2, 8, 1), (3, 10, 7), (6, 30, 5), (12, 48, 33), (4, 32, 300),
    (16, 64, 10), (8, 32, 2), (32, 128, 16), (128, 256, 4), (64, 512, 12),
    (256, 256, 5),      # MAX_C codebooks of one dim each (S <= 255 C < 2^16)
    (8, 32, 1000),      # M = 1000: 250 table words per code, tables beyond shared memory
]


@pytest.mark.parametrize("C,D,M", SHAPES)
def test_exact_shapes(mdn, C, D, M):
    om, blob, A = _model(C, D)
    B = np.random.default_rng([1, C, D, M]).standard_normal((D, M)).astype(np.float32)
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, 0)
    codes_o, S_o, out_o = O.amm(A, om, O.make_luts(om, B, "exact"))
    dA = torch.from_numpy(A).cuda()
    codes = torch.empty((A.shape[0], (C + 1) // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode(model, dA, codes)
    assert (codes.cpu().numpy() == O.pack_codes(codes_o)).all()
    sums = torch.empty((A.shape[0], M), dtype=torch.int32, device="cuda")
    mdn.mdn_scan(luts, codes, sums=sums)
    assert (sums.cpu().numpy() == S_o).all()
    out = torch.empty((A.shape[0], M), device="cuda")
    mdn.mdn_amm(model, luts, dA, out)
    _check(out.cpu().numpy(), out_o)


@pytest.mark.parametrize("U", [1, 2, 4, 8, 16, 32])
def test_avg_every_U(mdn, U):
    C, D, M = 32, 128, 16
    om, blob, A = _model(C, D)
    B = np.random.default_rng([2, U]).standard_normal((D, M)).astype(np.float32)
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, 1, U)
    oluts = O.make_luts(om, B, "avg", U)
    codes_o, S_o, out_o = O.amm(A, om, oluts)
    out = torch.empty((A.shape[0], M), device="cuda")
    mdn.mdn_amm(model, luts, torch.from_numpy(A).cuda(), out)
    _check(out.cpu().numpy(), out_o)
    sums = torch.empty((A.shape[0], M), dtype=torch.int32, device="cuda")
    codes = torch.from_numpy(O.pack_codes(codes_o)).cuda()
    mdn.mdn_scan(luts, codes, sums=sums)
    assert (sums.cpu().numpy() == S_o).all()


def test_fast_and_generic_paths_agree(mdn):
    """The same inputs through the TMA kernel (aligned) and the generic kernel
    (A offset by one float) give identical bytes."""
    om, blob, A = _model(16, 64)
    B = np.random.default_rng(3).standard_normal((64, 16)).astype(np.float32)
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, 1, 16)
    dA = torch.from_numpy(A).cuda()
    big = torch.zeros((A.shape[0], 65), device="cuda")
    big[:, 1:] = dA
    o1 = torch.empty((A.shape[0], 16), device="cuda")
    o2 = torch.empty((A.shape[0], 16), device="cuda")
    mdn.mdn_amm(model, luts, dA, o1)
    mdn.mdn_amm(model, luts, big[:, 1:], o2)
    assert mdn.mdn_amm_variant(model, luts, 64).startswith("ws_tma")
    assert torch.equal(o1, o2)


def test_constant_and_degenerate_tables(mdn):
    """B = 0 -> all tables equal per codebook -> l = 0, Tq = 0, out = sum_c delta_c = 0."""
    om, blob, A = _model(8, 32)
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, np.zeros((32, 4), np.float32), 0)
    assert luts.l == 0 and luts.alpha == 1.0 and luts.beta32 == 0.0
    out = torch.full((A.shape[0], 4), 7.0, device="cuda")
    mdn.mdn_amm(model, luts, torch.from_numpy(A).cuda(), out)
    assert torch.count_nonzero(out) == 0


def test_concurrent_streams(mdn):
    """Handles are immutable: the same model/luts on two streams at once."""
    om, blob, A = _model(32, 128)
    B = np.random.default_rng(4).standard_normal((128, 16)).astype(np.float32)
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, 0)
    want = O.amm(A, om, O.make_luts(om, B, "exact"))[2]
    dA = torch.from_numpy(A).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1 = torch.empty((A.shape[0], 16), device="cuda")
    o2 = torch.empty((A.shape[0], 16), device="cuda")
    torch.cuda.synchronize()
    for _ in range(5):
        mdn.mdn_amm(model, luts, dA, o1, stream=s1)
        mdn.mdn_amm(model, luts, dA, o2, stream=s2)
    torch.cuda.synchronize()
    _check(o1.cpu().numpy(), want)
    _check(o2.cpu().numpy(), want)
