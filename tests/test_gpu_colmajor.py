"""GPU parity of the column-major path:
mdn_encode_cm / mdn_amm_cm on At = A^T against the oracle's encode / amm on
the same A (the oracle's definition of g does not depend on the storage order).
Codes and fp32 outputs bit-exact."""
import numpy as np
import pytest

import oracle as O
from datagen.synth import CONFIGS, relu_W, relu_lowrank_torch
from test_gpu_parity import MODES, _assert_out, _setup

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mdn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as m
    return m


def _At(A, pad=0):
    """A^T on the device, D x N with row stride N + pad."""
    N, D = A.shape
    big = torch.zeros((D, N + pad), device="cuda")
    big[:, :N] = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    return big[:, :N]


CFGS = ["tiny", "cls10_c16", "cls10_c64", "cls100", "image", "scale"]


@pytest.mark.parametrize("name", CFGS)
def test_encode_cm_bit_exact(mdn, name):
    model, om, A, B = _setup(mdn, name)
    A = A[:50_000]
    codes = torch.empty((A.shape[0], (om.C + 1) // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_cm(model, _At(A), codes)
    want = O.pack_codes(O.encode(A, om))
    got = codes.cpu().numpy()
    assert (got == want).all(), f"{(got != want).sum()} code bytes differ"


@pytest.mark.parametrize("name", CFGS)
@pytest.mark.parametrize("mode", MODES, ids=["exact", "avg"])
def test_amm_cm_bit_exact(mdn, name, mode):
    model, om, A, B = _setup(mdn, name)
    A = A[:50_000]
    spec = CONFIGS[name]
    luts = mdn.mdn_build_luts(model, B, mode[1], spec.U)
    want = O.amm(A, om, O.make_luts(om, B, mode[0], spec.U))[2]
    out = torch.full((A.shape[0], spec.M), float("nan"), device="cuda")
    mdn.mdn_amm_cm(model, luts, _At(A), out)
    _assert_out(out.cpu().numpy(), want)


@pytest.mark.parametrize("N", [1, 31, 257, 4099])
def test_cm_ragged_strided(mdn, N):
    """Ragged N, ldt > N (padded columns), ldo > M (paired / scalar stores)."""
    model, om, A, B = _setup(mdn, "cls10_c32")
    luts = mdn.mdn_build_luts(model, B, 1, 16)
    A = A[:N]
    want = O.amm(A, om, O.make_luts(om, B, "avg", 16))[2]
    outbig = torch.zeros((N, 13), device="cuda")
    out = outbig[:, :10]
    mdn.mdn_amm_cm(model, luts, _At(A, pad=5), out)
    _assert_out(out.cpu().numpy(), want)
    codes = torch.empty((N, 16), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_cm(model, _At(A, pad=3), codes)
    assert (codes.cpu().numpy() == O.pack_codes(O.encode(A, om))).all()


def test_cm_errors(mdn):
    model, om, A, B = _setup(mdn, "tiny")
    luts = mdn.mdn_build_luts(model, B, 0)
    At = _At(A[:100])
    out = torch.empty((100, 4), device="cuda")
    with pytest.raises(ValueError):
        mdn.mdn_amm_cm(model, luts, At.t(), out)            # not D x N
    # ldt < N is refused by the library itself
    import paper_2106_10860_b200 as m
    st = m._lib.mdn_amm_cm(model._h, luts._h, At.data_ptr(), 100, 50, out.data_ptr(), 4, None)
    assert st == -1
    mdn.mdn_amm_cm(model, luts, At[:, :0], out[:0])           # N = 0 is a no-op


def test_cm_bench_size_sampled_parity(mdn):
    """cls100 at the bench size (2^21 rows, At 4 GiB) as bench.py --layout col
    launches it; 65536 sampled rows + the tail against the oracle."""
    name, n_rows = "cls100", 1 << 21
    spec = CONFIGS[name]
    model, om, _, B = _setup(mdn, name)
    A = relu_lowrank_torch(relu_W(name), n_rows, 0, "cuda")
    At = A.t().contiguous()
    rng = np.random.default_rng(321)
    rows = np.unique(np.concatenate([rng.integers(0, n_rows, 65536), np.arange(n_rows - 300, n_rows)]))
    idx = torch.from_numpy(rows).cuda()
    As = A.index_select(0, idx).cpu().numpy()
    del A
    for mode, mi in MODES:
        luts = mdn.mdn_build_luts(model, B, mi, spec.U)
        out = torch.empty((n_rows, spec.M), device="cuda")
        mdn.mdn_amm_cm(model, luts, At, out)
        torch.cuda.synchronize()
        got = out.index_select(0, idx).cpu().numpy()
        _assert_out(got, O.amm(As, om, O.make_luts(om, B, mode, spec.U))[2])
        del out
    del At
    torch.cuda.empty_cache()


def test_cm_slot_padding_and_repeated_dims(mdn):
    """The gather4 producer pads the split-column slots to a multiple of 4 with
    the last column: a model whose distinct split columns are not a multiple
    of 4 (repeated split dims, reading R3) must still match the oracle."""
    import copy
    from test_gpu_shapes import _model
    om0, _, A = _model(16, 64)
    om = copy.deepcopy(om0)                    # the cached model is shared with other tests
    om.dims[0] = om.dims[0, 0]                 # codebook 0: one dim at every level
    om.dims[1, 2] = om.dims[1, 0]
    n_cols = len(set(om.dims.reshape(-1).tolist()))
    if n_cols % 4 == 0:                        # make the count odd for certain
        om.dims[2, 3] = om.dims[2, 0]
        n_cols = len(set(om.dims.reshape(-1).tolist()))
    assert n_cols % 4 != 0
    blob = O.write_model(om)
    B = np.random.default_rng(5).standard_normal((64, 12)).astype(np.float32)
    model = mdn.mdn_model_load(blob, 0)
    for mode, mi in (("exact", 0), ("avg", 1)):
        luts = mdn.mdn_build_luts(model, B, mi, 16)
        codes_o, _, want = O.amm(A, om, O.make_luts(om, B, mode, 16))
        out = torch.full((A.shape[0], 12), float("nan"), device="cuda")
        mdn.mdn_amm_cm(model, luts, _At(A), out)
        _assert_out(out.cpu().numpy(), want)
    codes = torch.empty((A.shape[0], 8), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_cm(model, _At(A), codes)
    assert (codes.cpu().numpy() == O.pack_codes(codes_o)).all()


@pytest.mark.parametrize("name", ["tiny", "image"])
@pytest.mark.parametrize("N", [1, 3, 5, 1027, 70_001])
@pytest.mark.parametrize("pad", [0, 1, 2])
def test_cm_rows_per_thread(mdn, name, N, pad):
    """k_amm_cm with several consecutive rows per thread (vector loads of a
    split column): ragged N (N % 4 != 0 clamps the last group), and column
    strides ldt = N + pad that allow 4-, 2- or only 1-row vectors."""
    model, om, A, B = _setup(mdn, name)
    A = np.concatenate([A] * (1 + N // A.shape[0]))[:N] if N > A.shape[0] else A[:N]
    spec = CONFIGS[name]
    luts = mdn.mdn_build_luts(model, B, 0)
    codes_o, _, want = O.amm(A, om, O.make_luts(om, B, "exact"))
    out = torch.full((N, spec.M), float("nan"), device="cuda")
    mdn.mdn_amm_cm(model, luts, _At(A, pad=pad), out)
    _assert_out(out.cpu().numpy(), want)
    wide = torch.full((N, spec.M + 2), float("nan"), device="cuda")   # ldo != M: per-row stores
    mdn.mdn_amm_cm(model, luts, _At(A, pad=pad), wide[:, :spec.M])
    _assert_out(wide[:, :spec.M].cpu().numpy(), want)
    assert torch.isnan(wide[:, spec.M:]).all()
    codes = torch.empty((N, spec.C // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_cm(model, _At(A, pad=pad), codes)
    assert (codes.cpu().numpy() == O.pack_codes(codes_o)).all()


@pytest.mark.parametrize("name", ["tiny", "image"])
def test_cm_encode_unaligned_codes(mdn, name):
    """mdn_encode_cm into codes that are not 8-byte aligned (the grouped 8-byte
    code stores fall back to per-row stores)."""
    model, om, A, B = _setup(mdn, name)
    A = A[:4097]
    N, nb = A.shape[0], CONFIGS[name].C // 2
    raw = torch.zeros(N * nb + 8, dtype=torch.uint8, device="cuda")
    codes = raw[nb:nb + N * nb].view(N, nb)          # offset by one row of codes
    mdn.mdn_encode_cm(model, _At(A, pad=4), codes)
    assert (codes.cpu().numpy() == O.pack_codes(O.encode(A, om))).all()


@pytest.mark.parametrize("name,chunk", [("cls100", 1536), ("cls10_c16", 1001), ("tiny", 4096)])
def test_cm_host_executor(mdn, name, chunk):
    """mdn_amm_cm_host: column-major host A through the pipelined executor
    (only split columns cross PCIe), ragged last chunk, ldt > N, ldo > M,
    chunk sizes with and without 16-byte column alignment on the device."""
    model, om, A, B = _setup(mdn, name)
    A = A[:5003]
    N = A.shape[0]
    spec = CONFIGS[name]
    luts = mdn.mdn_build_luts(model, B, 1, spec.U)
    want = O.amm(A, om, O.make_luts(om, B, "avg", spec.U))[2]
    At_h = torch.zeros((spec.D, N + 7)).pin_memory()
    At_h[:, :N] = torch.from_numpy(np.ascontiguousarray(A.T))
    out_h = torch.full((N, spec.M + 3), float("nan")).pin_memory()
    ex = mdn.mdn_exec_create(model, luts, chunk_rows=chunk, n_slots=3)
    mdn.mdn_amm_cm_host(ex, At_h[:, :N], out_h[:, :spec.M])
    codes_h = torch.empty((N, (spec.C + 1) // 2), dtype=torch.uint8).pin_memory()
    mdn.mdn_encode_cm_host(ex, At_h[:, :N], codes_h)
    assert (codes_h.numpy() == O.pack_codes(O.encode(A, om))).all()
    ex.close()
    _assert_out(out_h[:, :spec.M].numpy(), want)
    assert torch.isnan(out_h[:, spec.M:]).all()
