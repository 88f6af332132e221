"""GPU parity of the PQ comparator encoder (PAPER.md Eq. pqLoss
L182-184) against oracle/pq.py: every GPU code is a valid nearest prototype
under reading P1 (its fp64 distance within the fp32 rounding bound of the
minimum, so the first argmin wherever the margin exceeds the bound), near-ties
are rare, and the GPU's codes through mdn_scan are bit-exact to the oracle's
scan of the same codes."""
import os

import numpy as np
import pytest

import oracle as O
from datagen.synth import CONFIGS, make_config_data
from helpers import ARTIFACTS, model_bytes
from test_gpu_parity import MODES, _assert_out

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mdn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as m
    return m


_data = {}


def _setup(mdn, base, n=20_000):
    if not os.path.exists(os.path.join(ARTIFACTS, f"{base}_pq.mdnm")):
        pytest.skip(f"{base}_pq model not trained (scripts/make_models.py {base}_pq)")
    if base not in _data:
        _, A, B = make_config_data(base, n_test=n if base != "scale" else 4096)
        _data[base] = (A[:n], B)
    blob = model_bytes(f"{base}_pq")
    return mdn.mdn_model_load(blob, 0), O.read_model(blob), *_data[base]


PQ_CFGS = ["tiny", "cls10_c16", "cls100", "scale"]


def _check(A, om, packed):
    """Reading P1: valid codes, and the first fp64 argmin on all but a few
    near-tied rows."""
    got = O.unpack_codes(packed, om.C)
    ok, why = O.check_pq_codes(A, om, got)
    assert ok, why
    ref = O.encode_pq(A, om)
    assert (got != ref).mean() < 1e-3, why
    return got


@pytest.mark.parametrize("base", PQ_CFGS)
def test_encode_pq_valid(mdn, base):
    model, om, A, B = _setup(mdn, base)
    codes = torch.empty((A.shape[0], om.C // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, torch.from_numpy(A).cuda(), codes)
    _check(A, om, codes.cpu().numpy())


def test_encode_pq_margin_forces_argmin(mdn):
    """Rows built at a prototype plus a small offset (margin far above the
    rounding bound) must get exactly that prototype; rows exactly between two
    prototypes may get either, never a third."""
    model, om, A, B = _setup(mdn, "cls10_c16")
    rng = np.random.default_rng(5)
    n = 4096
    k = rng.integers(0, 16, (n, om.C))
    X = np.zeros((n, om.D), np.float32)
    for c, (b, e) in enumerate(om.sub):
        X[:, b:e] = om.P[16 * c + k[:, c], b:e] + 1e-3 * rng.standard_normal((n, e - b))
    codes = torch.empty((n, om.C // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, torch.from_numpy(X).cuda(), codes)
    got = O.unpack_codes(codes.cpu().numpy(), om.C)
    assert (got == k).all()
    # midpoints of prototypes 3 and 9 of every codebook
    M = np.zeros((64, om.D), np.float32)
    for c, (b, e) in enumerate(om.sub):
        M[:, b:e] = (om.P[16 * c + 3, b:e].astype(np.float64) + om.P[16 * c + 9, b:e]) / 2
    codes = torch.empty((64, om.C // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, torch.from_numpy(M).cuda(), codes)
    got = O.unpack_codes(codes.cpu().numpy(), om.C)
    assert O.check_pq_codes(M, om, got)[0]


@pytest.mark.parametrize("base", ["tiny", "cls100"])
@pytest.mark.parametrize("mode", MODES, ids=["exact", "avg"])
def test_pq_codes_through_scan(mdn, base, mode):
    model, om, A, B = _setup(mdn, base)
    spec = CONFIGS[base]
    luts = mdn.mdn_build_luts(model, B, mode[1], spec.U)
    codes = torch.empty((A.shape[0], om.C // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, torch.from_numpy(A).cuda(), codes)
    got = _check(A, om, codes.cpu().numpy())
    want = O.amm_pq(A, om, O.make_luts(om, B, mode[0], spec.U), codes=got)[2]
    out = torch.empty((A.shape[0], spec.M), device="cuda")
    mdn.mdn_scan(luts, codes, out=out)
    _assert_out(out.cpu().numpy(), want)


@pytest.mark.parametrize("N", [1, 7, 33, 1001])
def test_encode_pq_ragged_and_generic(mdn, N):
    """Ragged N on the fast kernel, and a 4-byte-offset A (generic kernel)."""
    model, om, A, B = _setup(mdn, "cls10_c16")
    A = np.ascontiguousarray(A[:N])
    codes = torch.empty((N, 8), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, torch.from_numpy(A).cuda(), codes)
    assert O.check_pq_codes(A, om, O.unpack_codes(codes.cpu().numpy(), om.C))[0]
    big = torch.zeros((N, 513), device="cuda")
    big[:, 1:] = torch.from_numpy(A).cuda()
    codes2 = torch.empty((N, 8), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, big[:, 1:], codes2)
    assert O.check_pq_codes(A, om, O.unpack_codes(codes2.cpu().numpy(), om.C))[0]


def test_pq_model_state_errors(mdn):
    model, om, A, B = _setup(mdn, "tiny")
    dA = torch.from_numpy(A[:64]).cuda()
    codes = torch.empty((64, 2), dtype=torch.uint8, device="cuda")
    with pytest.raises(mdn.MdnError) as e:
        mdn.mdn_encode(model, dA, codes)              # PQ model has no hash trees
    assert e.value.status == -5
    mdd = mdn.mdn_model_load(model_bytes("tiny"), 0)
    with pytest.raises(mdn.MdnError) as e:
        mdn.mdn_encode_pq(mdd, dA, codes)             # MADDNESS model is not a PQ model
    assert e.value.status == -5
    luts = mdn.mdn_build_luts(model, B, 0)
    out = torch.empty((64, 4), device="cuda")
    with pytest.raises(mdn.MdnError):
        mdn.mdn_amm(model, luts, dA, out)


@pytest.mark.parametrize("base", ["cls100", "tiny"])
def test_encode_pq_bench_size_sampled(mdn, base):
    """The PQ encoder at the bench size, on the rows bench.py --encoder pq
    generates (cls100: 2^21, tiny: 2^25); 65536 sampled rows + the tail vs the
    oracle: valid codes (reading P1)."""
    import bench
    model, om, _, _ = _setup(mdn, base)
    A = bench._bench_rows(base, 0, 1, "cuda")
    n = A.shape[0]
    codes = torch.empty((n, om.C // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, A, codes)
    torch.cuda.synchronize()
    rng = np.random.default_rng(99)
    rows = np.unique(np.concatenate([rng.integers(0, n, 65536), np.arange(n - 300, n)]))
    idx = torch.from_numpy(rows).cuda()
    _check(A.index_select(0, idx).cpu().numpy(), om, codes.index_select(0, idx).cpu().numpy())
    del A, codes
    torch.cuda.empty_cache()


@pytest.mark.parametrize("base", ["tiny", "cls100"])
def test_pq_host_executor(mdn, base):
    """mdn_encode_pq_host / mdn_amm_pq_host through a PQ executor (ragged last
    chunk, strided host rows) equal the oracle; the tree-based host calls
    refuse the PQ executor and the PQ calls a MADDNESS one (MDN_ESTATE)."""
    model, om, A, B = _setup(mdn, base)
    A = A[:3001]
    N, D = A.shape
    luts = mdn.mdn_build_luts(model, B, 1, CONFIGS[base].U)
    ex = mdn.mdn_exec_create(model, luts, chunk_rows=1000, n_slots=3)
    A_h = torch.zeros((N, D + 4)).pin_memory()
    A_h[:, :D] = torch.from_numpy(A)
    c_h = torch.empty((N, om.C // 2), dtype=torch.uint8).pin_memory()
    mdn.mdn_encode_pq_host(ex, A_h[:, :D], c_h)
    got = _check(A, om, c_h.numpy())
    want = O.amm_pq(A, om, O.make_luts(om, B, "avg", CONFIGS[base].U), codes=got)[2]
    out_h = torch.empty((N, B.shape[1])).pin_memory()
    mdn.mdn_amm_pq_host(ex, A_h[:, :D], out_h)
    _assert_out(out_h.numpy(), want)
    with pytest.raises(mdn.MdnError) as e:
        mdn.mdn_amm_host(ex, A_h[:, :D], torch.empty((N, B.shape[1])))
    assert e.value.status == -5
    ex.close()
    mdd = mdn.mdn_model_load(model_bytes(base), 0)
    ex2 = mdn.mdn_exec_create(mdd, mdn.mdn_build_luts(mdd, B, 0), chunk_rows=1000, n_slots=2)
    with pytest.raises(mdn.MdnError) as e:
        mdn.mdn_encode_pq_host(ex2, A_h[:, :D], c_h)
    assert e.value.status == -5
    ex2.close()
