"""GPU parity of the PQ comparator encoder (PAPER.md Eq. pqLoss
L182-184) against oracle/pq.py: codes bit-exact (the fp32 distance is
evaluated in the same order and rounding on both sides, reading P1), and the
PQ codes through mdn_scan bit-exact to the oracle's amm_pq."""
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


@pytest.mark.parametrize("base", PQ_CFGS)
def test_encode_pq_bit_exact(mdn, base):
    model, om, A, B = _setup(mdn, base)
    codes = torch.empty((A.shape[0], om.C // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, torch.from_numpy(A).cuda(), codes)
    want = O.pack_codes(O.encode_pq(A, om))
    got = codes.cpu().numpy()
    assert (got == want).all(), f"{(got != want).sum()} code bytes differ"


@pytest.mark.parametrize("base", ["tiny", "cls100"])
@pytest.mark.parametrize("mode", MODES, ids=["exact", "avg"])
def test_pq_codes_through_scan(mdn, base, mode):
    model, om, A, B = _setup(mdn, base)
    spec = CONFIGS[base]
    luts = mdn.mdn_build_luts(model, B, mode[1], spec.U)
    want = O.amm_pq(A, om, O.make_luts(om, B, mode[0], spec.U))[2]
    codes = torch.empty((A.shape[0], om.C // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, torch.from_numpy(A).cuda(), codes)
    out = torch.empty((A.shape[0], spec.M), device="cuda")
    mdn.mdn_scan(luts, codes, out=out)
    _assert_out(out.cpu().numpy(), want)


@pytest.mark.parametrize("N", [1, 7, 33, 1001])
def test_encode_pq_ragged_and_generic(mdn, N):
    """Ragged N on the fast kernel, and a 4-byte-offset A (generic kernel)."""
    model, om, A, B = _setup(mdn, "cls10_c16")
    A = np.ascontiguousarray(A[:N])
    want = O.pack_codes(O.encode_pq(A, om))
    codes = torch.empty((N, 8), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, torch.from_numpy(A).cuda(), codes)
    assert (codes.cpu().numpy() == want).all()
    big = torch.zeros((N, 513), device="cuda")
    big[:, 1:] = torch.from_numpy(A).cuda()
    codes2 = torch.empty((N, 8), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_pq(model, big[:, 1:], codes2)
    assert (codes2.cpu().numpy() == want).all()


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
    oracle, bit-exact codes."""
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
    got = codes.index_select(0, idx).cpu().numpy()
    want = O.pack_codes(O.encode_pq(A.index_select(0, idx).cpu().numpy(), om))
    assert (got == want).all(), f"{(got != want).sum()} code bytes differ"
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
    codes_o, _, want = O.amm_pq(A, om, O.make_luts(om, B, "avg", CONFIGS[base].U))
    ex = mdn.mdn_exec_create(model, luts, chunk_rows=1000, n_slots=3)
    A_h = torch.zeros((N, D + 4)).pin_memory()
    A_h[:, :D] = torch.from_numpy(A)
    c_h = torch.empty((N, om.C // 2), dtype=torch.uint8).pin_memory()
    mdn.mdn_encode_pq_host(ex, A_h[:, :D], c_h)
    assert (c_h.numpy() == O.pack_codes(codes_o)).all()
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
