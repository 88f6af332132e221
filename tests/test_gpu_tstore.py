"""GPU parity of the wide-table output paths that leave by TMA tensor stores
(`k_scan_ts` for mdn_scan, the column-major fused kernel's scanner parts):
ragged N around the 32-row boxes and the 512-row blocks, row pitch ldo > M
with 16-B-aligned rows (the only layout that takes the TMA path), and an out
base 16-B but not 128-B aligned. Outputs bit-exact to the oracle (Eq. 2 /
App. D on the same codes), nothing written outside the N x M window (the
tensor map clips rows >= N and columns >= M), and int32 sums written
alongside the TMA-stored outputs bit-exact too."""
import numpy as np
import pytest

import oracle as O
from datagen.synth import CONFIGS
from test_gpu_colmajor import _At
from test_gpu_parity import MODES, _assert_out, _setup

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mdn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as m
    return m


def _padded_out(n, M, ldo, off):
    """out = an n x M view of a NaN buffer with row pitch ldo, base shifted
    by off floats; returns (raw buffer, view)."""
    raw = torch.full((n * ldo + off + 8,), float("nan"), device="cuda")
    return raw, raw[off:off + n * ldo].view(n, ldo)[:, :M]


def _assert_untouched(raw, n, M, ldo, off):
    rest = raw.clone()
    rest[off:off + n * ldo].view(n, ldo)[:, :M] = 0
    assert torch.isnan(rest[rest != 0]).all(), "a store landed outside the N x M window"


@pytest.mark.parametrize("mode", MODES, ids=["exact", "avg"])
@pytest.mark.parametrize("N", [1, 31, 33, 511, 1000, 8209])
@pytest.mark.parametrize("ldo_pad,off", [(0, 0), (4, 0), (28, 4)])
def test_scan_tstore(mdn, mode, N, ldo_pad, off):
    model, om, A, B = _setup(mdn, "cls100")
    A = A[:N]
    M = CONFIGS["cls100"].M
    luts = mdn.mdn_build_luts(model, B, mode[1], CONFIGS["cls100"].U)
    codes_o, S_o, want = O.amm(A, om, O.make_luts(om, B, mode[0], CONFIGS["cls100"].U))
    codes = torch.from_numpy(O.pack_codes(codes_o)).cuda()
    ldo = M + ldo_pad
    raw, out = _padded_out(N, M, ldo, off)
    sums = torch.empty((N, M), dtype=torch.int32, device="cuda") if mode[1] == 0 else None
    mdn.mdn_scan(luts, codes, sums=sums, out=out)
    torch.cuda.synchronize()
    _assert_out(out.cpu().numpy(), want)
    _assert_untouched(raw, N, M, ldo, off)
    if sums is not None:
        assert (sums.cpu().numpy() == S_o).all()


@pytest.mark.parametrize("mode", MODES, ids=["exact", "avg"])
@pytest.mark.parametrize("N", [1, 31, 4099])
@pytest.mark.parametrize("ldo_pad,off", [(0, 0), (8, 4)])
def test_cm_tstore(mdn, mode, N, ldo_pad, off):
    model, om, A, B = _setup(mdn, "cls100")
    A = A[:N]
    M = CONFIGS["cls100"].M
    luts = mdn.mdn_build_luts(model, B, mode[1], CONFIGS["cls100"].U)
    want = O.amm(A, om, O.make_luts(om, B, mode[0], CONFIGS["cls100"].U))[2]
    ldo = M + ldo_pad
    raw, out = _padded_out(N, M, ldo, off)
    mdn.mdn_amm_cm(model, luts, _At(A, pad=4), out)
    torch.cuda.synchronize()
    _assert_out(out.cpu().numpy(), want)
    _assert_untouched(raw, N, M, ldo, off)


def test_scan_tstore_back_to_back(mdn):
    """Two scans into the same buffer on one stream: the second launch's
    outputs replace the first's (the bulk stores of a launch are complete
    when it ends)."""
    model, om, A, B = _setup(mdn, "cls100")
    A = A[:5000]
    luts0 = mdn.mdn_build_luts(model, B, 0)
    luts1 = mdn.mdn_build_luts(model, -B, 0)
    codes_o = O.encode(A, om)
    codes = torch.from_numpy(O.pack_codes(codes_o)).cuda()
    out = torch.empty((A.shape[0], CONFIGS["cls100"].M), device="cuda")
    mdn.mdn_scan(luts0, codes, out=out)
    mdn.mdn_scan(luts1, codes, out=out)
    torch.cuda.synchronize()
    want = O.amm(A, om, O.make_luts(om, -B, "exact"))[2]
    _assert_out(out.cpu().numpy(), want)
