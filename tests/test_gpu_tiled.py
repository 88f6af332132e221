"""Table widths without a compiled kernel (M not in the BASELINE configs):
the tiled fused kernel (`ws_tma_tiled`: tables cut into 16-column tiles,
every row walks the tiles) and the tiled `mdn_scan` must equal the oracle bit
for bit -- codes, int32 sums and fp32 outputs, exact and averaging sums,
ragged N, ldo > M -- exactly like the compiled widths. (Tables too wide for
shared memory in tiles -- e.g. C = 64 with M = 257, 278 KB -- still run the
generic kernel; covered by test_gpu_shapes.)"""
import numpy as np
import pytest

import oracle as O
from datagen.synth import CONFIGS, make_config_data
from helpers import model_bytes
from test_gpu_parity import _assert_out

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mdn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as m
    return m


_rows = {}


def _A(name, n):
    if name not in _rows:
        _rows[name] = make_config_data(name, n_test=3000 if CONFIGS[name].kind == "relu" else 20_000,
                                       n_train=0)[1]
    return np.ascontiguousarray(_rows[name][:n])


CASES = [("cls100", 20), ("cls100", 64), ("cls100", 128), ("cls10_c16", 33), ("cls10_c16", 257),
         ("cls10_c64", 48), ("image", 12), ("tiny", 9)]


@pytest.mark.parametrize("name,M", CASES)
@pytest.mark.parametrize("mode", ["exact", "avg"])
def test_tiled_widths_bit_exact(mdn, name, M, mode):
    spec = CONFIGS[name]
    blob = model_bytes(name)
    om = O.read_model(blob)
    model = mdn.mdn_model_load(blob, 0)
    n = 2999
    A = _A(name, n)
    B = np.random.default_rng(M).standard_normal((spec.D, M)).astype(np.float32)
    U = spec.U
    luts = mdn.mdn_build_luts(model, B, 0 if mode == "exact" else 1, U)
    ol = O.make_luts(om, B, mode, U)
    codes, S, want = O.amm(A, om, ol)
    dA = torch.from_numpy(A).cuda()
    assert mdn.mdn_amm_variant(model, luts, spec.D) == "ws_tma_tiled"
    out = torch.empty((n, M), device="cuda")
    mdn.mdn_amm(model, luts, dA, out)
    _assert_out(out.cpu().numpy(), want)
    # ldo > M, unaligned row starts
    big = torch.zeros((n, M + 3), device="cuda")
    mdn.mdn_amm(model, luts, dA, big[:, :M])
    _assert_out(big[:, :M].cpu().numpy(), want)
    # the unfused halves: codes from mdn_encode, tiled mdn_scan (out and sums)
    pc = torch.empty((n, (om.C + 1) // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode(model, dA, pc)
    assert (pc.cpu().numpy() == O.pack_codes(codes)).all()
    sums = torch.empty((n, M), dtype=torch.int32, device="cuda")
    out2 = torch.empty((n, M), device="cuda")
    mdn.mdn_scan(luts, pc, sums=sums, out=out2)
    assert (sums.cpu().numpy() == S).all()              # U * block sums in avg mode
    _assert_out(out2.cpu().numpy(), want)
