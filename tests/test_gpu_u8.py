"""GPU parity of the 8-bit input path (App. B,
L839) against the oracle's encode_u8 / amm_u8, bit-exact."""
import os

import numpy as np
import pytest

import oracle as O
from datagen.synth import CONFIGS, make_config_data
from helpers import ARTIFACTS, model_bytes

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mdn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as m
    return m


_data = {}


def _u8_setup(name):
    if name not in _data:
        if name == "image_u8":
            _, A, B = make_config_data("image_u8", n_test=300_000, n_train=0)
        else:  # fp32-trained model applied to byte data (exercises other subspace widths)
            spec = CONFIGS[name]
            rng = np.random.default_rng([7, spec.D])
            A = np.clip(np.rint(127.5 + 50 * rng.standard_normal((20011, spec.D))), 0, 255).astype(np.uint8)
            B = rng.standard_normal((spec.D, spec.M)).astype(np.float32)
        _data[name] = (A, B)
    return _data[name]


U8_CFGS = ["image_u8", "tiny", "cls10_c16", "scale"]


@pytest.mark.parametrize("name", U8_CFGS)
@pytest.mark.parametrize("mode", [("exact", 0), ("avg", 1)], ids=["exact", "avg"])
def test_u8_parity(mdn, name, mode):
    if name == "image_u8" and not os.path.exists(os.path.join(ARTIFACTS, "image_u8.mdnm")):
        pytest.skip("image_u8 model not trained")
    spec = CONFIGS[name]
    blob = model_bytes(name)
    om = O.read_model(blob)
    A, B = _u8_setup(name)
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, mode[1], spec.U)
    codes_o, S_o, out_o = O.amm_u8(A, om, O.make_luts(om, B, mode[0], spec.U))
    assert (codes_o == O.encode(A.astype(np.float32), om)).all()     # App. B reading R11
    dA = torch.from_numpy(A).cuda()
    codes = torch.empty((A.shape[0], (spec.C + 1) // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_u8(model, dA, codes)
    assert (codes.cpu().numpy() == O.pack_codes(codes_o)).all()
    out = torch.empty((A.shape[0], spec.M), device="cuda")
    mdn.mdn_amm_u8(model, luts, dA, out)
    assert (out.cpu().numpy().view(np.uint32) == out_o.view(np.uint32)).all()


def test_u8_generic_fallback_and_ragged(mdn):
    """A byte offset of 1 (no TMA: generic kernel) and ragged N give the same bytes."""
    blob = model_bytes("tiny")
    om = O.read_model(blob)
    A, B = _u8_setup("tiny")
    A = A[:3333]
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, 0)
    want = O.amm_u8(A, om, O.make_luts(om, B, "exact"))[2]
    big = torch.zeros((A.shape[0], 33), dtype=torch.uint8, device="cuda")
    big[:, 1:] = torch.from_numpy(A).cuda()
    for view in (big[:, 1:], torch.from_numpy(np.ascontiguousarray(A)).cuda()):
        out = torch.empty((A.shape[0], 4), device="cuda")
        mdn.mdn_amm_u8(model, luts, view, out)
        assert (out.cpu().numpy().view(np.uint32) == want.view(np.uint32)).all()


def test_u8_host_executor(mdn):
    """mdn_amm_host_u8: pinned host 8-bit rows through the pipelined executor
    (chunks smaller than N, so several slots cycle) equal the oracle."""
    blob = model_bytes("image_u8")
    om = O.read_model(blob)
    _, A, B = make_config_data("image_u8", n_test=50_001, n_train=0)
    model = mdn.mdn_model_load(blob, 0)
    luts = mdn.mdn_build_luts(model, B, 1, 8)
    want = O.amm_u8(A, om, O.make_luts(om, B, "avg", 8))[2]
    ex = mdn.mdn_exec_create(model, luts, chunk_rows=4096, n_slots=3)
    A_h = torch.from_numpy(A).pin_memory()
    out_h = torch.empty((A.shape[0], 2)).pin_memory()
    mdn.mdn_amm_host_u8(ex, A_h, out_h)
    assert (out_h.numpy().view(np.uint32) == want.view(np.uint32)).all()
    codes_h = torch.empty((A.shape[0], 4), dtype=torch.uint8).pin_memory()
    mdn.mdn_encode_host_u8(ex, A_h, codes_h)                     # g on host 8-bit rows
    assert (codes_h.numpy() == O.pack_codes(O.encode_u8(A, om))).all()
