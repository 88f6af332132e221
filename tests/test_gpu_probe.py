"""mdn_amm_probe (diagnostic): the fused kernel's pipeline with encode and scan
removed writes beta32 to every output of every row (ragged N too), refuses
shapes the general pipeline does not serve, and checks arguments like
mdn_amm."""
import numpy as np
import pytest

from helpers import model_bytes

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mdn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as m
    return m


@pytest.mark.parametrize("name,D,M", [("cls100", 512, 100), ("cls10_c16", 512, 10), ("scale", 256, 16)])
@pytest.mark.parametrize("N", [1, 255, 4099, 70001])
def test_probe_writes_beta_everywhere(mdn, name, D, M, N):
    model = mdn.mdn_model_load(model_bytes(name), 0)
    B = np.random.default_rng(0).standard_normal((D, M)).astype(np.float32)
    luts = mdn.mdn_build_luts(model, B, 0)
    A = torch.randn((N, D), device="cuda")
    out = torch.full((N, M), float("nan"), device="cuda")
    mdn.mdn_amm_probe(model, luts, A, out)
    o = out.cpu().numpy()
    assert np.isfinite(o).all()
    assert (o.view(np.uint32) == np.float32(luts.beta32).view(np.uint32)).all()


def test_probe_refuses_register_tree_shapes(mdn):
    model = mdn.mdn_model_load(model_bytes("tiny"), 0)
    B = np.random.default_rng(0).standard_normal((32, 4)).astype(np.float32)
    luts = mdn.mdn_build_luts(model, B, 0)
    A = torch.randn((1000, 32), device="cuda")
    out = torch.empty((1000, 4), device="cuda")
    with pytest.raises(mdn.MdnError) as e:
        mdn.mdn_amm_probe(model, luts, A, out)
    assert e.value.status == -1
