"""Stage geometry of the TMA pipeline (`k_amm_ws`): the rows per stage R and
the ring depth are chosen at run time from the shared-memory budget
(`plan()`), so the default build runs R = 16 (cls100), 32
(cls10) and 64 (scale). The A/B knobs MDN_WS_MINNS / MDN_WS_RMAX force other
geometries (R = 8 ... 128, 2 ... 16 stages); the fused and the encode-only
kernels must stay bit-identical to the oracle under every one of them, on a
ragged row count (tails inside a stage and inside a tile). The knobs are read
once per process, so each geometry runs in a child process."""
import json
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tests")
import oracle as O
import paper_2106_10860_b200 as mdn
from datagen.synth import CONFIGS, make_config_data
from helpers import model_bytes
res = {}
for name in ("cls100", "cls10_c32", "scale"):
    spec = CONFIGS[name]
    blob = model_bytes(name)
    om = O.read_model(blob)
    model = mdn.mdn_model_load(blob, 0)
    _, A, B = make_config_data(name, n_test=2000, n_train=0)
    A = np.ascontiguousarray(np.concatenate([A, A[:1003][::-1]]))       # 3003 rows: ragged
    dA = torch.from_numpy(A).cuda()
    for mode, mc in (("exact", mdn.MDN_SUM_EXACT), ("avg", mdn.MDN_SUM_AVG)):
        luts = mdn.mdn_build_luts(model, B, mc, spec.U)
        out = torch.empty((A.shape[0], spec.M), device="cuda")
        mdn.mdn_amm(model, luts, dA, out)
        torch.cuda.synchronize()
        want_codes, _, want = O.amm(A, om, O.make_luts(om, B, mode, spec.U))
        got = out.cpu().numpy()
        res[f"{name}_{mode}"] = int((got.view(np.uint32) != want.view(np.uint32)).any(axis=1).sum())
    codes = torch.empty((A.shape[0], (spec.C + 1) // 2), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode(model, dA, codes)
    torch.cuda.synchronize()
    res[f"{name}_encode"] = int((codes.cpu().numpy() != O.pack_codes(want_codes)).any(axis=1).sum())
    res[f"{name}_variant"] = mdn.mdn_amm_variant(model, luts, spec.D)
print(json.dumps(res))
"""


@pytest.mark.parametrize("knobs", [{"MDN_WS_MINNS": "2"}, {"MDN_WS_MINNS": "4"},
                                   {"MDN_WS_RMAX": "16"}, {"MDN_WS_RMAX": "8"}],
                         ids=["minns2", "minns4", "rmax16", "rmax8"])
def test_stage_geometry_bit_exact(knobs):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, **knobs)
    p = subprocess.run([sys.executable, "-c", f"ROOT = {ROOT!r}\n" + CHILD], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    res = json.loads(p.stdout.strip().splitlines()[-1])
    bad = {k: v for k, v in res.items() if not k.endswith("_variant") and v != 0}
    assert not bad, f"rows differing from the oracle under {knobs}: {bad} ({res})"
    assert all(res[f"{n}_variant"].startswith("ws") for n in ("cls100", "cls10_c32", "scale")), res
