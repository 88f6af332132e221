"""k_u8_rows (lane = row for the 8-bit byte trees and the scan, mdn_small.cu)
is the default kernel of mdn_amm_u8 / mdn_encode_u8 for 8-bit rows whose 8
codebooks are the row's 4-byte words (App. B; image_u8). The
k_amm_rt byte-tree kernel it replaced stays reachable with MDN_U8_ROWS=0
(read once per process): both must equal the oracle bit for bit."""
import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
import torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import oracle as O
import paper_2106_10860_b200 as mdn
from helpers import model_bytes
from datagen.synth import make_config_data
blob = model_bytes("image_u8")
om = O.read_model(blob)
_, A, B = make_config_data("image_u8", n_test=70_001, n_train=0)
model = mdn.mdn_model_load(blob, 0)
bad = 0
for n in (70_001, 4_097, 255, 1):
    dA = torch.from_numpy(A[:n]).cuda()
    codes = torch.empty((n, 4), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_u8(model, dA, codes)
    want_codes = O.encode_u8(A[:n], om)
    bad += int((codes.cpu().numpy() != O.pack_codes(want_codes)).any())
    for mode, mi in (("exact", 0), ("avg", 1)):
        for M in (1, 2, 3, 4):
            Bm = np.random.default_rng([11, M]).standard_normal((32, M)).astype(np.float32)
            luts = mdn.mdn_build_luts(model, Bm, mi, 8)
            want = O.amm_u8(A[:n], om, O.make_luts(om, Bm, mode, 8))[2]
            out = torch.empty((n, M), device="cuda")
            mdn.mdn_amm_u8(model, luts, dA, out)
            bad += int((out.cpu().numpy().view(np.uint32) != want.view(np.uint32)).any())
print("BAD", bad)
"""


@pytest.mark.parametrize("rows_kernel", ["1", "0"], ids=["k_u8_rows", "k_amm_rt"])
def test_u8_kernels_match_oracle(rows_kernel):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, MDN_U8_ROWS=rows_kernel)
    p = subprocess.run([sys.executable, "-c", SCRIPT, ROOT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    assert "BAD 0" in p.stdout, p.stdout[-2000:]
