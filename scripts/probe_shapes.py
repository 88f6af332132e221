"""Throughput of mdn_amm for table widths without a compiled fast kernel
(generic fallback) next to compiled ones, on the cls100 model (C = 32)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2106_10860_b200 as mdn
from datagen.synth import relu_W, relu_lowrank_torch
blob = open("artifacts/cls100.mdnm", "rb").read()
model = mdn.mdn_model_load(blob, 0)
A = relu_lowrank_torch(relu_W("cls100"), 1 << 20, 0, "cuda")
res = {}
for M in (10, 16, 20, 32, 48, 64, 100, 128):
    B = np.random.default_rng(M).standard_normal((512, M)).astype(np.float32)
    luts = mdn.mdn_build_luts(model, B, 0)
    out = torch.empty((A.shape[0], M), device="cuda")
    for _ in range(3): mdn.mdn_amm(model, luts, A, out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): mdn.mdn_amm(model, luts, A, out)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 / 1e3
    res[M] = {"variant": mdn.mdn_amm_variant(model, luts, 512), "rows_per_s": A.shape[0] / t,
              "gbs": A.shape[0] * (2048 + 4 * M) / t / 1e9}
    print(M, res[M], flush=True)
    # the unfused scan of the same tables
    codes = torch.empty((A.shape[0], 16), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode(model, A, codes)
    for _ in range(3): mdn.mdn_scan(luts, codes, out=out)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10): mdn.mdn_scan(luts, codes, out=out)
    e1.record(); torch.cuda.synchronize()
    res[M]["scan_rows_per_s"] = A.shape[0] / (e0.elapsed_time(e1) / 10 / 1e3)
    print(M, res[M], flush=True)
import os as _os
_os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/probe_shapes.json", "w"), indent=1)
