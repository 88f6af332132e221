#!/usr/bin/env python
"""Small, ragged invocations of every hot-path kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py

(One tool per run: see the profiling recipe.) Covers the general TMA kernel,
the register-tree kernel (fp32 and 8-bit), the column-major kernels, the PQ
encoder, the unfused encode / scan, the generic fallbacks and GPU training,
each checked against the oracle so a silent corruption also fails.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import paper_2106_10860_b200 as mdn  # noqa: E402
from datagen.synth import CONFIGS, make_config_data  # noqa: E402

BAD = []


def _check(tag, got, want):
    if not (np.asarray(got).view(np.uint32) == np.asarray(want).view(np.uint32)).all():
        print("MISMATCH", tag)
        BAD.append(tag)


def _blob(name):
    return open(os.path.join(ROOT, "artifacts", f"{name}.mdnm"), "rb").read()


def main():
    for name, n in (("tiny", 1000), ("image", 999), ("cls100", 777), ("cls10_c64", 301),
                    ("scale", 513)):
        spec = CONFIGS[name]
        blob = _blob(name)
        om = O.read_model(blob)
        _, A, B = make_config_data(name, n_test=n, n_train=0 if name == "image" else None)
        A = A[:n]
        model = mdn.mdn_model_load(blob, 0)
        dA = torch.from_numpy(A).cuda()
        At = dA.t().contiguous()
        for mode_name, mode in (("exact", 0), ("avg", 1)):
            luts = mdn.mdn_build_luts(model, B, mode, spec.U)
            want = O.amm(A, om, O.make_luts(om, B, mode_name, spec.U))[2]
            out = torch.empty((n, spec.M), device="cuda")
            mdn.mdn_amm(model, luts, dA, out)
            codes = torch.empty((n, (spec.C + 1) // 2), dtype=torch.uint8, device="cuda")
            mdn.mdn_encode(model, dA, codes)
            sums = torch.empty((n, spec.M), dtype=torch.int32, device="cuda")
            out2 = torch.empty((n, spec.M), device="cuda")
            mdn.mdn_scan(luts, codes, sums=sums, out=out2)
            out3 = torch.empty((n, spec.M), device="cuda")
            mdn.mdn_amm_cm(model, luts, At, out3)
            # generic fallback: 4-byte-offset A
            big = torch.zeros((n, spec.D + 1), device="cuda")
            big[:, 1:] = dA
            out4 = torch.empty((n, spec.M), device="cuda")
            mdn.mdn_amm(model, luts, big[:, 1:], out4)
            torch.cuda.synchronize()
            for tag, t in (("amm", out), ("scan", out2), ("amm_cm", out3), ("generic", out4)):
                _check(f"{name} {mode_name} {tag}", t.cpu().numpy(), want)
    # 8-bit rows (register-tree byte-threshold kernel)
    blob = _blob("image_u8")
    om = O.read_model(blob)
    _, A, B = make_config_data("image_u8", n_test=1001, n_train=0)
    model = mdn.mdn_model_load(blob, 0)
    for mode_name, mode in (("exact", 0), ("avg", 1)):
        luts = mdn.mdn_build_luts(model, B, mode, 8)
        out = torch.empty((A.shape[0], 2), device="cuda")
        mdn.mdn_amm_u8(model, luts, torch.from_numpy(A).cuda(), out)
        torch.cuda.synchronize()
        _check(f"image_u8 {mode_name}", out.cpu().numpy(),
               O.amm_u8(A, om, O.make_luts(om, B, mode_name, 8))[2])
    # PQ encoder
    pblob = os.path.join(ROOT, "artifacts", "cls10_c16_pq.mdnm")
    if os.path.exists(pblob):
        blob = open(pblob, "rb").read()
        om = O.read_model(blob)
        _, A, _ = make_config_data("cls10_c16", n_test=333)
        model = mdn.mdn_model_load(blob, 0)
        codes = torch.empty((333, 8), dtype=torch.uint8, device="cuda")
        mdn.mdn_encode_pq(model, torch.from_numpy(A).cuda(), codes)
        torch.cuda.synchronize()
        if not O.check_pq_codes(A, om, O.unpack_codes(codes.cpu().numpy(), om.C))[0]:
            print("MISMATCH pq")
            BAD.append("pq")
    # GPU training (small)
    A = make_config_data("tiny", n_test=0, n_train=4096)[0]
    trained = O.read_model(mdn.mdn_train(torch.from_numpy(A).cuda(), 4, 1.0))
    if trained.C != 4:
        BAD.append("train")
    print("sanitize_run done, mismatches:", len(BAD), BAD)
    return 1 if BAD else 0


if __name__ == "__main__":
    sys.exit(main())
