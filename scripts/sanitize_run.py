#!/usr/bin/env python
"""Small, ragged invocations of every hot-path kernel, for compute-sanitizer.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
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


def main():
    bad = 0
    for name, n in (("tiny", 1000), ("cls100", 777), ("cls10_c64", 301), ("scale", 513)):
        spec = CONFIGS[name]
        blob = open(os.path.join(ROOT, "artifacts", f"{name}.mdnm"), "rb").read()
        om = O.read_model(blob)
        _, A, B = make_config_data(name, n_test=n)
        model = mdn.mdn_model_load(blob, 0)
        dA = torch.from_numpy(A).cuda()
        for mode_name, mode in (("exact", 0), ("avg", 1)):
            luts = mdn.mdn_build_luts(model, B, mode, spec.U)
            out = torch.empty((n, spec.M), device="cuda")
            mdn.mdn_amm(model, luts, dA, out)
            codes = torch.empty((n, (spec.C + 1) // 2), dtype=torch.uint8, device="cuda")
            mdn.mdn_encode(model, dA, codes)
            sums = torch.empty((n, spec.M), dtype=torch.int32, device="cuda")
            out2 = torch.empty((n, spec.M), device="cuda")
            mdn.mdn_scan(luts, codes, sums=sums, out=out2)
            torch.cuda.synchronize()
            want = O.amm(A, om, O.make_luts(om, B, mode_name, spec.U))[2]
            for t in (out, out2):
                if not (t.cpu().numpy().view(np.uint32) == want.view(np.uint32)).all():
                    print("MISMATCH", name, mode_name)
                    bad += 1
    print("sanitize_run done, mismatches:", bad)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
