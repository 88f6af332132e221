#!/usr/bin/env python
"""Train every config's model with the ORACLE and write artifacts/<config>.mdnm.

This committed script is the only writer of the model files both paths
consume (north_star: "the oracle ... serializes the model that both paths
consume"). It calls only ``oracle/`` and ``datagen/``.

Usage: python scripts/make_models.py [config ...]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from datagen.synth import CONFIGS, make_config_data  # noqa: E402

OUT = os.path.join(ROOT, "artifacts")


PQ_MODELS = ("tiny", "cls10_c16", "cls100", "scale")   # <name>_pq.mdnm


def main(names):
    os.makedirs(OUT, exist_ok=True)
    man_path = os.path.join(OUT, "manifest.json")
    manifest = json.load(open(man_path)) if os.path.exists(man_path) else {}
    for name in names:
        if name.endswith("_pq"):
            manifest[name] = train_pq_model(name[:-3])
            with open(man_path, "w") as f:
                json.dump(manifest, f, indent=1, sort_keys=True)
            continue
        spec = CONFIGS[name]
        t0 = time.time()
        n_test = 10000 if name in ("scale",) else min(spec.n_test, 200_000)
        A_train, A_test, B = make_config_data(name, n_test=n_test)
        # 8-bit configs train on the pixel values as floats (the trees see the
        # same numbers the u8 encoder compares against ceil(v), App. B reading R11)
        model = O.train(A_train.astype(np.float32), spec.C, lam=1.0, seed=spec.seed)
        blob = O.write_model(model)
        with open(os.path.join(OUT, f"{name}.mdnm"), "wb") as f:
            f.write(blob)
        exact = A_test.astype(np.float64) @ B.astype(np.float64)
        amm = O.amm_u8 if A_test.dtype == np.uint8 else O.amm
        rec = {"C": spec.C, "D": spec.D, "M": spec.M, "n_train": int(A_train.shape[0]),
               "sha256": hashlib.sha256(blob).hexdigest(), "bytes": len(blob),
               "train_s": round(time.time() - t0, 1), "nmse_rows": int(A_test.shape[0])}
        for mode in ("exact", "avg"):
            luts = O.make_luts(model, B, mode, spec.U)
            _, _, out = amm(A_test, model, luts)
            rec[f"nmse_{mode}"] = O.nmse(out, exact)
        manifest[name] = rec
        print(name, rec, flush=True)
        with open(man_path, "w") as f:
            json.dump(manifest, f, indent=1, sort_keys=True)


def train_pq_model(base):
    """The PQ comparator model (oracle K-means per subspace, L155-163) for a
    config, written as artifacts/<base>_pq.mdnm (flags bit1)."""
    spec = CONFIGS[base]
    t0 = time.time()
    n_test = 10000 if base in ("scale",) else min(spec.n_test, 200_000)
    A_train, A_test, B = make_config_data(base, n_test=n_test)
    model = O.train_pq(A_train.astype(np.float32), spec.C, n_iter=25, seed=spec.seed)
    blob = O.write_model(model)
    with open(os.path.join(OUT, f"{base}_pq.mdnm"), "wb") as f:
        f.write(blob)
    exact = A_test.astype(np.float64) @ B.astype(np.float64)
    rec = {"C": spec.C, "D": spec.D, "M": spec.M, "n_train": int(model.n_train), "pq": True,
           "sha256": hashlib.sha256(blob).hexdigest(), "bytes": len(blob),
           "train_s": round(time.time() - t0, 1), "nmse_rows": int(A_test.shape[0])}
    for mode in ("exact", "avg"):
        luts = O.make_luts(model, B, mode, spec.U)
        _, _, out = O.amm_pq(A_test, model, luts)
        rec[f"nmse_{mode}"] = O.nmse(out, exact)
    print(base + "_pq", rec, flush=True)
    return rec


if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIGS) + [n + "_pq" for n in PQ_MODELS])
