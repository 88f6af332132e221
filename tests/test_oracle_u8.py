"""Pins for the 8-bit input path (App. B)."""
import numpy as np

import oracle as O
from conftest import golden


def _one_tree_model(thr15, dims=(0, 1, 2, 3), D=4):
    return O.Model(C=1, D=D, sub=[(0, D)], dims=np.asarray([dims]),
                   thr=np.asarray([thr15], np.float32), P=np.zeros((16, D), np.float32))


def test_golden_split_values():
    for case in golden("split_values_u8.json")["cases"]:
        m = _one_tree_model([case["v"]] * 15)
        assert O.split_values_u8(m)[0, 0] == case["q"], case


def test_exhaustive_byte_compare_equivalence():
    """For every byte x and 2000 thresholds (integers, half-integers, +-1 ulp
    around integers, negatives, > 255): [x >= q(v)] == [float(x) >= v]."""
    rng = np.random.default_rng(30)
    ints = rng.integers(-5, 262, 500).astype(np.float32)
    v = np.concatenate([ints, ints + 0.5, np.nextafter(ints, np.float32(1e9)),
                        np.nextafter(ints, np.float32(-1e9)),
                        rng.uniform(-20, 280, 400).astype(np.float32)])[:2000]
    x = np.arange(256)
    for chunk in np.array_split(v, 10):
        thr = np.resize(chunk, (len(chunk) // 15 + 1) * 15)[:15 * (len(chunk) // 15 or 1)]
        for k in range(0, len(thr) - 14, 15):
            m = _one_tree_model(thr[k:k + 15])
            q = O.split_values_u8(m)[0]
            want = x[:, None].astype(np.float32) >= thr[k:k + 15][None, :]
            got = x[:, None] >= q[None, :]
            assert (want == got).all()


def test_encode_u8_equals_fp32_encode_on_bytes():
    """With the 8-bit split values the codes of uint8 rows are exactly the fp32
    codes of the same values (Alg. 1 decisions unchanged)."""
    rng = np.random.default_rng(31)
    A = np.clip(np.rint(127.5 + 60 * rng.standard_normal((3000, 32))), 0, 255).astype(np.uint8)
    m = O.train(A[:2000].astype(np.float32), 8)
    assert (O.encode_u8(A, m) == O.encode(A.astype(np.float32), m)).all()
    B = rng.standard_normal((32, 3)).astype(np.float32)
    luts = O.make_luts(m, B, "exact")
    assert (O.amm_u8(A, m, luts)[2] == O.amm(A.astype(np.float32), m, luts)[2]).all()
