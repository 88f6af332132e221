"""Pins for Algorithm 1 and the code packing (L147, L608)."""
import numpy as np
import pytest

import oracle as O
from conftest import golden


def _model_from_tree(dims, levels, D):
    thr = np.concatenate([np.asarray(v, np.float32) for v in levels])[None, :]
    return O.Model(C=1, D=D, sub=[(0, D)], dims=np.asarray([dims]), thr=thr,
                   P=np.zeros((16, D), np.float32))


def test_golden_hash_traces():
    g = golden("hash_traces.json")
    dims, levels = g["tree"]["split_idxs"], g["tree"]["thresholds"]
    m = _model_from_tree(dims, levels, 4)
    for case in g["cases"]:
        assert O.maddness_hash(case["x"], dims, levels) == case["leaf"], case["why"]
        code = O.encode(np.asarray([case["x"]], np.float32), m)[0, 0]
        assert code == case["leaf"] - 1


def _random_tree(rng, D, distinct=True):
    dims = rng.choice(D, 4, replace=not distinct)
    levels = [np.sort(rng.standard_normal(1 << t)).astype(np.float32) for t in range(4)]
    return dims, levels


def test_bruteforce_steering_every_leaf():
    """Brute force: for random trees with distinct split dims, a probe vector
    steered with x = v (goes right) or x = prev_float(v) (goes left) at each
    level's node must land in the intended leaf, for all 16 leaves."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        D = int(rng.integers(4, 12))
        dims, levels = _random_tree(rng, D)
        m = _model_from_tree(dims, levels, D)
        probes = []
        for leaf in range(16):
            bits = [(leaf >> (3 - t)) & 1 for t in range(4)]
            x = rng.standard_normal(D).astype(np.float32)
            p = 0
            for t in range(4):
                v = np.float32(levels[t][p])
                x[dims[t]] = v if bits[t] else np.nextafter(v, np.float32(-np.inf))
                p = 2 * p + bits[t]
            assert O.maddness_hash(x, dims, levels) == leaf + 1
            probes.append(x)
        codes = O.encode(np.stack(probes), m)[:, 0]
        assert list(codes) == list(range(16))


def test_encode_matches_literal_alg1_with_repeated_dims():
    """Vectorised encode == the literal per-vector Algorithm 1, including trees
    that reuse a split dim at several levels (reading R3)."""
    rng = np.random.default_rng(2)
    for _ in range(30):
        D = int(rng.integers(2, 6))
        dims, levels = _random_tree(rng, D, distinct=False)
        m = _model_from_tree(dims, levels, D)
        X = rng.standard_normal((64, D)).astype(np.float32)
        X[rng.random(X.shape) < 0.2] = 0.0
        want = [O.maddness_hash(x, dims, levels) - 1 for x in X]
        got = O.encode(X, m)[:, 0]
        assert list(got) == want
        assert got.min() >= 0 and got.max() < 16


def test_pack_unpack_roundtrip_and_layout():
    rng = np.random.default_rng(3)
    for C in (1, 2, 3, 7, 32, 64):
        codes = rng.integers(0, 16, (17, C)).astype(np.uint8)
        packed = O.pack_codes(codes)
        assert packed.shape == (17, (C + 1) // 2)
        assert (O.unpack_codes(packed, C) == codes).all()
        # low nibble = codebook 2i, high nibble = 2i + 1
        assert (packed[:, 0] & 0xF == codes[:, 0]).all()
        if C > 1:
            assert (packed[:, 0] >> 4 == codes[:, 1]).all()
        if C % 2:
            assert (packed[:, -1] >> 4 == 0).all()


def test_subspaces_partition():
    for D, C in [(32, 4), (512, 32), (27, 8), (10, 3), (5, 5)]:
        sub = O.subspaces(D, C)
        cols = [j for b, e in sub for j in range(b, e)]
        assert cols == list(range(D))
        w = [e - b for b, e in sub]
        assert max(w) - min(w) <= 1 and w == sorted(w, reverse=True)
    with pytest.raises(ValueError):
        O.subspaces(3, 4)
