"""Pins for Algorithms 3 and 4 (App. C)."""
import numpy as np

import oracle as O
from conftest import golden


def test_golden_split_and_cumsse():
    g = golden("split_examples.json")
    for case in g["split"]:
        v, loss = O.optimal_split_threshold(np.asarray(case["X"], np.float32), case["j"])
        assert float(v) == case["threshold"], case["why"]
        assert abs(loss - case["loss"]) <= 1e-12, case["why"]
    for case in g["cumsse"]:
        out = O.cumulative_sse(np.asarray(case["X"], np.float64), case["reverse"])
        assert np.allclose(out, case["out"], atol=1e-12), case["why"]


def test_empty_bucket():
    v, loss = O.optimal_split_threshold(np.zeros((0, 3), np.float32), 1)
    assert float(v) == 0.0 and loss == 0.0


def test_cumsse_matches_two_pass_every_prefix_and_suffix():
    rng = np.random.default_rng(4)
    for _ in range(100):
        N, d = int(rng.integers(1, 65)), int(rng.integers(1, 9))
        X = rng.standard_normal((N, d)) * rng.uniform(0.1, 10)
        head = O.cumulative_sse(X, False)
        tail = O.cumulative_sse(X, True)
        for n in range(N):
            h = O.sse_two_pass(X[:n + 1])
            t = O.sse_two_pass(X[n:])
            assert abs(head[n] - h) <= 1e-9 * max(1.0, h)
            assert abs(tail[n] - t) <= 1e-9 * max(1.0, t)


def _brute_split(X, j):
    """O(N^2) brute force: every threshold between two adjacent distinct sorted
    values of column j; realised partition {x_j < v} / {x_j >= v}; loss by
    two-pass SSE. Returns all (threshold, loss) candidates."""
    xs = np.unique(X[:, j])
    cands = []
    for a, b in zip(xs[:-1], xs[1:]):
        v = np.float32(float(a) + (float(b) - float(a)) / 2.0)
        if v <= a:
            v = np.nextafter(np.float32(a), np.float32(np.inf))
        left, right = X[X[:, j] < v], X[X[:, j] >= v]
        cands.append((v, O.sse_two_pass(left) + O.sse_two_pass(right)))
    if not cands:       # constant column
        return [(np.float32(X[0, j]), O.sse_two_pass(X))]
    return cands


def test_split_matches_bruteforce():
    """200 random buckets (<= 64 rows, <= 8 dims), with relu-style exact zeros
    and repeated values to exercise reading R9 (acceptance criterion S:L567)."""
    rng = np.random.default_rng(5)
    for it in range(200):
        N, d = int(rng.integers(1, 65)), int(rng.integers(1, 9))
        X = rng.standard_normal((N, d)).astype(np.float32)
        if it % 2:
            X = np.maximum(X, 0)                       # ~50% exact zeros
        if it % 3 == 0:
            X = np.round(X * 2) / 2                    # many ties
        X = X.astype(np.float32)
        j = int(rng.integers(0, d))
        v, loss = O.optimal_split_threshold(X, j)
        cands = _brute_split(X, j)
        bloss = min(c[1] for c in cands)
        assert abs(loss - bloss) <= 1e-9 * max(1.0, bloss), (it, loss, bloss)
        # realised loss of the returned threshold equals the reported loss (R9)
        real = O.sse_two_pass(X[X[:, j] < v]) + O.sse_two_pass(X[X[:, j] >= v])
        assert abs(real - loss) <= 1e-9 * max(1.0, loss)
        near = [c[0] for c in cands if c[1] <= bloss + 1e-9 * max(1.0, bloss)]
        assert float(v) in [float(x) for x in near]
        if len(near) == 1:                      # unique optimum -> same threshold
            assert float(v) == float(near[0])


def test_midpoint_is_strictly_between_in_fp32():
    a = np.float32(1.0)
    b = np.nextafter(a, np.float32(2))
    v = O.maddness._midpoint_threshold(a, b)
    assert a < v <= b
    X = np.array([[a], [b]], np.float32)
    v2, loss = O.optimal_split_threshold(X, 0)
    assert (X[:, 0] >= v2).sum() == 1 and loss == 0.0
