"""Pins for Algorithm 2 / tree learning (Sec. 4.2)."""
import numpy as np

import oracle as O


def test_select_idxs_bruteforce_and_ties():
    rng = np.random.default_rng(6)
    for _ in range(50):
        d = int(rng.integers(1, 9))
        X = rng.standard_normal((40, d)).astype(np.float32)
        X[:, rng.random(d) < 0.3] = 1.0        # some constant columns (ties at 0)
        buckets = [np.arange(0, 13), np.arange(13, 40)]
        L = [sum(O.sse_two_pass(X[b][:, [j]]) for b in buckets) for j in range(d)]
        want = sorted(sorted(range(d), key=lambda j: (-round(L[j], 9), j))[:min(4, d)])
        assert O.heuristic_select_idxs(buckets, X) == want
    # all columns constant -> lowest indices (R3)
    X = np.ones((5, 6), np.float32)
    assert O.heuristic_select_idxs([np.arange(5)], X) == [0, 1, 2, 3]


def test_tree_partition_monotone_and_consistent():
    """50 random training sets: buckets partition the rows at every level,
    level loss equals the realised SSE of the buckets and never increases
    (acceptance S:L568), and re-encoding reproduces the leaves (self-consistency
    under reading R9)."""
    rng = np.random.default_rng(7)
    for it in range(50):
        N, d = int(rng.integers(20, 300)), int(rng.integers(1, 9))
        X = rng.standard_normal((N, d)).astype(np.float32)
        if it % 2:
            X = np.maximum(X, 0)
        buckets = [np.arange(N)]
        prev = O.sse_two_pass(X)
        for t in range(4):
            buckets, l, j, v = O.add_tree_level(buckets, X)
            assert len(buckets) == 1 << (t + 1)
            allrows = np.sort(np.concatenate(buckets))
            assert (allrows == np.arange(N)).all()
            real = sum(O.sse_two_pass(X[b]) for b in buckets)
            assert abs(real - l) <= 1e-8 * max(1.0, real)
            assert l <= prev * (1 + 1e-12) + 1e-12
            prev = l
        dims, thr, leaves, losses = O.learn_hash_tree(X)
        m = O.Model(C=1, D=d, sub=[(0, d)], dims=dims[None], thr=thr[None],
                    P=np.zeros((16, d), np.float32))
        codes = O.encode(X, m)[:, 0]
        for k in range(16):
            assert (np.sort(np.nonzero(codes == k)[0]) == np.sort(leaves[k])).all()


def test_sixteen_clusters_one_per_leaf():
    """16 well separated 1-D clusters -> each leaf holds exactly one cluster
    (SPEC.md L142 derived example)."""
    rng = np.random.default_rng(8)
    centers = np.arange(16) * 10.0
    X = (np.repeat(centers, 25) + rng.uniform(-1, 1, 16 * 25)).astype(np.float32)[:, None]
    dims, thr, leaves, losses = O.learn_hash_tree(X)
    for k, b in enumerate(leaves):
        cl = np.unique(np.round(X[b, 0] / 10.0))
        assert cl.size == 1
    within = sum(O.sse_two_pass(X[np.abs(X[:, 0] - c) < 5]) for c in centers)
    assert abs(losses[-1] - within) <= 1e-6 * within


def test_single_repeated_row_zero_loss():
    X = np.tile(np.array([[1.0, 2.0, 3.0]], np.float32), (50, 1))
    dims, thr, leaves, losses = O.learn_hash_tree(X)
    assert all(l == 0.0 for l in losses)
    # constant data: every split goes right (>= rule), all rows in leaf 15
    assert len(leaves[15]) == 50


def test_train_dims_inside_subspace():
    rng = np.random.default_rng(9)
    A = np.maximum(rng.standard_normal((500, 24)), 0).astype(np.float32)
    m = O.train(A, 3)
    for c, (b, e) in enumerate(m.sub):
        assert ((m.dims[c] >= b) & (m.dims[c] < e)).all()
