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


def test_select_idxs_hand_example_per_bucket_not_pooled():
    """Alg. 2 line 2 (L265, L259): candidates rank by the loss summed over the
    buckets, sum_B sum_{x in B} (x_j - mean_B x_j)^2, top 4 descending, ties to
    the lower index (R3). Hand-computed values (2 buckets of 2 rows):

        dim  bucket 0  bucket 1  per-bucket L  pooled SSE
        0    0, 0      10, 10    0             100
        1    0, 2      0, 2      2 + 2 = 4     4
        2    0, 4      0, 0      8             12
        3    1, 1      1, 1      0             0
        4    0, 6      5, 5      18            22
        5    0, 1      0, 1      0.5+0.5 = 1   1
        6    0, 1      0, 1      1             1

    per-bucket top 4 = {4, 2, 1, 5} (5 beats 6 on the tie); pooled would give
    {0, 4, 2, 1}; the bottom 4 would give {0, 3, 5, 6}."""
    cols = [((0, 0), (10, 10)), ((0, 2), (0, 2)), ((0, 4), (0, 0)), ((1, 1), (1, 1)),
            ((0, 6), (5, 5)), ((0, 1), (0, 1)), ((0, 1), (0, 1))]
    X = np.array([[c[0][0] for c in cols], [c[0][1] for c in cols],
                  [c[1][0] for c in cols], [c[1][1] for c in cols]], np.float32)
    buckets = [np.array([0, 1]), np.array([2, 3])]
    assert O.heuristic_select_idxs(buckets, X) == [1, 2, 4, 5]
    assert O.heuristic_select_idxs([np.arange(4)], X) == [0, 1, 2, 4]      # one bucket: pooled
    assert O.heuristic_select_idxs(buckets, X[:, :3]) == [0, 1, 2]         # d < 4: all dims


def _brute_split_loss(Xb: np.ndarray, j: int) -> float:
    """min over every realisable split {x_j < v} / {x_j >= v} of the summed
    two-pass SSE of both children over all dims (v at each distinct value of
    x_j; v = the minimum puts every row right, which is the constant-column
    case). Empty bucket -> 0."""
    if Xb.shape[0] == 0:
        return 0.0
    best = np.inf
    for v in np.unique(Xb[:, j]):
        lo, hi = Xb[Xb[:, j] < v], Xb[Xb[:, j] >= v]
        best = min(best, O.sse_two_pass(lo) + O.sse_two_pass(hi))
    return best


def test_add_tree_level_picks_first_bruteforce_argmin():
    """Alg. 2 lines 4-15 (L281-293): the chosen dim minimises the bucket-summed
    optimal split loss over the candidates, and is the FIRST (lowest-index)
    minimiser (strict `<`, L289). Brute force over every realisable split,
    on random relu / Gaussian data and at each level of a tree."""
    rng = np.random.default_rng(10)
    for it in range(40):
        N, d = int(rng.integers(6, 60)), int(rng.integers(2, 9))
        X = rng.standard_normal((N, d)).astype(np.float32)
        if it % 2:
            X = np.maximum(X, 0)
        buckets = [np.arange(N)]
        for t in range(3):
            cands = O.heuristic_select_idxs(buckets, X)
            tot = {j: sum(_brute_split_loss(X[b], j) for b in buckets) for j in cands}
            new, l, j, v = O.add_tree_level(buckets, X)
            lo = min(tot.values())
            tol = 1e-9 * max(1.0, lo)
            assert abs(l - lo) <= tol and abs(tot[j] - lo) <= tol
            assert all(tot[jj] > lo + tol for jj in cands if jj < j), (tot, j)
            buckets = new


def test_add_tree_level_exact_tie_goes_to_lower_index():
    """Two identical columns give bit-identical split losses: the lower index
    must win (a `<=` at L289, or returning the last candidate, fails here);
    with the better column in the middle of the candidates it must be found."""
    rng = np.random.default_rng(11)
    base = rng.standard_normal(64).astype(np.float32)
    X = np.stack([rng.standard_normal(64) * 0.1, base, base, rng.standard_normal(64) * 0.1],
                 1).astype(np.float32)
    _, l, j, _ = O.add_tree_level([np.arange(64)], X)
    assert j == 1
    # the clear winner (two far clusters) in the middle of 4 candidates
    Y = rng.standard_normal((64, 4)).astype(np.float32) * 0.1
    Y[:, 2] += np.where(np.arange(64) < 32, -5.0, 5.0).astype(np.float32)
    _, _, j, v = O.add_tree_level([np.arange(64)], Y)
    assert j == 2 and -5 < v[0] < 5
