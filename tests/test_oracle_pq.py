"""Pins for the PQ comparator oracle (Sec. 3).

encode_pq follows Eq. pqLoss (L182-184) in fp32 with separately rounded
operations (reading P1); these tests tie it to the fp64 definition, to exact
hits and hand-placed grids, and K-means to its defining properties."""
import numpy as np

import oracle as O


def _random_pq_model(rng, C, d, scale=1.0):
    D = C * d
    P = np.zeros((16 * C, D), np.float32)
    sub = O.subspaces(D, C)
    for c, (b, e) in enumerate(sub):
        P[16 * c:16 * (c + 1), b:e] = (scale * rng.standard_normal((16, e - b))).astype(np.float32)
    return O.Model(C=C, D=D, sub=sub, dims=np.array([[b] * 4 for b, _ in sub]),
                   thr=np.zeros((C, 15), np.float32), P=P, ridge=False, lam=0.0, pq=True)


def test_encode_pq_matches_fp64_definition_off_ties():
    """argmin_k sum_j (a_j - P_kj)^2 in fp64 (the plain definition) equals the
    fp32 oracle wherever the best and second-best fp64 distances differ by more
    than the fp32 evaluation error can move them."""
    rng = np.random.default_rng(40)
    for C, d in ((4, 8), (8, 4), (3, 16)):
        m = _random_pq_model(rng, C, d)
        A = rng.standard_normal((4000, C * d)).astype(np.float32)
        got = O.encode_pq(A, m)
        for c, (b, e) in enumerate(m.sub):
            X = A[:, b:e].astype(np.float64)
            Pc = m.P[16 * c:16 * (c + 1), b:e].astype(np.float64)
            dist = ((X[:, None, :] - Pc[None]) ** 2).sum(2)
            srt = np.sort(dist, 1)
            margin = srt[:, 1] - srt[:, 0]
            # bound on the fp32 error of each distance: ~ (d + 2) ulp of the sum
            tol = (e - b + 2) * np.finfo(np.float32).eps * 4 * srt[:, 1]
            ok = margin > tol
            assert ok.mean() > 0.99
            assert (got[ok, c] == dist[ok].argmin(1)).all()


def test_encode_pq_exact_hits_and_lowest_index_ties():
    rng = np.random.default_rng(41)
    m = _random_pq_model(rng, 2, 6)
    # rows equal to prototype k of codebook 0 and prototype 15-k of codebook 1
    A = np.zeros((16, 12), np.float32)
    for k in range(16):
        A[k, 0:6] = m.P[k, 0:6]
        A[k, 6:12] = m.P[16 + 15 - k, 6:12]
    codes = O.encode_pq(A, m)
    assert (codes[:, 0] == np.arange(16)).all()
    assert (codes[:, 1] == 15 - np.arange(16)).all()
    # duplicate prototypes: the lower index wins (reading P2)
    m.P[16 + 9, 6:12] = m.P[16 + 4, 6:12]
    A[0, 6:12] = m.P[16 + 4, 6:12]
    assert O.encode_pq(A[:1], m)[0, 1] == 4


def test_encode_pq_hand_grid():
    """C = 1, d = 2, prototypes on the 4 x 4 grid {0,10,20,30}^2 with index
    4*row + col; points jittered by < 5 map to their grid point."""
    P = np.zeros((16, 2), np.float32)
    for r in range(4):
        for cc in range(4):
            P[4 * r + cc] = (10 * r, 10 * cc)
    m = O.Model(C=1, D=2, sub=[(0, 2)], dims=np.zeros((1, 4), np.int64),
                thr=np.zeros((1, 15), np.float32), P=P, ridge=False, lam=0.0, pq=True)
    rng = np.random.default_rng(42)
    idx = rng.integers(0, 16, 500)
    A = (P[idx] + rng.uniform(-4.9, 4.9, (500, 2))).astype(np.float32)
    assert (O.encode_pq(A, m)[:, 0] == idx).all()


def test_pq_distances_literal_scalar_loop():
    """The vectorised distances equal a literal scalar loop over j (fp32
    subtract, multiply, add; j ascending) bit for bit."""
    rng = np.random.default_rng(43)
    m = _random_pq_model(rng, 2, 5)
    A = rng.standard_normal((20, 10)).astype(np.float32)
    for c, (b, e) in enumerate(m.sub):
        got = O.pq_distances(A, m, c)
        for n in range(20):
            for k in range(16):
                s = np.float32(0)
                for j in range(b, e):
                    t = np.float32(A[n, j]) - np.float32(m.P[16 * c + k, j])
                    s = np.float32(s + np.float32(t * t))
                assert got[n, k].view(np.uint32) == s.view(np.uint32)


def test_kmeans_properties():
    rng = np.random.default_rng(44)
    centers = rng.uniform(-100, 100, (16, 3))
    X = np.concatenate([c + rng.standard_normal((200, 3)) for c in centers])
    cent, assign, obj = O.kmeans(X, 16, 30, seed=1)
    # Lloyd's objective never increases
    assert all(b <= a * (1 + 1e-12) for a, b in zip(obj, obj[1:]))
    # fixed point: every centroid is the mean of its members
    for i in range(16):
        if (assign == i).any():
            assert np.allclose(cent[i], X[assign == i].mean(0), atol=1e-9)
    # 16 separated clusters (std 1, >= ~10 apart) are recovered one per centroid
    d = np.sqrt(((cent[:, None] - centers[None]) ** 2).sum(2))
    assert sorted(d.argmin(1)) == list(range(16))
    assert d.min(1).max() < 0.5


def test_train_pq_model_roundtrip():
    rng = np.random.default_rng(45)
    A = rng.standard_normal((2000, 16)).astype(np.float32)
    m = O.train_pq(A, 4, n_iter=5)
    m2 = O.read_model(O.write_model(m))
    assert m2.pq and not m2.ridge
    assert (m2.P == m.P).all()
    # prototypes live inside their subspaces (zero elsewhere, as the dense P of h(B))
    for c, (b, e) in enumerate(m.sub):
        blk = m.P[16 * c:16 * (c + 1)]
        assert (blk[:, :b] == 0).all() and (blk[:, e:] == 0).all()
    assert (O.encode_pq(A, m2) == O.encode_pq(A, m)).all()
