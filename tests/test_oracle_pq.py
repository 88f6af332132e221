"""Pins for the PQ comparator oracle (Sec. 3).

encode_pq is Eq. pqLoss (L182-184) in fp64, first argmin (readings P1, P2);
these tests tie it to exact hits, hand-placed grids, the 1-D Voronoi closed
form and translation / permutation invariance; the rounding bound of P1 to
two real fp32 evaluations; check_pq_codes to what it must accept and reject;
and K-means to its defining properties."""
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


def _fp32_direct(A, m, c):
    """An fp32 implementation of Eq. pqLoss: subtract, multiply, add each
    rounded, j ascending (no FMA)."""
    b, e = m.sub[c]
    P = m.P[16 * c:16 * (c + 1), b:e].astype(np.float32)
    d = np.zeros((A.shape[0], 16), np.float32)
    for j in range(e - b):
        t = A[:, b + j, None].astype(np.float32) - P[None, :, j]
        d = d + t * t
    return d


def _fp32_expanded(A, m, c):
    """Another fp32 implementation: ||p||^2 (rounded once) + sum_j a_j (-2 p_j),
    accumulated in fp32 -- the argmin-invariant form a fast kernel uses."""
    b, e = m.sub[c]
    P = m.P[16 * c:16 * (c + 1), b:e]
    acc = np.broadcast_to((P.astype(np.float64) ** 2).sum(1).astype(np.float32),
                          (A.shape[0], 16)).copy()
    for j in range(e - b):
        acc = acc + A[:, b + j, None].astype(np.float32) * (np.float32(-2) * P[None, :, j])
    return acc


def test_rounding_bound_covers_fp32_evaluations():
    """eps(k) of reading P1 bounds the actual error of both fp32 forms against
    the fp64 definition, on every row and prototype (incl. large offsets that
    make the expanded form cancel)."""
    rng = np.random.default_rng(40)
    for C, d, shift in ((4, 8, 0.0), (8, 4, 0.0), (3, 16, 0.0), (2, 32, 50.0)):
        m = _random_pq_model(rng, C, d)
        m.P[:] += np.float32(shift) * (m.P != 0)
        A = (shift + rng.standard_normal((3000, C * d))).astype(np.float32)
        for c, (b, e) in enumerate(m.sub):
            d64 = O.pq_distances(A, m, c)
            eps = O.pq_rounding_bound(A, m, c)
            an = (A[:, b:e].astype(np.float64) ** 2).sum(1)[:, None]
            assert (np.abs(_fp32_direct(A, m, c) - d64) <= eps).all()
            assert (np.abs(_fp32_expanded(A, m, c).astype(np.float64) + an - d64) <= eps).all()


def test_check_pq_codes_accepts_fp32_and_rejects_wrong_codes():
    """fp32 argmins (either form) pass check_pq_codes; off near-ties they are
    the fp64 first argmin; replacing a code by the second-best prototype where
    the margin exceeds the bound fails."""
    rng = np.random.default_rng(46)
    for C, d in ((4, 8), (8, 4), (3, 16)):
        m = _random_pq_model(rng, C, d)
        A = rng.standard_normal((4000, C * d)).astype(np.float32)
        ref = O.encode_pq(A, m)
        for form in (_fp32_direct, _fp32_expanded):
            got = np.stack([form(A, m, c).argmin(1) for c in range(C)], 1)
            ok, _ = O.check_pq_codes(A, m, got)
            assert ok
            assert (got != ref).mean() < 0.01
        bad = ref.copy()
        d64 = O.pq_distances(A, m, 0)
        eps = O.pq_rounding_bound(A, m, 0)
        second = np.argsort(d64, 1, kind="stable")[:, 1]
        r = np.arange(len(A))
        far = d64[r, second] - d64[r, ref[:, 0]] > 10 * (eps[r, second] + eps[r, ref[:, 0]])
        assert far.any()
        n0 = int(np.flatnonzero(far)[0])
        bad[n0, 0] = second[n0]
        assert not O.check_pq_codes(A, m, bad)[0]
        bad[n0, 0] = 16                                 # out of range
        assert not O.check_pq_codes(A, m, bad)[0]


def test_encode_pq_one_dim_voronoi():
    """C = 1, d = 1: the nearest of 16 sorted points on a line is the one whose
    interval between neighbouring midpoints holds a (closed form)."""
    rng = np.random.default_rng(47)
    pts = np.sort(rng.uniform(-10, 10, 16)).astype(np.float32)
    perm = rng.permutation(16)
    P = pts[perm].reshape(16, 1)
    m = O.Model(C=1, D=1, sub=[(0, 1)], dims=np.zeros((1, 4), np.int64),
                thr=np.zeros((1, 15), np.float32), P=P, ridge=False, lam=0.0, pq=True)
    a = rng.uniform(-12, 12, 5000).astype(np.float32)
    mids = (pts[:-1].astype(np.float64) + pts[1:]) / 2
    rank = np.searchsorted(mids, a.astype(np.float64))          # index into sorted points
    keep = np.abs(a[:, None] - mids[None, :]).min(1) > 1e-4     # off the exact boundaries
    want = np.argsort(perm)[rank]                                # sorted rank -> prototype index
    got = O.encode_pq(a.reshape(-1, 1), m)[:, 0]
    assert (got[keep] == want[keep]).all()


def test_encode_pq_translation_and_permutation_invariance():
    """Shifting rows and prototypes by the same vector keeps the codes;
    permuting the prototypes permutes the codes."""
    rng = np.random.default_rng(48)
    m = _random_pq_model(rng, 4, 4)
    A = rng.standard_normal((2000, 16)).astype(np.float32)
    ref = O.encode_pq(A, m)
    shift = np.float32(0.5)                                     # exact in fp32 at these magnitudes
    m2 = _random_pq_model(rng, 4, 4)
    m2.P[:] = m.P + shift * (m.P != 0)
    assert (O.encode_pq(A + shift, m2) == ref).mean() > 0.999
    perm = rng.permutation(16)
    m3 = _random_pq_model(rng, 4, 4)
    for c in range(4):
        m3.P[16 * c:16 * (c + 1)] = m.P[16 * c + perm]
    inv = np.argsort(perm)
    assert (O.encode_pq(A, m3) == inv[ref]).all()


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
