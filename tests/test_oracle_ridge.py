"""Pins for the prototype step (Sec. 4.3; bucket means L218)."""
import numpy as np

import oracle as O
from conftest import golden


def test_paper_G_example():
    g = golden("ridge_examples.json")["G_example"]
    codes = np.asarray([[c - 1 for c in g["codes_1based"]]], np.uint8)
    # build_G's K is fixed to 16 by the method; check the paper's K=4 example by
    # taking each codebook's first K columns of the 16-wide one-hot block.
    G = O.build_G(codes, g["C"])
    row = np.concatenate([G[0, 16 * c:16 * c + g["K"]] for c in range(g["C"])])
    assert row.tolist() == g["row"]
    assert G.sum() == g["C"]


def test_ridge_closed_forms():
    for case in golden("ridge_examples.json")["closed_forms"]:
        codes = np.asarray(case["codes"], np.uint8)
        A = np.asarray(case["A"], np.float64)
        P = O.ridge_prototypes(A, codes, 1, case["lam"])
        for k, want in case["P_rows"].items():
            assert np.allclose(P[int(k)], want, atol=1e-12), case["why"]
        unused = [k for k in range(16) if str(k) not in case["P_rows"]]
        assert np.allclose(P[unused], 0.0)


def _objective(A, G, P, lam):
    return float(np.sum((A - G @ P) ** 2) + lam * np.sum(P ** 2))


def test_ridge_stationarity_and_optimality():
    """Acceptance S:L569: ||G^T(A - GP) - lam P|| <= 1e-4 ||G^T A|| and the
    ridge objective at P_ridge <= objective at the bucket means."""
    rng = np.random.default_rng(10)
    for _ in range(30):
        N, C = int(rng.integers(20, 200)), int(rng.integers(1, 4))
        D = int(rng.integers(C, 9))
        A = rng.standard_normal((N, D))
        codes = rng.integers(0, 16, (N, C)).astype(np.uint8)
        lam = 1.0
        P = O.ridge_prototypes(A, codes, C, lam)
        G = O.build_G(codes, C)
        grad = G.T @ (A - G @ P) - lam * P
        assert np.linalg.norm(grad) <= 1e-4 * np.linalg.norm(G.T @ A)
        P0 = O.bucket_means(A.astype(np.float32), codes, O.subspaces(D, C))
        assert _objective(A, G, P, lam) <= _objective(A, G, P0, lam) + 1e-9


def test_bucket_means():
    A = np.array([[0, 2, 9], [2, 4, 9], [5, 5, 5]], np.float32)
    codes = np.array([[3], [3], [1]], np.uint8)
    P = O.bucket_means(A, codes, [(0, 3)])
    assert np.allclose(P[3], [1, 3, 9]) and np.allclose(P[1], [5, 5, 5])
    assert np.allclose(np.delete(P, [1, 3], axis=0), 0)
    # two codebooks: prototypes are zero outside their own subspace (L316)
    P2 = O.bucket_means(A, np.array([[3, 0], [3, 0], [1, 0]], np.uint8), [(0, 2), (2, 3)])
    assert np.allclose(P2[3], [1, 3, 0]) and np.allclose(P2[16], [0, 0, 23 / 3])


def test_large_lambda_shrinks():
    rng = np.random.default_rng(11)
    A = rng.standard_normal((50, 4))
    codes = rng.integers(0, 16, (50, 1)).astype(np.uint8)
    assert np.linalg.norm(O.ridge_prototypes(A, codes, 1, 1e9)) < 1e-6
