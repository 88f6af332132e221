"""Pins for aggregation f (Sec. 4.4), AISE (App. D),
dequantisation (Eq. 1, App. A) and NMSE (L492)."""
import itertools
import math

import numpy as np

import oracle as O
from conftest import golden


def test_exact_scan_is_onehot_product():
    """S = G Tq (the one-hot definition, L316-317 + L331) via a dense matmul."""
    rng = np.random.default_rng(14)
    for C, M, N in [(1, 1, 5), (4, 4, 100), (32, 100, 64), (64, 10, 33)]:
        codes = rng.integers(0, 16, (N, C)).astype(np.uint8)
        Tq = rng.integers(0, 256, (C, 16, M)).astype(np.uint8)
        G = O.build_G(codes, C)
        want = (G @ Tq.reshape(16 * C, M).astype(np.float64)).astype(np.int64)
        assert (O.scan_exact(codes, Tq) == want).all()


def test_exact_scan_bruteforce_all_code_tuples():
    rng = np.random.default_rng(15)
    for C in (1, 2, 3):
        Tq = rng.integers(0, 256, (C, 16, 3)).astype(np.uint8)
        tuples = np.array(list(itertools.product(range(16), repeat=C)), np.uint8)
        S = O.scan_exact(tuples, Tq)
        for r, tup in enumerate(tuples):
            for m in range(3):
                tot = 0
                for c in range(C):
                    tot += int(Tq[c, tup[c], m])
                assert S[r, m] == tot


def test_all_equal_tables_both_modes():
    rng = np.random.default_rng(16)
    codes = rng.integers(0, 16, (50, 32)).astype(np.uint8)
    Tq = np.full((32, 16, 5), 77, np.uint8)
    assert (O.scan_exact(codes, Tq) == 32 * 77).all()
    for U in (1, 2, 4, 8, 16, 32):
        assert (O.scan_avg(codes, Tq, U) == 32 * 77).all()


def test_golden_aise():
    g = golden("aise_examples.json")
    for a, b, mu in g["mean_pair"]:
        assert O.mean_pair_u8(a, b) == mu
    for case in g["block"]:
        est = case["U"] * int(O.aise_block([np.int64(v) for v in case["vals"]]))
        assert est == case["estimate"], case["why"]


def test_aise_u2_exhaustive_bytes():
    """U = 2 over all 256^2 byte pairs: error in {0, 1}, mean exactly 1/2
    (Lemma L718-724; acceptance S:L566)."""
    a, b = np.meshgrid(np.arange(256), np.arange(256))
    err = 2 * O.mean_pair_u8(a, b) - (a + b)
    assert err.min() == 0 and err.max() == 1
    assert err.mean() == 0.5


def test_aise_bernoulli_pair_lemmas():
    """Lemmas L718-744 on the four equiprobable Bernoulli(.5) pairs: mean 1/2, variance 1/4."""
    errs = [2 * int(O.mean_pair_u8(a, b)) - (a + b) for a in (0, 1) for b in (0, 1)]
    assert np.mean(errs) == 0.5 and np.var(errs) == 0.25


def test_aise_u16_uniform_bytes_bias():
    """Theorem L766-771 checked the paper's way (L777): >= 10^6 uniform bytes,
    U = C = 16: mean(s^ - s) within 5% of C log2(U)/4 = 16; always s^ >= s and
    s^ - s <= U log2(U)/2 (acceptance S:L565-566)."""
    rng = np.random.default_rng(17)
    n_blocks = 65536
    vals = rng.integers(0, 256, (n_blocks, 16))
    est = 16 * O.aise_block([vals[:, i] for i in range(16)])
    err = est - vals.sum(axis=1)
    assert abs(err.mean() - 16.0) <= 0.05 * 16.0
    assert err.min() >= 0 and err.max() <= 16 * 4 // 2
    # through scan_avg: a C = 16 "table" whose entry k of codebook c is byte vals
    Tq = rng.integers(0, 256, (16, 16, 1)).astype(np.uint8)
    codes = rng.integers(0, 16, (n_blocks, 16)).astype(np.uint8)
    d = O.scan_avg(codes, Tq, 16)[:, 0].astype(np.int64) - O.scan_exact(codes, Tq)[:, 0]
    assert abs(d.mean() - 16.0) <= 0.05 * 16.0 and d.min() >= 0


def test_aise_u1_equals_exact_and_bound_small_U():
    rng = np.random.default_rng(18)
    codes = rng.integers(0, 16, (200, 8)).astype(np.uint8)
    Tq = rng.integers(0, 256, (8, 16, 7)).astype(np.uint8)
    assert (O.scan_avg(codes, Tq, 1) == O.scan_exact(codes, Tq)).all()
    for U in (2, 4, 8):
        d = O.scan_avg(codes, Tq, U).astype(np.int64) - O.scan_exact(codes, Tq)
        assert d.min() >= 0 and d.max() <= (8 // U) * U * math.log2(U) / 2
    for bad in (3, 16):
        try:
            O.scan_avg(codes, Tq, bad)
            raise AssertionError("expected ValueError")
        except ValueError:
            pass


def test_dequant_identity_and_exactness():
    S = np.array([[0, 1, 255, 8160]], np.int32)
    assert (O.dequantize(S, np.float32(1.0), np.float32(0.0)) == S).all()
    out = O.dequantize(S, np.float32(0.25), np.float32(-3.0))
    assert out.dtype == np.float32
    assert out.tolist() == [[-3.0, -2.75, 60.75, 2037.0]]


def test_quantisation_bound_end_to_end():
    """|alpha S + sum_c delta_c - sum_c T[c][code_c]| <= C alpha / 2 (+ fp32
    rounding) in exact mode; averaging mode adds at most alpha C log2(U)/4
    (App. A + App. D; survey pin table)."""
    rng = np.random.default_rng(19)
    C, D, M, N = 16, 32, 6, 400
    A = np.maximum(rng.standard_normal((N, D)), 0).astype(np.float32)
    model = O.train(A, C)
    B = rng.standard_normal((D, M)).astype(np.float32)
    for mode, U in (("exact", 1), ("avg", 16), ("avg", 4)):
        luts = O.make_luts(model, B, mode, U)
        codes, S, out = O.amm(A, model, luts)
        real = sum(luts.T[c][codes[:, c].astype(int)] for c in range(C))
        a = float(luts.alpha)
        bound = C * a / 2 + (C * math.log2(U) / 4 * a if mode == "avg" else 0.0)
        ulp = np.spacing(np.abs(out).astype(np.float32)).astype(np.float64)
        assert (np.abs(out.astype(np.float64) - real) <= bound + ulp + 1e-9).all()


def test_golden_nmse():
    for case in golden("nmse_examples.json")["cases"]:
        assert abs(O.nmse(np.array(case["approx"]), np.array(case["exact"])) - case["nmse"]) < 1e-12
    X = np.random.default_rng(20).standard_normal((4, 3))
    assert abs(O.nmse(3 * X, 3 * (X + 0.1)) - O.nmse(X, X + 0.1)) < 1e-12


def test_nmse_trend_with_codebooks():
    """NMSE non-increasing as C doubles on relu low-rank data (the
    qualitative trend of the paper's speed/quality curves, L455)."""
    from datagen.synth import _relu_rows
    rng = np.random.default_rng(22)
    W = rng.standard_normal((8, 32))
    Atr, Ate = _relu_rows(rng, 3000, W), _relu_rows(rng, 1000, W)
    B = (rng.standard_normal((32, 8)) / np.sqrt(32)).astype(np.float32)
    exact = Ate.astype(np.float64) @ B.astype(np.float64)
    prev = np.inf
    for C in (2, 4, 8, 16):
        m = O.train(Atr, C)
        _, _, out = O.amm(Ate, m, O.make_luts(m, B, "exact"))
        e = O.nmse(out, exact)
        assert e <= prev + 1e-3
        prev = e
    assert prev < 0.5
