"""Pins for h(B) (Sec. 3; L896) and App. A (L593-604)."""
import math

import numpy as np

import oracle as O
from conftest import golden


def test_tables_vs_textbook_gemm():
    """T = P B computed term by term equals a library fp64 GEMM of the same
    operands (special case -> textbook routine), to fp64 rounding."""
    rng = np.random.default_rng(12)
    for C, D, M in [(1, 4, 1), (4, 32, 4), (8, 27, 2), (32, 64, 10)]:
        P = rng.standard_normal((16 * C, D)).astype(np.float32)
        B = rng.standard_normal((D, M)).astype(np.float32)
        T = O.build_tables(P, B)
        ref = np.einsum("kd,dm->km", P.astype(np.float64), B.astype(np.float64)).reshape(C, 16, M)
        assert np.allclose(T, ref, rtol=1e-12, atol=1e-12)
    # unit-basis prototype picks a row of B; B = 0 gives zero tables
    P = np.zeros((16, 3), np.float32)
    P[5, 0] = 1
    B = np.array([[7.0, 1.0], [0, 0], [0, 0]], np.float32)
    T = O.build_tables(P, B)
    assert T[0, 5].tolist() == [7.0, 1.0] and T.sum() == 8.0
    assert not O.build_tables(P, np.zeros_like(B)).any()


def test_golden_quantization():
    for case in golden("quant_examples.json")["cases"]:
        T = np.asarray(case["T"], np.float64)
        Tq, delta, l, alpha = O.quantize_tables(T)
        assert l == case["l"], case.get("why")
        assert delta.tolist() == case["delta"]
        assert Tq.tolist() == case["Tq"], case.get("why")
        assert float(alpha) == 2.0 ** -l


def test_quantization_properties():
    """Round trip |alpha Tq + delta_c - T| <= alpha/2, alpha an exact
    power of two, l maximal (2^{l+1} R > 255), per-codebook monotonicity."""
    rng = np.random.default_rng(13)
    for _ in range(100):
        C, M = int(rng.integers(1, 9)), int(rng.integers(1, 12))
        T = rng.standard_normal((C, 16, M)) * 10 ** rng.uniform(-3, 3)
        Tq, delta, l, alpha = O.quantize_tables(T)
        a = float(alpha)
        assert math.frexp(a)[0] == 0.5
        err = np.abs(a * Tq + delta[:, None, None] - T)
        assert err.max() <= a / 2 * (1 + 1e-12)
        R = (T - delta[:, None, None]).max()
        assert math.ldexp(R, l) <= 255 < math.ldexp(R, l + 1)
        for c in range(C):
            o = np.argsort(T[c].ravel(), kind="stable")
            assert (np.diff(Tq[c].ravel()[o].astype(int)) >= 0).all()


def test_beta_and_debias():
    for b in golden("aise_examples.json")["bias"]:
        assert abs(O.debias_constant(b["C"], b["U"], "avg")) == b["magnitude"]
        assert O.debias_constant(b["C"], b["U"], "avg") <= 0
    assert O.debias_constant(32, 16, "exact") == 0.0
    delta = np.array([1.5, -0.25, 3.0])
    assert O.beta32(delta, np.float32(0.5), 0.0) == np.float32(4.25)
    assert O.beta32(delta, np.float32(0.5), -2.0) == np.float32(3.25)
