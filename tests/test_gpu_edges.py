"""GPU parity of Algorithm 1's compare at its edges, for every encoder family.

Alg. 1 line 4 sends x to the right child iff x >= v. Trained
models on relu / image data almost never put an input exactly on a threshold,
so these tests build models and rows that do (readings R10, R20, R11):

* crafted models (valid model.mdnm files written by the oracle) whose
  thresholds include 0.0, -0.0, subnormals, +-FLT_MAX, +-inf and ordinary
  values, 4 distinct split dims per codebook;
* rows steered to every one of the 16 leaves of every tree, with the visited
  node's input exactly at v (-> right) or at nextafter(v, -inf) (-> left);
* rows of +-0.0, NaN (-> left, R20), +-inf, subnormals and threshold values;
* 8-bit rows at q - 1, q, q + 1 around every q = ceil(v) (R11), including
  q = 0 (v <= 0) and q = 256 (v > 255: every byte goes left).

Each shape is chosen so that a specific kernel family runs:
register-tree `k_amm_rt` (C in {4, 8}, D = 32, M <= 4), `k_amm_ws` with
SUBF = 1 (4-column subspaces), SUBF = 2 (8-column) and SUBF = 0 (wide
subspaces), the column-major kernels (thread-per-row for C <= 8, TMA gather4
for C >= 16), the generic fallbacks (misaligned A), the encode-only variants,
and the 8-bit kernels (byte-threshold register trees when every q <= 255,
else the general kernel). Codes and fp32 outputs must equal the oracle's bit
for bit."""
import numpy as np
import pytest

import oracle as O
from test_gpu_parity import _assert_out

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F32 = np.float32
SPECIAL_THR = np.array([0.0, -0.0, 1.4e-45, -1.4e-45, 1e-39, -1e-39, 3.4028235e38, -3.4028235e38,
                        np.inf, -np.inf, 1.0, -1.0, 0.5, 2.75, -7.25, 1e-7], F32)
SPECIAL_X = np.array([0.0, -0.0, np.nan, -np.nan, np.inf, -np.inf, 1.4e-45, -1.4e-45, 1e-39,
                      3.4028235e38, -3.4028235e38], F32)


@pytest.fixture(scope="module")
def mdn():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2106_10860_b200 as m
    return m


def crafted_model(C, D, seed, thr_kind="special"):
    """A valid model with 4 distinct split dims per codebook (reading R2:
    inside its subspace) and thresholds from the special pool (fp32 rows) or
    from byte-relevant values (8-bit rows)."""
    rng = np.random.default_rng(seed)
    sub = O.subspaces(D, C)
    dims = np.zeros((C, 4), np.int64)
    thr = np.zeros((C, 15), F32)
    for c, (b, e) in enumerate(sub):
        w = e - b
        dims[c] = b + (rng.permutation(w)[:4] if w >= 4 else rng.integers(0, w, 4))
        if thr_kind == "special":
            pool = np.concatenate([SPECIAL_THR, rng.standard_normal(16).astype(F32)])
            thr[c] = rng.choice(pool, 15)
        elif thr_kind == "u8":           # every q = ceil(v) in [0, 255]: byte-threshold kernels
            thr[c] = rng.choice(np.concatenate([np.arange(0, 256, 17, dtype=F32),
                                                 rng.uniform(-0.5, 254.9, 16).astype(F32)]), 15)
        else:                            # "u8x": q = 0 and q = 256 too (general 8-bit kernel)
            thr[c] = rng.choice(np.array([-3.0, 0.0, 0.25, 255.0, 255.5, 300.0, 1e30, -np.inf,
                                          np.inf, 17.0, 17.01, 128.5], F32), 15)
    P = rng.standard_normal((16 * C, D)).astype(F32)
    return O.Model(C=C, D=D, sub=sub, dims=dims, thr=thr, P=P, lam=0.0, ridge=False)


def steered_rows_f32(om, rng, reps=2):
    """For every leaf k and codebook c: x at each visited node's threshold
    (bit 1) or one ulp below it (bit 0), the other columns random."""
    with np.errstate(over="ignore", invalid="ignore"):      # nextafter(-FLT_MAX) = -inf
        return _steered_rows_f32(om, rng, reps)


def _steered_rows_f32(om, rng, reps):
    rows = []
    for _ in range(reps):
        for k in range(16):
            x = rng.standard_normal(om.D).astype(F32)
            for c in range(om.C):
                kk = (k + 5 * c) % 16          # different leaves per codebook in one row
                p = 0
                for t in range(4):
                    bit = (kk >> (3 - t)) & 1
                    v = om.thr[c, (1 << t) - 1 + p]
                    x[om.dims[c, t]] = v if bit else np.nextafter(v, F32(-np.inf))
                    p = 2 * p + bit
            rows.append(x)
    for v in SPECIAL_X:                                       # whole rows of one special value
        rows.append(np.full(om.D, v, F32))
    thr_vals = np.concatenate([om.thr.ravel(), SPECIAL_X])
    for _ in range(64):                                       # random mixes of them
        x = rng.choice(thr_vals, om.D).astype(F32)
        flip = rng.random(om.D) < 0.3
        x[flip] = np.nextafter(x[flip], F32(-np.inf))
        rows.append(x)
    return np.stack(rows).astype(F32)


def steered_rows_u8(om, rng):
    q = O.split_values_u8(om)
    rows = []
    for k in range(16):
        for delta in (-1, 0, 1):
            x = rng.integers(0, 256, om.D)
            for c in range(om.C):
                kk = (k + 3 * c) % 16
                p = 0
                for t in range(4):
                    bit = (kk >> (3 - t)) & 1
                    qq = int(q[c, (1 << t) - 1 + p])
                    x[om.dims[c, t]] = np.clip(qq + (delta if bit else -1 - abs(delta)), 0, 255)
                    p = 2 * p + bit
            rows.append(x)
    for v in (0, 1, 127, 128, 254, 255):
        rows.append(np.full(om.D, v))
    qs = np.unique(np.clip(np.concatenate([q.ravel() - 1, q.ravel(), q.ravel() + 1]), 0, 255))
    for _ in range(64):
        rows.append(rng.choice(qs, om.D))
    return np.stack(rows).astype(np.uint8)


def _tile(A, n_min=2048):
    """Repeat the rows past a few tiles (and a ragged tail) so the pipelined
    kernels run several stages."""
    reps = -(-n_min // A.shape[0])
    return np.ascontiguousarray(np.concatenate([A] * reps)[: n_min + 36])


def _luts(mdn, model, om, M, mode, seed):
    B = np.random.default_rng(seed).standard_normal((om.D, M)).astype(F32)
    U = om.C if om.C < 16 else 16
    mm = "exact" if mode == 0 else "avg"
    return mdn.mdn_build_luts(model, B, mode, U), O.make_luts(om, B, mm, U)


# (C, D, M) -> the kernel family the fused call takes
FP32_SHAPES = [
    (4, 32, 4, "rt"), (8, 32, 2, "rt"), (8, 32, 8, "ws_sub4"), (16, 64, 10, "ws_sub4"),
    (16, 128, 16, "ws_sub8"), (32, 512, 100, "ws"), (16, 512, 10, "ws"), (12, 48, 3, "generic"),
]


@pytest.mark.parametrize("C,D,M,family", FP32_SHAPES)
@pytest.mark.parametrize("mode", [0, 1], ids=["exact", "avg"])
def test_fp32_threshold_edges(mdn, C, D, M, family, mode):
    om = crafted_model(C, D, seed=C * 1000 + D)
    model = mdn.mdn_model_load(O.write_model(om), 0)
    rng = np.random.default_rng(C + D + M)
    A = _tile(steered_rows_f32(om, rng))
    if C % 16 and C > 8 and mode == 1:
        pytest.skip("averaging needs U | C")
    luts, ol = _luts(mdn, model, om, M, mode, seed=M)
    variant = mdn.mdn_amm_variant(model, luts, D)
    expect = {"rt": lambda v: v.startswith("rt"),
              "ws_sub4": lambda v: v.startswith("ws") and v.endswith("_sub4"),
              "ws_sub8": lambda v: v.startswith("ws") and v.endswith("_sub8"),
              "ws": lambda v: v.startswith("ws") and "_sub" not in v,
              "generic": lambda v: v == "generic"}[family]
    assert expect(variant), variant
    want_codes = O.encode(A, om)
    S = O.scan_exact(want_codes, ol.Tq) if mode == 0 else O.scan_avg(want_codes, ol.Tq, ol.U)
    want = O.dequantize(S, ol.alpha, ol.beta32)
    dA = torch.from_numpy(A).cuda()
    # fused g + f
    out = torch.empty((A.shape[0], M), device="cuda")
    mdn.mdn_amm(model, luts, dA, out)
    _assert_out(out.cpu().numpy(), want)
    # encode only
    nb = (C + 1) // 2
    codes = torch.empty((A.shape[0], nb), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode(model, dA, codes)
    assert (codes.cpu().numpy() == O.pack_codes(want_codes)).all()
    # generic fallbacks: A at a 4-byte offset (no TMA / vector loads)
    big = torch.zeros((A.shape[0], D + 1), device="cuda")
    big[:, 1:] = dA
    out2 = torch.empty_like(out)
    mdn.mdn_amm(model, luts, big[:, 1:], out2)
    _assert_out(out2.cpu().numpy(), want)
    codes2 = torch.empty_like(codes)
    mdn.mdn_encode(model, big[:, 1:], codes2)
    assert (codes2.cpu().numpy() == O.pack_codes(want_codes)).all()
    # column-major A: thread-per-row (C <= 8) or TMA gather4 (C >= 16)
    if C in (4, 8, 16, 32):
        At = dA.t().contiguous()
        out3 = torch.empty_like(out)
        mdn.mdn_amm_cm(model, luts, At, out3)
        _assert_out(out3.cpu().numpy(), want)
        codes3 = torch.empty_like(codes)
        mdn.mdn_encode_cm(model, At, codes3)
        assert (codes3.cpu().numpy() == O.pack_codes(want_codes)).all()


U8_SHAPES = [(8, 32, 2, "u8"), (8, 32, 2, "u8x"), (16, 64, 10, "u8"), (16, 128, 16, "u8x"),
             (32, 512, 100, "u8x"), (4, 32, 4, "u8x"), (4, 32, 4, "u8")]


@pytest.mark.parametrize("C,D,M,kind", U8_SHAPES)
@pytest.mark.parametrize("mode", [0, 1], ids=["exact", "avg"])
def test_u8_split_value_edges(mdn, C, D, M, kind, mode):
    om = crafted_model(C, D, seed=7 * C + D, thr_kind=kind)
    q = O.split_values_u8(om)
    if kind == "u8x":
        assert (q == 0).any() and (q == 256).any()
    else:
        assert q.max() <= 255
    model = mdn.mdn_model_load(O.write_model(om), 0)
    rng = np.random.default_rng(C * D)
    A = _tile(steered_rows_u8(om, rng), 4096)
    luts, ol = _luts(mdn, model, om, M, mode, seed=M + 1)
    want_codes = O.encode_u8(A, om)
    S = O.scan_exact(want_codes, ol.Tq) if mode == 0 else O.scan_avg(want_codes, ol.Tq, ol.U)
    want = O.dequantize(S, ol.alpha, ol.beta32)
    dA = torch.from_numpy(A).cuda()
    out = torch.empty((A.shape[0], M), device="cuda")
    mdn.mdn_amm_u8(model, luts, dA, out)
    _assert_out(out.cpu().numpy(), want)
    nb = (C + 1) // 2
    codes = torch.empty((A.shape[0], nb), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode_u8(model, dA, codes)
    assert (codes.cpu().numpy() == O.pack_codes(want_codes)).all()
    # 8-bit codes equal the fp32 codes of the same values (reading R11)
    assert (want_codes == O.encode(A.astype(F32), om)).all()
    # generic 8-bit fallback: 1-byte offset
    big = torch.zeros((A.shape[0], D + 1), dtype=torch.uint8, device="cuda")
    big[:, 1:] = dA
    codes2 = torch.empty_like(codes)
    mdn.mdn_encode_u8(model, big[:, 1:], codes2)
    assert (codes2.cpu().numpy() == O.pack_codes(want_codes)).all()


def test_trained_image_model_zero_threshold_codebook(mdn):
    """The trained image model's all-padding codebook 7 has constant (0.0)
    thresholds (reading R10 / constant column: every row right). Rows with
    -0.0, +0.0 and one ulp below 0 in the padding columns."""
    from helpers import model_bytes
    blob = model_bytes("image")
    om = O.read_model(blob)
    assert (om.thr[7] == 0).all()
    model = mdn.mdn_model_load(blob, 0)
    rng = np.random.default_rng(3)
    A = rng.standard_normal((3000, 32)).astype(F32)
    pads = np.array([0.0, -0.0, -1.4e-45, 1.4e-45, np.nan], F32)
    A[:, 27:] = rng.choice(pads, (3000, 5))
    dA = torch.from_numpy(A).cuda()
    codes = torch.empty((3000, 4), dtype=torch.uint8, device="cuda")
    mdn.mdn_encode(model, dA, codes)
    assert (codes.cpu().numpy() == O.pack_codes(O.encode(A, om))).all()
