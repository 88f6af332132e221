"""MADDNESS oracle arithmetic -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Step-by-step restatement of the paper, in its order and notation:

  train:   subspaces J^(c) (R1) -> per codebook, 4x Algorithm 2 (with Alg. 3/4)
           -> re-encode A~ with Alg. 1 -> G -> ridge P (Sec. 4.3)
  h(B):    T = P B (Sec. 3 "Table Construction", generalised to dense P,
           App. F.1) -> App. A 8-bit quantisation (delta_c, alpha = 2^-l)
  g(A):    Algorithm 1 per codebook -> 4-bit codes
  f:       exact sum (Sec. 4.4) or the averaging estimator AISE (App. D)
  out:     alpha * f + beta   (Eq. 1; beta per App. A)

Nothing here is blocked, fused or reordered beyond what the paper states.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

K = 16          # prototypes per codebook; 4-level trees -> 16 leaves (L224, L608)
LEVELS = 4      # tree depth (Alg. 1 "for t <- 1 to 4", L235)
N_CAND = 4      # heuristic candidate count n = 4 (L265)

__all__ = [
    "K", "LEVELS", "Model", "subspaces", "maddness_hash", "encode", "pack_codes",
    "unpack_codes", "cumulative_sse", "optimal_split_threshold",
    "heuristic_select_idxs", "add_tree_level", "learn_hash_tree", "bucket_means",
    "build_G", "ridge_prototypes", "train", "build_tables", "quantize_tables",
    "beta32", "debias_constant", "mean_pair_u8", "aise_block", "scan_exact",
    "scan_avg", "dequantize", "nmse", "amm", "Luts", "make_luts", "sse_two_pass",
    "split_values_u8", "encode_u8", "amm_u8",
]


# ---------------------------------------------------------------------------
# Model container
# ---------------------------------------------------------------------------

@dataclass
class Model:
    """Trained MADDNESS g and prototypes P (L227 split params; L316 P).

    dims[c, t]  : global column index j^{t+1} of codebook c (L227), t = 0..3
    thr[c, :]   : the 15 thresholds v^1..v^4 (lengths 1,2,4,8; L227) stored in
                  heap order: level t, node p (0-based) at index 2^t - 1 + p
    P           : (K*C, D) float32 prototypes (L316)
    """
    C: int
    D: int
    sub: list            # [(begin, end)] per codebook (R1)
    dims: np.ndarray     # (C, 4) int
    thr: np.ndarray      # (C, 15) float32
    P: np.ndarray        # (16C, D) float32
    lam: float = 1.0
    n_train: int = 0
    seed: int = 0
    ridge: bool = True
    level_losses: list = field(default_factory=list)   # per codebook, 4 floats
    pq: bool = False     # PQ comparator model (oracle/pq.py): P = K-means prototypes, no trees


# ---------------------------------------------------------------------------
# Subspaces (R1)
# ---------------------------------------------------------------------------

def subspaces(D: int, C: int) -> list[tuple[int, int]]:
    """Mutually exclusive, collectively exhaustive index sets J^(c) (L157).

    Reading R1: contiguous equal blocks; when D % C != 0 the first D mod C
    blocks get one extra column.
    """
    if not (1 <= C <= D):
        raise ValueError("need 1 <= C <= D")
    base, extra = divmod(D, C)
    out, b = [], 0
    for c in range(C):
        w = base + (1 if c < extra else 0)
        out.append((b, b + w))
        b += w
    return out


# ---------------------------------------------------------------------------
# Algorithm 1: MaddnessHash  (Sec. 4.1)
# ---------------------------------------------------------------------------

def maddness_hash(x, split_idxs, split_thresholds) -> int:
    """Algorithm 1, literally, for one vector.

    split_idxs       = (j^1, .., j^4)
    split_thresholds = (v^1, .., v^4) with len(v^t) = 2^{t-1}  (L227)
    Returns the leaf index i in 1..16 (1-based, as in the paper).
    """
    i = 1                                              # L233
    for t in range(1, LEVELS + 1):                     # L235
        v = split_thresholds[t - 1][i - 1]             # L239  v <- v^t_i
        b = 1 if np.float32(x[split_idxs[t - 1]]) >= np.float32(v) else 0   # L240
        i = 2 * i - 1 + b                              # L242
    return i                                           # L244


def _levels_from_heap(thr_row: np.ndarray) -> list[np.ndarray]:
    return [thr_row[(1 << t) - 1:(1 << (t + 1)) - 1] for t in range(LEVELS)]


def encode(A: np.ndarray, model: Model) -> np.ndarray:
    """g(A): Algorithm 1 applied to every row and codebook (L228-248).

    Vectorised over rows only: for each codebook, the same four steps of
    Alg. 1 run on all rows at once. Comparisons are fp32 ``x >= v`` (L240).
    Returns codes (N, C) uint8 with code = leaf - 1 in [0, 16).
    """
    A = np.asarray(A, dtype=np.float32)
    N = A.shape[0]
    codes = np.empty((N, model.C), np.uint8)
    for c in range(model.C):
        levels = _levels_from_heap(model.thr[c])
        i = np.ones(N, np.int64)                             # L233
        for t in range(1, LEVELS + 1):                       # L235
            v = levels[t - 1][i - 1]                         # L239
            b = (A[:, model.dims[c, t - 1]] >= v).astype(np.int64)   # L240
            i = 2 * i - 1 + b                                # L242
        codes[:, c] = (i - 1).astype(np.uint8)
    return codes


def pack_codes(codes: np.ndarray) -> np.ndarray:
    """4-bit codes (L147, L608), two per byte: low nibble = codebook 2i,
    high nibble = codebook 2i+1; an odd last codebook leaves the high nibble 0."""
    N, C = codes.shape
    out = np.zeros((N, (C + 1) // 2), np.uint8)
    for c in range(C):
        out[:, c // 2] |= (codes[:, c].astype(np.uint8) & 0xF) << (4 * (c % 2))
    return out


def unpack_codes(packed: np.ndarray, C: int) -> np.ndarray:
    out = np.empty((packed.shape[0], C), np.uint8)
    for c in range(C):
        out[:, c] = (packed[:, c // 2] >> (4 * (c % 2))) & 0xF
    return out


# ---------------------------------------------------------------------------
# App. B: 8-bit split values, for natively 8-bit data (L839)
# ---------------------------------------------------------------------------

def split_values_u8(model: Model) -> np.ndarray:
    """8-bit split values for inputs that are already 8-bit integers.

    App. B quantises x and v with x -> gamma_j (x - delta_j) so that line 4 of
    Alg. 1 can compare bytes (L610-616). When the data are natively 8-bit
    (image pixels, L839) the x-quantiser is the identity (gamma = 1,
    delta = 0) and the threshold v must map to the integer q with
    x >= v  <=>  x >= q for every integer x, i.e. q = ceil(v) (reading R11).
    q is clamped to [0, 256]: v <= 0 -> 0 (every x goes right),
    v > 255 -> 256 (every x goes left). Returns (C, 15) int64 in heap order.
    """
    v = np.asarray(model.thr, np.float64)
    q = np.ceil(v)
    return np.clip(q, 0, 256).astype(np.int64)


def encode_u8(A_u8: np.ndarray, model: Model) -> np.ndarray:
    """Algorithm 1 (L228-248) on uint8 rows with the 8-bit split values:
    b <- x_{j^t} >= q^t_i, integer compare."""
    A_u8 = np.asarray(A_u8)
    assert A_u8.dtype == np.uint8
    q = split_values_u8(model)
    N = A_u8.shape[0]
    codes = np.empty((N, model.C), np.uint8)
    for c in range(model.C):
        levels = [q[c, (1 << t) - 1:(1 << (t + 1)) - 1] for t in range(LEVELS)]
        i = np.ones(N, np.int64)                                         # L233
        for t in range(1, LEVELS + 1):                                   # L235
            qq = levels[t - 1][i - 1]                                    # L239
            b = (A_u8[:, model.dims[c, t - 1]].astype(np.int64) >= qq).astype(np.int64)  # L240
            i = 2 * i - 1 + b                                            # L242
        codes[:, c] = (i - 1).astype(np.uint8)
    return codes


# ---------------------------------------------------------------------------
# Appendix C: Algorithms 3 and 4
# ---------------------------------------------------------------------------

def cumulative_sse(X: np.ndarray, reverse: bool) -> np.ndarray:
    """Algorithm 4 (L647-682) with the two readings:

    R5: lines 673-674 read X_{n,d} (the printed X_{1,d} is a typo).
    R6: for reverse=True the output is re-reversed, so out[n] (0-based) is the
        SSE of rows n..N-1, pairing with head rows 0..n-1 in Alg. 3 line 7.
    out[n] (reverse=False) = SSE over rows 0..n summed over all columns.
    Running sums are the recurrence of lines 670-678 (np.cumsum is that
    sequential recurrence), in float64.
    """
    X = np.asarray(X, dtype=np.float64)
    if reverse:                                         # L652-654
        X = X[::-1]
    N = X.shape[0]
    cumX = np.cumsum(X, axis=0)                         # L664, L673
    cumX2 = np.cumsum(X * X, axis=0)                    # L665, L674
    n = np.arange(1, N + 1, dtype=np.float64)[:, None]
    out = np.sum(cumX2 - cumX * cumX / n, axis=1)       # L677
    out[0] = 0.0                                        # L662
    if reverse:
        out = out[::-1].copy()
    return out


def sse_two_pass(X: np.ndarray) -> float:
    """Direct SSE of a set about its mean, summed over columns (L256-261)."""
    X = np.asarray(X, dtype=np.float64)
    if X.shape[0] == 0:
        return 0.0
    return float(np.sum((X - X.mean(axis=0)) ** 2))


def _midpoint_threshold(a: np.float32, b: np.float32) -> np.float32:
    """Alg. 3 line 9 midpoint (x_{n*} + x_{n*+1}) / 2 (L639), computed so that
    a < v <= b holds in fp32 (reading R9): fp64 midpoint rounded to fp32, and
    if that rounds down onto a, the next fp32 above a."""
    a64, b64 = float(a), float(b)
    v = np.float32(a64 + (b64 - a64) / 2.0)
    if v <= a:
        v = np.nextafter(np.float32(a), np.float32(np.inf))
    return np.float32(v)


def optimal_split_threshold(X: np.ndarray, j: int) -> tuple[np.float32, float]:
    """Algorithm 3 (L626-644): best threshold on column j of bucket X.

    Readings: R7 (n* ranges over 1..N-1), R8 (lowest position on ties),
    R9 (only positions with x_j[n] < x_j[n+1] -- a split between equal values
    is not realisable under the ">= goes right" rule of L240), R10 (empty
    bucket -> (0, 0)); a constant column -> (that value, SSE(B)), all rows go
    right.
    Returns (threshold fp32, loss = SSE(left) + SSE(right) over all columns).
    """
    X = np.asarray(X, dtype=np.float32)
    N = X.shape[0]
    if N == 0:                                                   # R10
        return np.float32(0.0), 0.0
    order = np.argsort(X[:, j], kind="stable")                   # L631 (ties: row order)
    Xs = X[order]
    head = cumulative_sse(Xs, reverse=False)                     # L632
    tail = cumulative_sse(Xs, reverse=True)                      # L633
    xj = Xs[:, j]
    valid = np.nonzero(xj[:-1] < xj[1:])[0]                      # R7 + R9
    if valid.size == 0:
        return np.float32(xj[0]), float(head[-1])
    losses = head[valid] + tail[valid + 1]                       # L634-635
    best = int(valid[int(np.argmin(losses))])                    # L638 (+R8: first min)
    return _midpoint_threshold(xj[best], xj[best + 1]), float(head[best] + tail[best + 1])


# ---------------------------------------------------------------------------
# Algorithm 2 and tree learning (Sec. 4.2)
# ---------------------------------------------------------------------------

def _per_dim_sse(X: np.ndarray) -> np.ndarray:
    """L(j, B) for every j (L259)."""
    if X.shape[0] == 0:
        return np.zeros(X.shape[1])
    X = X.astype(np.float64)
    return np.sum((X - X.mean(axis=0)) ** 2, axis=0)


def heuristic_select_idxs(buckets: list[np.ndarray], X: np.ndarray, n: int = N_CAND) -> list[int]:
    """Alg. 2 line 2 (L265): the top-n indices by loss summed over all buckets.

    Reading R3: ties -> lower index; d < n -> all indices. Returned ascending
    (the evaluation order of Alg. 2 lines 4-15).
    """
    d = X.shape[1]
    L = np.zeros(d)
    for B in buckets:
        L += _per_dim_sse(X[B])
    ranked = sorted(range(d), key=lambda jj: (-L[jj], jj))[:min(n, d)]
    return sorted(ranked)


def add_tree_level(buckets: list[np.ndarray], X: np.ndarray):
    """Algorithm 2 (L272-305). buckets are arrays of row ids into X.

    Returns (new_buckets, l_min, j_min, v_min)."""
    cands = heuristic_select_idxs(buckets, X)                    # L278
    l_min, j_min, v_min = math.inf, None, None                   # L280
    for j in cands:                                              # L281
        l = 0.0                                                  # L282
        v = []                                                   # L283
        for B in buckets:                                        # L284
            vi, li = optimal_split_threshold(X[B], j)            # L285
            v.append(vi)                                         # L286
            l += li                                              # L287
        if l < l_min:                                            # L289 (strict: R8)
            l_min, j_min, v_min = l, j, v                        # L290
    new = []                                                     # L296
    for B, vi in zip(buckets, v_min):                            # L297
        xj = X[B, j_min]
        new.append(B[xj < vi])                                   # L298 below
        new.append(B[xj >= vi])                                  # L298 above (>= rule, L240)
    return new, l_min, j_min, np.array(v_min, np.float32)


def learn_hash_tree(X: np.ndarray):
    """Four applications of Alg. 2 starting from B^0_1 = all rows (L255).

    Returns (local split dims (4,), thresholds in heap order (15,), leaf buckets
    (16 arrays of row ids), per-level losses (4,))."""
    X = np.asarray(X, dtype=np.float32)
    buckets = [np.arange(X.shape[0])]
    dims, thr, losses = [], np.zeros(15, np.float32), []
    for t in range(LEVELS):
        buckets, l, j, v = add_tree_level(buckets, X)
        dims.append(j)
        thr[(1 << t) - 1:(1 << (t + 1)) - 1] = v
        losses.append(l)
    return np.array(dims), thr, buckets, losses


# ---------------------------------------------------------------------------
# Prototypes (Sec. 4.3; MADDNESS-PQ bucket means L218, L420)
# ---------------------------------------------------------------------------

def build_G(codes: np.ndarray, C: int) -> np.ndarray:
    """One-hot assignment matrix G (L316-317): row = concatenated one-hot codes."""
    N = codes.shape[0]
    G = np.zeros((N, K * C), np.float64)
    rows = np.arange(N)
    for c in range(C):
        G[rows, K * c + codes[:, c].astype(np.int64)] = 1.0
    return G


def bucket_means(A: np.ndarray, codes: np.ndarray, sub: list) -> np.ndarray:
    """Prototype = mean of the subvectors hashing to each bucket (L218);
    zero outside J^(c) (L316 diagonal blocks); empty bucket -> zero (R10)."""
    N, D = A.shape
    C = len(sub)
    P = np.zeros((K * C, D), np.float64)
    for c, (b, e) in enumerate(sub):
        for k in range(K):
            rows = codes[:, c] == k
            if rows.any():
                P[K * c + k, b:e] = A[rows, b:e].astype(np.float64).mean(axis=0)
    return P


def ridge_prototypes(A: np.ndarray, codes: np.ndarray, C: int, lam: float,
                     chunk: int = 8192) -> np.ndarray:
    """P = (G^T G + lambda I)^{-1} G^T A~ (L318-321), float64.

    G^T G and G^T A~ are accumulated from dense one-hot row chunks of G (a
    plain matmul per chunk); the SPD system is solved by Cholesky.
    """
    import scipy.linalg

    N, D = A.shape
    GtG = np.zeros((K * C, K * C))
    GtA = np.zeros((K * C, D))
    for s in range(0, N, chunk):
        G = build_G(codes[s:s + chunk], C)
        GtG += G.T @ G
        GtA += G.T @ A[s:s + chunk].astype(np.float64)
    Mtx = GtG + lam * np.eye(K * C)
    cf = scipy.linalg.cho_factor(Mtx, lower=True)
    return scipy.linalg.cho_solve(cf, GtA)


def train(A_train: np.ndarray, C: int, lam: float = 1.0, seed: int = 0) -> Model:
    """Offline training (L252-323). lam = 0 is the MADDNESS-PQ sentinel
    (bucket-mean prototypes, no ridge step; L420)."""
    A_train = np.asarray(A_train, dtype=np.float32)
    N, D = A_train.shape
    sub = subspaces(D, C)
    dims = np.zeros((C, LEVELS), np.int64)
    thr = np.zeros((C, 15), np.float32)
    level_losses = []
    for c, (b, e) in enumerate(sub):
        jl, th, _, losses = learn_hash_tree(A_train[:, b:e])
        dims[c] = b + jl                      # R2: split dims stay inside J^(c)
        thr[c] = th
        level_losses.append(losses)
    model = Model(C=C, D=D, sub=sub, dims=dims, thr=thr,
                  P=np.zeros((K * C, D), np.float32), lam=lam, n_train=N, seed=seed,
                  ridge=lam > 0, level_losses=level_losses)
    codes = encode(A_train, model)            # R12: G from re-encoding A~
    if lam > 0:
        P = ridge_prototypes(A_train, codes, C, lam)
    else:
        P = bucket_means(A_train, codes, sub)
    model.P = P.astype(np.float32)
    return model


# ---------------------------------------------------------------------------
# h(B): tables and their quantisation (Sec. 3; App. A)
# ---------------------------------------------------------------------------

def build_tables(P: np.ndarray, B: np.ndarray) -> np.ndarray:
    """T[c, k, m] = sum_j P[(c,k), j] B[j, m]  (L190-192, dense P per L896).

    A plain fp64 sum in ascending j, one term at a time (each product of two
    fp32 values is exact in fp64). Returns (C, 16, M) float64."""
    P = np.asarray(P, dtype=np.float32).astype(np.float64)
    B = np.asarray(B, dtype=np.float32).astype(np.float64)
    KC, D = P.shape
    T = np.zeros((KC, B.shape[1]))
    for j in range(D):
        T += P[:, j:j + 1] * B[j:j + 1, :]
    return T.reshape(KC // K, K, B.shape[1])


def quantize_tables(T: np.ndarray):
    """App. A (L597-603) with readings R13-R15.

    delta_c = min_{m,k} T[m,c,k]                               (L598, R13)
    l       = max{ l : 2^l * max_c max_{m,k}(T - delta_c) <= 255 }   (R14)
    T^q     = rint(2^l (T - delta_c))  ties-to-even             (L602, R15)
    alpha   = 2^-l                                              (L599)
    Returns (Tq uint8 (C,16,M), delta fp64 (C,), l int, alpha fp32).
    """
    C = T.shape[0]
    delta = T.reshape(C, -1).min(axis=1)
    diff = T - delta[:, None, None]
    R = float(diff.max()) if diff.size else 0.0
    if R == 0.0:
        l = 0
    else:
        l = int(math.floor(math.log2(255.0 / R)))
        while math.ldexp(R, l + 1) <= 255.0:       # exact adjustment around log2 rounding
            l += 1
        while math.ldexp(R, l) > 255.0:
            l -= 1
    if abs(l) > 100:
        raise ValueError(f"table scale exponent l={l} out of range")
    q = np.rint(np.ldexp(diff, l))
    assert q.min() >= 0 and q.max() <= 255
    return q.astype(np.uint8), delta, l, np.float32(math.ldexp(1.0, -l))


def debias_constant(C: int, U: int, mode: str) -> float:
    """App. D (L687, L766-775), reading R16: the averaging estimator
    over-estimates by C log2(U) / 4 in expectation; the correction added to the
    integer estimate is -C log2(U)/4 (0 in exact mode)."""
    if mode == "exact":
        return 0.0
    return -C * math.log2(U) / 4.0


def beta32(delta: np.ndarray, alpha: np.float32, debias: float) -> np.float32:
    """beta = sum_c delta_c plus the debiasing constant (L604), reading R18:
    fl32(sum_c delta_c + alpha * debias), the delta sum in fp64, ascending c."""
    s = 0.0
    for d in delta:
        s += float(d)
    return np.float32(s + float(alpha) * debias)


@dataclass
class Luts:
    Tq: np.ndarray      # (C, 16, M) uint8
    delta: np.ndarray   # (C,) float64
    l: int
    alpha: np.float32
    beta32: np.float32
    mode: str
    U: int
    T: np.ndarray       # (C, 16, M) float64, unquantised (for bounds)


def make_luts(model: Model, B: np.ndarray, mode: str = "exact", U: int = 16) -> Luts:
    """h(B) + App. A + beta (the oracle's mdn_build_luts)."""
    if mode == "avg":
        _check_U(model.C, U)
    T = build_tables(model.P, B)
    Tq, delta, l, alpha = quantize_tables(T)
    b = beta32(delta, alpha, debias_constant(model.C, U, mode))
    return Luts(Tq, delta, l, alpha, b, mode, U if mode == "avg" else 1, T)


# ---------------------------------------------------------------------------
# f: aggregation (Sec. 4.4; App. D)
# ---------------------------------------------------------------------------

def scan_exact(codes: np.ndarray, Tq: np.ndarray) -> np.ndarray:
    """f(g(A), h(B))_{n,m} = sum_c T^q_{m,c,k}, k = g^(c)(a_n)  (L331), exact."""
    N, C = codes.shape
    S = np.zeros((N, Tq.shape[2]), np.int64)
    for c in range(C):
        S += Tq[c][codes[:, c].astype(np.int64)]
    return S.astype(np.int32)


def mean_pair_u8(a, b):
    """mu(a, b) = floor((a + b + 1) / 2)  (L715; vpavgb semantics L335)."""
    return (np.asarray(a, np.int64) + np.asarray(b, np.int64) + 1) // 2


def aise_block(vals: list):
    """s^_U (L698-706): x_1 if |x| = 1, else mu(s^_U(x_left), s^_U(x_right))
    with x_left / x_right the first / last half (R16, R17: halves recursion)."""
    if len(vals) == 1:
        return np.asarray(vals[0], np.int64)
    h = len(vals) // 2
    return mean_pair_u8(aise_block(vals[:h]), aise_block(vals[h:]))


def _check_U(C: int, U: int):
    if U < 1 or (U & (U - 1)) != 0 or C % U != 0:
        raise ValueError("U must be a power of two dividing C (App. D L694)")


def scan_avg(codes: np.ndarray, Tq: np.ndarray, U: int) -> np.ndarray:
    """AISE sum (L697 + L687): s^(x) = U * sum_{k=1}^{C/U} s^_U(x_{i_k:j_k}),
    blocks of U consecutive codebooks [kU, (k+1)U) (R16). Integer result."""
    N, C = codes.shape
    _check_U(C, U)
    S = np.zeros((N, Tq.shape[2]), np.int64)
    for k in range(C // U):
        vals = [Tq[c][codes[:, c].astype(np.int64)] for c in range(k * U, (k + 1) * U)]
        S += aise_block(vals)
    return (U * S).astype(np.int32)


def dequantize(S: np.ndarray, alpha: np.float32, beta: np.float32) -> np.ndarray:
    """alpha f + beta (Eq. 1): one fp32 expression. alpha*S is exact in
    fp32 (S < 2^24, alpha a power of two), so the fp32 add is the only
    rounding."""
    return np.float32(alpha) * S.astype(np.float32) + np.float32(beta)


def amm(A: np.ndarray, model: Model, luts: Luts):
    """Full inference: codes, integer sums, fp32 output."""
    codes = encode(A, model)
    if luts.mode == "exact":
        S = scan_exact(codes, luts.Tq)
    else:
        S = scan_avg(codes, luts.Tq, luts.U)
    return codes, S, dequantize(S, luts.alpha, luts.beta32)


def amm_u8(A_u8: np.ndarray, model: Model, luts: Luts):
    """Full inference on 8-bit rows: encode_u8, then the same f and dequant."""
    codes = encode_u8(A_u8, model)
    if luts.mode == "exact":
        S = scan_exact(codes, luts.Tq)
    else:
        S = scan_avg(codes, luts.Tq, luts.U)
    return codes, S, dequantize(S, luts.alpha, luts.beta32)


def nmse(approx: np.ndarray, exact: np.ndarray) -> float:
    """||C^ - AB||_F^2 / ||AB||_F^2  (L492, reading R21)."""
    approx = np.asarray(approx, np.float64)
    exact = np.asarray(exact, np.float64)
    if approx.shape != exact.shape:
        raise ValueError("shape mismatch")
    den = float(np.sum(exact * exact))
    if den == 0.0:
        raise ValueError("zero-norm exact matrix")
    return float(np.sum((approx - exact) ** 2)) / den
