"""Product Quantization (PQ) comparator -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

SURVEY N4: the classic vector-quantisation encoder MADDNESS replaces, feeding
the same LUT scan, so that the encode-speed comparison of PAPER.md Sec. 5.1
(L427-438, "Maddness is up to two orders of magnitude faster than existing
methods") can be reproduced in shape on B200. Restated from Sec. 3 (L132-190):

  Prototype Learning (L144, L155-163): a separate K-means in each of the C
      disjoint subspaces J^(c), K = 16 prototypes each.
  Encoding Function (L178-184, Eq. pqLoss):
      g^(c)(a) = argmin_k sum_{j in J^(c)} (a_j - P^(c)_{k,j})^2
  Table Construction / Aggregation: identical to MADDNESS (dense P with zeros
      outside J^(c), App. A quantisation, exact or averaging scan).

Readings:
  P1  Floating point decides the integer code. The oracle evaluates Eq.
      pqLoss as written, in fp64 (pq_distances), and its code is the first
      argmin (encode_pq). An implementation that evaluates the distance in
      fp32 -- in any order, with fused multiply-adds, or in the argmin-
      invariant expanded form ||p||^2 - 2<a,p> (||a||^2 is the same for every
      k) -- may pick another prototype only when the two are closer than its
      rounding can resolve: check_pq_codes accepts code k iff
          d64(k) <= d64(k*) + eps(k) + eps(k*),   k* the first fp64 argmin,
      eps(k) = gamma_{2d+4} * (sum_j (a_j - p_kj)^2 + sum_j p_kj^2
                               + 2 sum_j |a_j p_kj|),
      gamma_n = n u / (1 - n u), u = 2^-24 (the standard bound on an n-term
      fp32 dot product / sum of squares, covering both forms). Outside that
      margin the code must be k*.
  P2  argmin ties -> the lowest k.
  P3  K-means (not specified beyond "K-means"): Lloyd iterations from a
      seeded k-means++ initialisation, fp64 arithmetic, a fixed iteration
      count; an empty cluster keeps its previous centroid. Training is not
      part of GPU parity (both paths consume the serialized model).
"""
from __future__ import annotations

import numpy as np

from .maddness import K, Model, subspaces


def kmeans(X: np.ndarray, k: int = K, n_iter: int = 25, seed: int = 0):
    """Lloyd's K-means on the rows of X (reading P3). Returns (centroids
    (k, d) fp64, assignments (N,), objective per iteration)."""
    X = np.asarray(X, np.float64)
    N = X.shape[0]
    rng = np.random.default_rng(seed)
    # k-means++ seeding
    cent = np.empty((k, X.shape[1]), np.float64)
    cent[0] = X[rng.integers(N)]
    d2 = ((X - cent[0]) ** 2).sum(1)
    for i in range(1, k):
        tot = d2.sum()
        idx = rng.integers(N) if tot == 0 else rng.choice(N, p=d2 / tot)
        cent[i] = X[idx]
        d2 = np.minimum(d2, ((X - cent[i]) ** 2).sum(1))
    objective = []
    assign = np.zeros(N, np.int64)
    for _ in range(n_iter):
        dist = ((X[:, None, :] - cent[None, :, :]) ** 2).sum(2)     # (N, k)
        assign = dist.argmin(1)
        objective.append(float(dist[np.arange(N), assign].sum()))
        for i in range(k):
            members = X[assign == i]
            if len(members):
                cent[i] = members.mean(0)
    return cent, assign, objective


def train_pq(A_train: np.ndarray, C: int, n_iter: int = 25, seed: int = 0,
             max_rows: int = 50_000) -> Model:
    """PQ prototype learning (L144, L155-163): K-means in each subspace
    J^(c) (reading R1 for the partition) on up to max_rows training rows.
    The prototypes are stored as the dense P of the MADDNESS model file (row
    16c + k = prototype k of codebook c, zero outside J^(c)), flagged pq=True;
    the hash-tree fields are unused (dims = subspace start, thresholds 0)."""
    A = np.asarray(A_train, np.float32)[:max_rows]
    N, D = A.shape
    sub = subspaces(D, C)
    P = np.zeros((K * C, D), np.float32)
    for c, (b, e) in enumerate(sub):
        cent, _, _ = kmeans(A[:, b:e], K, n_iter, seed + c)
        P[K * c:K * (c + 1), b:e] = cent.astype(np.float32)
    dims = np.array([[b] * 4 for b, _ in sub], np.int64)
    return Model(C=C, D=D, sub=sub, dims=dims, thr=np.zeros((C, 15), np.float32), P=P,
                 lam=0.0, n_train=N, seed=seed, ridge=False, pq=True)


def pq_distances(A: np.ndarray, model: Model, c: int) -> np.ndarray:
    """Eq. pqLoss (L182-184) as written: sum_{j in J^(c)} (a_j - P_kj)^2 for
    every row and k, in fp64 (reading P1). (N, K) float64."""
    A = np.asarray(A, np.float32).astype(np.float64)
    b, e = model.sub[c]
    proto = model.P[K * c:K * (c + 1), b:e].astype(np.float64)     # (K, d)
    return ((A[:, None, b:e] - proto[None, :, :]) ** 2).sum(2)


def pq_rounding_bound(A: np.ndarray, model: Model, c: int) -> np.ndarray:
    """eps(k) of reading P1 for every row and k: gamma_{2d+4} times the sum of
    the magnitudes an fp32 evaluation of Eq. pqLoss accumulates, in either the
    direct form (sum of squared differences) or the expanded form
    (||p||^2 - 2 <a, p>). (N, K) float64."""
    A = np.asarray(A, np.float32).astype(np.float64)
    b, e = model.sub[c]
    d = e - b
    proto = model.P[K * c:K * (c + 1), b:e].astype(np.float64)
    u = 2.0 ** -24
    n = 2 * d + 4
    gamma = n * u / (1 - n * u)
    mag = (pq_distances(A, model, c) + (proto ** 2).sum(1)[None, :]
           + 2 * np.abs(A[:, b:e]) @ np.abs(proto).T)
    return gamma * mag


def encode_pq(A: np.ndarray, model: Model) -> np.ndarray:
    """g(A) for PQ (Eq. pqLoss): per codebook the index of the
    nearest prototype by the fp64 distance, ties to the lowest k (readings P1,
    P2). (N, C) uint8."""
    if not getattr(model, "pq", False):
        raise ValueError("not a PQ model")
    codes = np.empty((np.asarray(A).shape[0], model.C), np.uint8)
    for c in range(model.C):
        codes[:, c] = pq_distances(A, model, c).argmin(1).astype(np.uint8)   # first minimum
    return codes


def check_pq_codes(A: np.ndarray, model: Model, codes: np.ndarray):
    """Validity of another implementation's PQ codes (N, C) against Eq. pqLoss
    (reading P1): every code's fp64 distance is within its rounding bound of
    the minimum, which forces the first argmin wherever the margin exceeds the
    bound. Returns (ok, detail)."""
    if not getattr(model, "pq", False):
        raise ValueError("not a PQ model")
    codes = np.asarray(codes).astype(np.int64)
    bad = differ = 0
    for c in range(model.C):
        dist = pq_distances(A, model, c)
        eps = pq_rounding_bound(A, model, c)
        kstar = dist.argmin(1)
        r = np.arange(dist.shape[0])
        k = codes[:, c]
        valid = (k >= 0) & (k < K)
        kk = np.where(valid, k, 0)
        within = dist[r, kk] <= dist[r, kstar] + eps[r, kk] + eps[r, kstar]
        bad += int((~(valid & within)).sum())
        differ += int((k != kstar).sum())
    return bad == 0, (f"{bad} codes outside the rounding bound; {differ} codes differ "
                      f"from the first fp64 argmin (near-ties)")


def amm_pq(A: np.ndarray, model: Model, luts, codes=None):
    """PQ codes through the same f and dequantisation as MADDNESS; `codes`
    (e.g. another implementation's codes, validated by check_pq_codes)
    replace encode_pq's where given."""
    from .maddness import dequantize, scan_avg, scan_exact
    if codes is None:
        codes = encode_pq(A, model)
    S = scan_exact(codes, luts.Tq) if luts.mode == "exact" else scan_avg(codes, luts.Tq, luts.U)
    return codes, S, dequantize(S, luts.alpha, luts.beta32)
