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
  P1  Floating point decides the integer code, so the distance is evaluated
      in the precision and order the GPU kernel uses: fp32, each operation
      rounded separately (t = a_j - p, t*t, running sum; no fused multiply-
      add), j ascending within J^(c). The plain fp64 definition agrees except
      where two distances are within that rounding error (pinned in tests).
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
    """sum_{j in J^(c)} (a_j - P_kj)^2 for every row and k, in fp32 with each
    operation rounded separately, j ascending (reading P1). (N, K) float32."""
    A = np.asarray(A, np.float32)
    b, e = model.sub[c]
    proto = model.P[K * c:K * (c + 1), b:e].astype(np.float32)     # (K, d)
    dist = np.zeros((A.shape[0], K), np.float32)
    for j in range(e - b):
        t = A[:, b + j, None] - proto[None, :, j]                  # fp32 subtract
        dist = dist + t * t                                        # fp32 mul, fp32 add
    return dist


def encode_pq(A: np.ndarray, model: Model) -> np.ndarray:
    """g(A) for PQ (Eq. pqLoss): per codebook the index of the
    nearest prototype, ties to the lowest k (reading P2). (N, C) uint8."""
    if not getattr(model, "pq", False):
        raise ValueError("not a PQ model")
    codes = np.empty((np.asarray(A).shape[0], model.C), np.uint8)
    for c in range(model.C):
        codes[:, c] = pq_distances(A, model, c).argmin(1).astype(np.uint8)   # first minimum
    return codes


def amm_pq(A: np.ndarray, model: Model, luts):
    """PQ codes through the same f and dequantisation as MADDNESS."""
    from .maddness import dequantize, scan_avg, scan_exact
    codes = encode_pq(A, model)
    S = scan_exact(codes, luts.Tq) if luts.mode == "exact" else scan_avg(codes, luts.Tq, luts.U)
    return codes, S, dequantize(S, luts.alpha, luts.beta32)
