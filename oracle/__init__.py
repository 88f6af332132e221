"""MADDNESS oracle -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (numpy, float64 wherever
the paper does not fix the precision) of everything the B200 hot path
computes, written from PAPER.md (Blalock & Guttag, "Multiplying Matrices
Without Multiplying", ICML 2021, arXiv 2106.10860) and nothing else.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs and its untimed per-rank parity
check (``rank_parity``) may import, call or execute
anything in this package. The product path (``paper_2106_10860_b200``,
``libmaddness``) never imports it and shares no code with it; the only
things the two sides share are the documented file formats
(``include/maddness.h``) and the seeded input generators in ``datagen/``.

Every function cites the passage it follows as ``PAPER.md L<line> (<section>)``.
Readings of ambiguous / garbled passages are labelled R1..R21 (DESIGN.md
"Readings").  Parity status: every function is pinned by ``tests/test_oracle_*``
except the absolute NMSE level of a trained model (no paper number survives:
the figures are missing) -- "parity unpinned" for that quantity only.
"""
from .maddness import *  # noqa: F401,F403
from .model_file import read_model, write_model  # noqa: F401
from .pq import (amm_pq, check_pq_codes, encode_pq, kmeans, pq_distances,  # noqa: F401
                 pq_rounding_bound, train_pq)
