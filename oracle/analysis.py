"""Attention-sparsity analysis metrics -- fp64 CPU oracle (TEST INFRASTRUCTURE
ONLY, see oracle/__init__.py).

top-k coverage ("retaining only the top 5.78% of attention weights ... suffices to
recall 95% of total attention"): for a query row i, the causal softmax p_ij (j <= i); sort
descending; k = the smallest count whose cumulative mass reaches `target`; reported as k / (i + 1).
attention recall of a sparse index ("reusing top-k indices ... leads to a significant drop";
SPEC's recall): the attention mass the admitted keys carry, sum_{j in A(i)} p_ij, equal to
exp(LSE_sparse(i) - LSE_dense(i)).
"""
from __future__ import annotations

import numpy as np


def causal_probs(q_row: np.ndarray, k: np.ndarray, i: int, tau: float) -> np.ndarray:
    z = (k[:i + 1] @ q_row) * tau
    z = z - z.max()
    e = np.exp(z)
    return e / e.sum()


def topk_coverage(q: np.ndarray, k: np.ndarray, rows, tau: float, target: float = 0.95):
    """(fractions, counts) per row: smallest k with top-k mass >= target, over the i + 1 keys."""
    fr, cnt = [], []
    for i in rows:
        p = np.sort(causal_probs(q[i], k, int(i), tau))[::-1]
        c = int(np.searchsorted(np.cumsum(p), target - 1e-15) + 1)
        c = min(c, p.size)
        cnt.append(c)
        fr.append(c / (int(i) + 1))
    return np.array(fr), np.array(cnt)


def attention_recall(q: np.ndarray, k: np.ndarray, mask_rows: np.ndarray, rows, tau: float) -> np.ndarray:
    """sum of the causal softmax mass of the admitted keys per row (mask_rows [len(rows), S])."""
    out = []
    for r, i in enumerate(rows):
        p = causal_probs(q[i], k, int(i), tau)
        out.append(float(p[mask_rows[r, :int(i) + 1]].sum()))
    return np.array(out)
