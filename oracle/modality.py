"""O1 — modality bookkeeping.

Alg.2 "Q̄ <- permute(Q, i_m)" and Alg.3 permute Q, K, V by
the modality index i_m.  Reading: the permutation is the
stable grouping P_0 || P_1 || ... of ascending positions per label, labels in
ascending id order; rho(i) = index of i inside P_lab(i).
"""
from __future__ import annotations

from typing import List, Tuple

import numpy as np


def modality_groups(labels: np.ndarray, n_mod: int) -> Tuple[List[np.ndarray], np.ndarray, np.ndarray]:
    """Returns (P, rho, perm): P[m] ascending positions with label m,
    rho[i] = rank of i within its modality, perm = concat(P)."""
    labels = np.asarray(labels)
    S = labels.shape[0]
    P = [np.nonzero(labels == m)[0].astype(np.int64) for m in range(n_mod)]
    rho = np.empty(S, dtype=np.int64)
    for m in range(n_mod):
        rho[P[m]] = np.arange(P[m].shape[0])
    perm = np.concatenate(P) if n_mod else np.arange(0)
    return P, rho, perm


def inverse_permutation(perm: np.ndarray) -> np.ndarray:
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.shape[0])
    return inv


def residue_permutation(n: int, s: int) -> np.ndarray:
    """Positions 0..n-1 grouped by residue class mod s, ascending inside a class
    (the row/column-wise grid permutation of Fig. grid_pattern_permutation,
    P:711-728)."""
    idx = np.arange(n)
    return np.concatenate([idx[idx % s == r] for r in range(s)])
