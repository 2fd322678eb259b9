"""O5/O6 — dense fp64 attention under an explicit boolean mask.

O[i] = sum_{j: M(i,j)} softmax_j(tau q_i . k_j) v_j, LSE[i] = log sum exp(tau q_i.k_j)
over admitted j.  This is the exact result that Alg.5-7's online softmax
(m, l, alpha = exp(m - m_new)) reaches up to rounding order; it is
written here as the plain definition.  Rows with no admitted key: zeros,
LSE = -inf, flagged.  Fingerprints (O6): per row |{j}|, sum j,
sum j^2 (mod 2^64) over admitted original key positions.
"""
from __future__ import annotations

import numpy as np


def masked_attention(q_rows: np.ndarray, k: np.ndarray, v: np.ndarray, mask: np.ndarray,
                     tau: float):
    """q_rows [R, D], k/v [S, D], mask [R, S] bool -> (O [R, D], LSE [R], empty [R])."""
    z = (q_rows @ k.T) * tau
    z = np.where(mask, z, -np.inf)
    empty = ~mask.any(axis=1)
    zmax = np.where(empty, 0.0, z.max(axis=1))
    e = np.where(mask, np.exp(z - zmax[:, None]), 0.0)
    l = e.sum(axis=1)
    safe_l = np.where(empty, 1.0, l)
    O = (e @ v) / safe_l[:, None]
    O[empty] = 0.0
    with np.errstate(divide="ignore"):
        lse = np.where(empty, -np.inf, zmax + np.log(safe_l))
    return O, lse, empty


def dense_causal_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, tau: float):
    S = q.shape[0]
    mask = np.arange(S)[None, :] <= np.arange(S)[:, None]
    return masked_attention(q, k, v, mask, tau)


def merge_partials(O1, lse1, O2, lse2):
    """Merge two normalised partials over disjoint key sets by their LSE
    (the alpha-rescaling rule of Alg.5, generalised to two partials)."""
    m = np.maximum(lse1, lse2)
    both_empty = np.isneginf(m)
    m_safe = np.where(both_empty, 0.0, m)
    w1 = np.where(np.isneginf(lse1), 0.0, np.exp(lse1 - m_safe))
    w2 = np.where(np.isneginf(lse2), 0.0, np.exp(lse2 - m_safe))
    tot = w1 + w2
    tot_safe = np.where(both_empty, 1.0, tot)
    O = (O1 * w1[:, None] + O2 * w2[:, None]) / tot_safe[:, None]
    O[both_empty] = 0.0
    with np.errstate(divide="ignore"):
        lse = np.where(both_empty, -np.inf, m_safe + np.log(tot_safe))
    return O, lse


def fingerprint(mask: np.ndarray):
    """Per-row (count, sum j, sum j^2 mod 2^64) over admitted keys."""
    S = mask.shape[1]
    j = np.arange(S, dtype=np.uint64)
    cnt = mask.sum(axis=1).astype(np.int64)
    sj = (mask.astype(np.uint64) * j[None, :]).sum(axis=1, dtype=np.uint64)
    sj2 = (mask.astype(np.uint64) * (j * j)[None, :]).sum(axis=1, dtype=np.uint64)
    return cnt, sj, sj2
