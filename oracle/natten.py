"""Neighborhood attention (NATTEN) for DiT video latents -- fp64 CPU oracle (TEST INFRASTRUCTURE
ONLY, see oracle/__init__.py).  SURVEY §8f f4; App. F P:884-895.

Tokens of a T x Hh x Ww grid in raster order, pos = (t * Hh + y) * Ww + x.  Query (t, y, x)
attends, bidirectionally (DiT attention is not causal), to the keys of its window: per dimension
d with extent L_d and window k_d, start_d = clamp(c_d - k_d // 2, 0, L_d - k_d) and the keys
c'_d in [start_d, start_d + k_d) -- NATTEN's clamped neighborhood, so every query sees exactly
kt * kh * kw keys (reading C25).  The permutation into 3D tiles does not change the result.
"""
from __future__ import annotations

import numpy as np

from .attention import masked_attention


def coords(cfg, pos):
    pos = np.asarray(pos, dtype=np.int64)
    return pos // (cfg.Hh * cfg.Ww), (pos // cfg.Ww) % cfg.Hh, pos % cfg.Ww


def window_start(c, k, L):
    return np.clip(np.asarray(c) - k // 2, 0, L - k)


def natten_mask_rows(cfg, rows) -> np.ndarray:
    S = cfg.seq_len
    qt, qy, qx = coords(cfg, rows)
    kt, ky, kx = coords(cfg, np.arange(S))
    m = np.ones((len(rows), S), dtype=bool)
    for qc, kc, k, L in ((qt, kt, cfg.kt, cfg.T), (qy, ky, cfg.kh, cfg.Hh), (qx, kx, cfg.kw, cfg.Ww)):
        st = window_start(qc, k, L)[:, None]
        m &= (kc[None, :] >= st) & (kc[None, :] < st + k)
    return m


def natten_attention(cfg, q, k, v, tau, rows=None):
    """(O, LSE, mask) for the given query rows (all rows by default)."""
    rows = np.arange(cfg.seq_len) if rows is None else np.asarray(rows)
    M = natten_mask_rows(cfg, rows)
    O, lse, _ = masked_attention(q[rows], k, v, M, tau)
    return O, lse, M
