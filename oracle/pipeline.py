"""End-to-end oracle for one head: estimate index (O2/O3) -> mask (O4) ->
masked attention + fingerprints (O5/O6), on all rows or a row sample.

The paper's pipeline: "online dynamic sparse approximation to build the
sparse index, and finally ... dynamic sparse computation".  The permutation
steps (Alg.1, Alg.2, Alg.3) do not change the result (SPEC
S:72 permutation equivariance), so the oracle computes in original order.
"""
from __future__ import annotations

from typing import Dict, Optional

import numpy as np

from synth.config import HeadConfig, Problem, KIND_GRID, BND_NONE, BND_K, BND_Q, BND_2D
from .attention import fingerprint, masked_attention
from .estimate import estimate_head
from .masks import head_mask_rows
from .modality import modality_groups

ROW_CHUNK = 256


def run_head(pb: Problem, cfg: HeadConfig, q_h: np.ndarray, k_g: np.ndarray, v_g: np.ndarray,
             labels: np.ndarray, rows: Optional[np.ndarray] = None,
             index: Optional[Dict] = None) -> Dict:
    """q_h, k_g, v_g: fp64 [S, D].  `index` overrides the oracle's own estimate
    (used to isolate kernel parity from estimation near-ties)."""
    S = q_h.shape[0]
    if index is None:
        index = estimate_head(pb, cfg, q_h, k_g, labels)
    _, rho, _ = modality_groups(labels, pb.n_modalities)
    if rows is None:
        rows = np.arange(S)
    rows = np.asarray(rows, dtype=np.int64)
    D = q_h.shape[1]
    O = np.zeros((rows.shape[0], D))
    lse = np.zeros(rows.shape[0])
    empty = np.zeros(rows.shape[0], dtype=bool)
    cnt = np.zeros(rows.shape[0], dtype=np.int64)
    sj = np.zeros(rows.shape[0], dtype=np.uint64)
    sj2 = np.zeros(rows.shape[0], dtype=np.uint64)
    for c0 in range(0, rows.shape[0], ROW_CHUNK):
        rr = rows[c0:c0 + ROW_CHUNK]
        hi = int(rr.max()) + 1
        M = head_mask_rows(cfg.boundary, index, labels, rho, rr, S)[:, :hi]
        o, l, e = masked_attention(q_h[rr], k_g[:hi], v_g[:hi], M, pb.tau)
        O[c0:c0 + rr.shape[0]] = o
        lse[c0:c0 + rr.shape[0]] = l
        empty[c0:c0 + rr.shape[0]] = e
        a, b, c = fingerprint(M)
        cnt[c0:c0 + rr.shape[0]], sj[c0:c0 + rr.shape[0]], sj2[c0:c0 + rr.shape[0]] = a, b, c
    return dict(index=index, rows=rows, O=O, lse=lse, empty=empty, count=cnt, sumj=sj, sumj2=sj2)


def hline_rows(boundary: int, index: Dict, labels: np.ndarray, rho: np.ndarray) -> np.ndarray:
    """Every horizontal-line query row of a head's grid instances (tab:search_space
    P:755-766), in original positions: No/K-boundary x = p (mod s); Q-boundary rows of
    modality m with x = p (mod s) (reading C12); 2D rows of modality a whose rank
    rho = p (mod s) (reading C13)."""
    S = labels.shape[0]
    x = np.arange(S)
    out = []
    if boundary in (BND_NONE, BND_K):
        insts = [(index["intra"][0], None, False)]
    elif boundary == BND_Q:
        insts = [(inst, m, False) for m, inst in enumerate(index["intra"])]
    else:
        insts = [(row[a], a, True) for a, row in enumerate(index["pair"])]
    for inst, m, ranked in insts:
        if inst.get("kind") != KIND_GRID or not inst.get("h"):
            continue
        coord = rho if ranked else x
        sel = np.mod(coord, inst["s"]) == inst["p"]
        if m is not None:
            sel &= labels == m
        out.append(x[sel])
    return np.concatenate(out) if out else np.zeros(0, dtype=np.int64)


def sample_rows(pb: Problem, labels: np.ndarray, index: Dict, seed: int = 0, n_random: int = 512,
                boundary: int = BND_NONE, with_hlines: bool = True) -> np.ndarray:
    """Row sample for large S: the first and last 128 rows, 8 rows
    either side of EVERY modality boundary, n_random seeded rows and (with_hlines)
    EVERY horizontal-line row of this head's grid instances."""
    S = labels.shape[0]
    rs = [np.arange(min(128, S)), np.arange(max(0, S - 128), S)]
    b = np.nonzero(labels[1:] != labels[:-1])[0] + 1
    if b.size:
        rs.append((b[:, None] + np.arange(-8, 8)[None, :]).ravel())
    rng = np.random.default_rng(seed)
    rs.append(rng.integers(0, S, size=n_random))
    if with_hlines:
        _, rho, _ = modality_groups(labels, pb.n_modalities)
        rs.append(hline_rows(boundary, index, labels, rho))
    r = np.unique(np.concatenate(rs))
    return r[(r >= 0) & (r < S)]
