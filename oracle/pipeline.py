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

from synth.config import HeadConfig, Problem
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


def sample_rows(pb: Problem, labels: np.ndarray, index: Dict, seed: int = 0, n_random: int = 512) -> np.ndarray:
    """Row sample for large S: first/last 128 rows, 8 rows either
    side of each modality boundary, n_random seeded rows, and the hline rows of a
    grid index (capped) when present."""
    S = labels.shape[0]
    rs = [np.arange(min(128, S)), np.arange(max(0, S - 128), S)]
    b = np.nonzero(labels[1:] != labels[:-1])[0] + 1
    for x in b[:64]:
        rs.append(np.arange(max(0, x - 8), min(S, x + 8)))
    rng = np.random.default_rng(seed)
    rs.append(rng.integers(0, S, size=n_random))
    inst = index.get("intra", [None])[0] if index.get("intra") else None
    if inst is not None and inst.get("kind") == 4 and inst.get("h"):
        hl = np.arange(inst["p"], S, inst["s"])
        rs.append(hl[:: max(1, hl.shape[0] // 64)])
    return np.unique(np.concatenate(rs))
