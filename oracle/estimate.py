"""O2/O3 — online sparse-index estimation, fp64, step by step.

O2 (Alg.1):
    A-hat = softmax( Q[R] K^T * tau + m_causal )   tau = 1/sqrt(d_h),
    m_causal additive -inf above the diagonal (reading C1), max-subtracted.
    R = last last_q rows (P:201, P:412 last_q = 64); for Q-/2D-boundary heads the
    last min(64, n_m) rows of each modality ("final segment of each modality's
    queries"; reading C3).
    c[j]  = sum_r A-hat[r, j]                         (column mass -> verticals)
    dg[o] = sum_r A-hat[r, pos_r - o]                 (diagonal mass -> slashes)
O3 (Alg.1 P:203-210 "max(view(A-hat, s))"; "indices for the vertical
    i_v and slash i_s lines"):
    VS:   V  = {0} + top (n_v - 1) columns by (c desc, j asc)      (C15)
          Sl = {0} + top (n_s - 1) offsets by (dg desc, o asc)
    Grid: "view" = fold of c by residue class mod s over W = [128, min R - 128)
          (C4, C6); score J(s,p) = m_s[p] - n_s[p] * T/|W| (excess mass over
          uniform, C5); argmax, ties -> smaller s, then smaller p.
Near-ties (north_star): candidates within 1e-3 relative of the cut-off are
reported, not failed.
"parity unpinned": the selection RULE (C5-C7, C15) is this
survey's reading, not the paper's text; see tests/test_oracle_estimate.py.
"""
from __future__ import annotations

from typing import Dict, List, Optional

import numpy as np

from synth.config import (KIND_NONE, KIND_FULL, KIND_ASHAPE, KIND_VSLASH, KIND_GRID,
                          KIND_TRISHAPE, KIND_SF_FIXED, KIND_SF_STRIDED,
                          BND_NONE, BND_K, BND_Q, BND_2D, Pattern, HeadConfig, Problem)
from .modality import modality_groups

FOLD_LO = 128       # reading C6: skip the sink block of keys
FOLD_GAP = 128      # reading C6: stop 128 keys before the slab
NEAR_TIE_REL = 1e-3


def slab_rows(positions: np.ndarray, last_q: int) -> np.ndarray:
    """Last min(last_q, n) entries of an ascending position list (reading C3)."""
    n = positions.shape[0]
    return positions[max(0, n - last_q):]


def slab_attention(q_rows: np.ndarray, k: np.ndarray, rows: np.ndarray, tau: float) -> np.ndarray:
    """A-hat[r, j] = softmax_j(tau * q_r . k_j + m_causal), rows at positions `rows`."""
    z = (q_rows @ k.T) * tau                                   # [R, S] fp64
    S = k.shape[0]
    causal = np.arange(S)[None, :] <= rows[:, None]
    z = np.where(causal, z, -np.inf)
    z = z - z.max(axis=1, keepdims=True)
    e = np.exp(z)
    return e / e.sum(axis=1, keepdims=True)


def column_mass(A: np.ndarray) -> np.ndarray:
    return A.sum(axis=0)


def diagonal_mass(A: np.ndarray, rows: np.ndarray) -> np.ndarray:
    """dg[o] = sum_r A[r, pos_r - o], o in [0, S)."""
    S = A.shape[1]
    dg = np.zeros(S)
    for r, pr in enumerate(rows):
        pr = int(pr)
        # keys j = pr - o for o in [0, pr]  ->  dg[0..pr] += A[r, pr::-1]
        dg[:pr + 1] += A[r, pr::-1]
    return dg


def diagonal_mass_ranked(A: np.ndarray, rows: np.ndarray, Pa: np.ndarray, rho: np.ndarray) -> np.ndarray:
    """2D same-modality pair in rank coordinates: dg_a[o] = sum_r A[r, P_a[rho(r) - o]]."""
    na = Pa.shape[0]
    dg = np.zeros(na)
    for r, pr in enumerate(rows):
        t = int(rho[int(pr)])
        dg[:t + 1] += A[r, Pa[t::-1]]
    return dg


def _topk_with_force(scores: np.ndarray, cand: np.ndarray, n: int, force: Optional[int]):
    """Ordered selection by (score desc, index asc); `force` always included and
    counts toward n.  Returns (sorted selection, near-tie list)."""
    sel = []
    pool = cand
    if force is not None and n >= 1:
        sel.append(int(force))
        pool = cand[cand != force]
        n -= 1
    if n <= 0 or pool.size == 0:
        return np.array(sorted(sel), dtype=np.int64), []
    order = np.lexsort((pool, -scores[pool]))                  # score desc, index asc
    take = pool[order[:n]]
    near = []
    if pool.size > n:
        cut = scores[take[-1]]
        tol = NEAR_TIE_REL * abs(cut)
        near = [int(j) for j in pool if abs(scores[j] - cut) <= tol]
    sel.extend(int(t) for t in take)
    return np.array(sorted(set(sel)), dtype=np.int64), near


def select_vs(c: np.ndarray, dg: np.ndarray, n_v: int, n_s: int, jmax: int, omax: int,
              force: bool = True, key_set: Optional[np.ndarray] = None) -> Dict:
    """O3 vertical-slash selection (reading C15)."""
    if key_set is None:
        cand_v = np.arange(jmax + 1, dtype=np.int64)
    else:
        cand_v = key_set[key_set <= jmax].astype(np.int64)
    V, near_v = _topk_with_force(c, cand_v, n_v, 0 if force else None)
    cand_s = np.arange(omax + 1, dtype=np.int64)
    if n_s > 0:
        Sl, near_s = _topk_with_force(dg, cand_s, n_s, 0 if force else None)
    else:
        Sl, near_s = np.zeros(0, dtype=np.int64), []
    return dict(V=V, Sl=Sl, near_v=near_v, near_s=near_s)


def grid_search(c: np.ndarray, w_lo: int, w_hi: int, candidates: List[int]) -> Dict:
    """O3 grid stride/phase search by residue folding of c over W = [w_lo, w_hi)."""
    w_lo = max(w_lo, 0)
    w_hi = min(w_hi, c.shape[0])
    N = max(0, w_hi - w_lo)
    best = None
    allJ = {}
    if N > 0:
        cw = c[w_lo:w_hi]
        jw = np.arange(w_lo, w_hi)
        T = float(cw.sum())
        for s in candidates:
            if s < 1 or N < s:
                continue
            res = jw % s
            m = np.bincount(res, weights=cw, minlength=s)[:s]
            n = np.bincount(res, minlength=s)[:s].astype(np.float64)
            J = m - n * T / N
            allJ[s] = J
            p = int(np.argmax(J))          # first max -> smallest p
            if best is None or J[p] > best[2]:   # strict: ties keep smaller s
                best = (s, p, float(J[p]))
    if best is None:
        s0 = int(min(candidates)) if candidates else 1
        return dict(s=s0, p=0, J=0.0, T=0.0, near=[], degenerate=True)
    s, p, Jb = best
    T = float(c[w_lo:w_hi].sum())
    tol = NEAR_TIE_REL * max(abs(Jb), 1e-6 * T)
    near = [(int(ss), int(pp)) for ss, J in allJ.items() for pp in np.nonzero(np.abs(J - Jb) <= tol)[0]
            if not (ss == s and pp == p)]
    return dict(s=s, p=p, J=Jb, T=T, near=near, degenerate=False)


def grid_candidates(p: Pattern) -> List[int]:
    """Reading C7: stride > 0 -> fixed frame_stride; else [stride_min, stride_max]."""
    if p.stride > 0:
        return [p.stride]
    return list(range(max(1, p.stride_min), p.stride_max + 1))


def _instance(p: Pattern, c, dg, jmax, omax, w_lo, w_hi, key_set=None, force=True, n=0) -> Dict:
    """n: extent of the pattern's coordinate system (rows of the head / of the modality)."""
    if p.kind in (KIND_NONE, KIND_FULL):
        return dict(kind=p.kind)
    if p.kind == KIND_ASHAPE:
        return dict(kind=p.kind, sink=p.sink, local=p.local)
    if p.kind == KIND_TRISHAPE:   # static: no estimation
        return dict(kind=p.kind, sink=p.sink, local=p.local, bottom=p.bottom, n=n)
    if p.kind in (KIND_SF_FIXED, KIND_SF_STRIDED):   # static
        return dict(kind=p.kind, local=p.local, stride=p.stride)
    if p.kind == KIND_VSLASH:
        d = select_vs(c, dg, p.n_vertical, p.n_slash, jmax, omax, force=force, key_set=key_set)
        d["kind"] = p.kind
        return d
    if p.kind == KIND_GRID:
        g = grid_search(c, w_lo, w_hi, grid_candidates(p))
        g.update(kind=p.kind, h=bool(p.use_hline), v=bool(p.use_vline), sl=bool(p.use_slash),
                 sink=p.sink, local=p.local)
        return g
    raise ValueError(p.kind)


def estimate_head(pb: Problem, cfg: HeadConfig, q_h: np.ndarray, k_g: np.ndarray,
                  labels: np.ndarray) -> Dict:
    """O2 + O3 for one head.  q_h, k_g: [S, D] fp64 (exact upcast of bf16)."""
    S = q_h.shape[0]
    tau = pb.tau
    P, rho, _ = modality_groups(labels, pb.n_modalities)
    out: Dict = dict(boundary=cfg.boundary)
    needs_est = lambda pat: pat.kind in (KIND_VSLASH, KIND_GRID)   # noqa: E731
    if cfg.boundary in (BND_NONE, BND_K):
        R = slab_rows(np.arange(S), pb.last_q)
        p = cfg.intra[0]
        c = dg = None
        if needs_est(p):
            A = slab_attention(q_h[R], k_g, R, tau)
            c, dg = column_mass(A), diagonal_mass(A, R)
        out["slab"] = [R]
        out["intra"] = [_instance(p, c, dg, int(R.max()), int(R.max()),
                                  FOLD_LO, int(R.min()) - FOLD_GAP, n=S)]
        out["c"], out["dg"] = [c], [dg]
        return out
    if cfg.boundary == BND_Q:
        out["intra"], out["slab"], out["c"], out["dg"] = [], [], [], []
        for m in range(pb.n_modalities):
            p = cfg.intra[m]
            if P[m].size == 0:
                out["intra"].append(dict(kind=KIND_NONE)); out["slab"].append(None)
                out["c"].append(None); out["dg"].append(None)
                continue
            R = slab_rows(P[m], pb.last_q)
            c = dg = None
            if needs_est(p):
                A = slab_attention(q_h[R], k_g, R, tau)
                c, dg = column_mass(A), diagonal_mass(A, R)
            out["intra"].append(_instance(p, c, dg, int(R.max()), int(R.max()),
                                          FOLD_LO, int(R.min()) - FOLD_GAP, n=S))
            out["slab"].append(R); out["c"].append(c); out["dg"].append(dg)
        return out
    if cfg.boundary == BND_2D:
        M = pb.n_modalities
        out["pair"] = [[dict(kind=KIND_NONE) for _ in range(M)] for _ in range(M)]
        out["slab"], out["c"], out["dg"] = [None] * M, [None] * M, [None] * M
        for a in range(M):
            if P[a].size == 0:
                continue
            R = slab_rows(P[a], pb.last_q)
            out["slab"][a] = R
            need = any(needs_est(cfg.pair[a][b]) for b in range(M))
            A = slab_attention(q_h[R], k_g, R, tau) if need else None
            c_full = column_mass(A) if need else None
            for b in range(M):
                p = cfg.pair[a][b]
                if P[b].size == 0:
                    continue
                if a == b:
                    ca = dga = None
                    if needs_est(p):
                        ca = c_full[P[a]]
                        dga = diagonal_mass_ranked(A, R, P[a], rho)
                        out["c"][a], out["dg"][a] = ca, dga
                    rR = rho[R]
                    out["pair"][a][a] = _instance(p, ca, dga, int(rR.max()), int(rR.max()),
                                                  FOLD_LO, int(rR.min()) - FOLD_GAP, n=int(P[a].size))
                else:
                    out["pair"][a][b] = _instance(p, c_full, None, int(R.max()), 0, 0, 0,
                                                  key_set=P[b], force=False)
        return out
    raise ValueError(cfg.boundary)
