"""Offline modality-aware pattern search (Alg.4; App. A) -- the
fp64 CPU oracle of the selection rule (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Alg.4:
  intra-modality   p_mi  <- KernelAwareSearch(Q, K, V, m_i)            for every modality m_i
  cross-modality   p_mi,mj <- KernelAwareSearch(Q, K, V, m_i, m_j)     for every pair
  inter-modality   p_i   <- argmin |sparse(Q, K, V, i) - attention(Q, K, V)| over the boundary types
KernelAwareSearch (App. A): among the candidates whose kernel-measured FLOPs fit the
budget ("comparable real-world FLOPs based on GPU kernel measurements"), the one that maximises
recall of the actual attention OUTPUT ("incorporates the V matrix").  Readings (C24):
  * distance = ||O_sparse - O_dense||_2 / ||O_dense||_2 over the query rows of the region (SPEC
    search module); ties -> the earlier candidate of the search space;
  * cost = computed 128x128 tiles of the candidate's sparse index for the head -- measured by
    the GPU kernel (the "kernel-aware" FLOPs) and passed IN to this oracle as a table;
    budget = the cost of A-shape(1024, 4096) ("1k global tokens and 4k local window");
  * intra search of modality m runs the candidate as a Q-boundary pattern for every modality and
    scores the rows of m; the global (No-boundary) pick scores all rows of No-boundary runs;
  * 2D: same-modality pairs are searched with cross pairs FULL, then cross pairs with the
    same-modality winners fixed (one candidate for every cross pair at a time, scored per query
    modality); cross candidates = NONE, FULL, A-shape, vertical-only VS (reading C13);
  * inter: No-boundary(global pick), Q-boundary(intra picks), 2D(pair picks), first minimum.
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence, Tuple

import numpy as np

from synth.config import (HeadConfig, Pattern, Problem, BND_NONE, BND_Q, BND_2D, MAX_MOD,
                          grid, ashape, vslash, full, none)
from .attention import dense_causal_attention
from .pipeline import run_head


def search_space(frame_stride: int = 256, vs=None, ashapes=None, cross_vertical=(1000, 2000, 3500)) -> Dict:
    """tab:search_space: 12 Grid, 3 A-shape, 9 Vertical-Slash intra candidates."""
    flags = [(True, False, False), (False, True, False), (False, False, True),
             (True, True, False), (False, True, True), (True, True, True)]
    intra = [grid(frame_stride, *f) for f in flags] + [grid(0, *f, stride_min=2, stride_max=1024) for f in flags]
    intra += [ashape(s, l) for s, l in (ashapes or [(128, 1024), (128, 2048), (128, 4096)])]
    intra += [vslash(a, b) for a, b in (vs or [(1000, 1024), (1000, 2048), (2000, 2048), (1000, 3096), (2000, 3096),
                                               (1000, 4096), (2000, 4096), (3500, 200), (1000, 2500)])]
    cross = [none(), full()] + [ashape(s, l) for s, l in (ashapes or [(128, 1024), (128, 2048), (128, 4096)])]
    cross += [vslash(n, 0) for n in cross_vertical]
    return dict(intra=intra, cross=cross)


def distance(O: np.ndarray, O_ref: np.ndarray, rows: np.ndarray) -> float:
    if rows.size == 0:
        return 0.0
    den = np.linalg.norm(O_ref[rows])
    return float(np.linalg.norm(O[rows] - O_ref[rows]) / max(den, 1e-300))


def select(dists: Sequence[float], costs: Sequence[float], budget: float) -> int:
    """KernelAwareSearch's rule: argmin distance over cost <= budget; ties -> first."""
    best = -1
    for i, (d, c) in enumerate(zip(dists, costs)):
        if c <= budget and (best < 0 or d < dists[best]):
            best = i
    if best < 0:
        raise ValueError(f"no candidate within the budget {budget} (cheapest {min(costs)})")
    return best


def q_config(pats: Sequence[Pattern], M: int) -> HeadConfig:
    return HeadConfig.q_boundary(list(pats[:M]))


def twod_config(same: Sequence[Pattern], cross: Sequence[Sequence[Pattern]], M: int) -> HeadConfig:
    pr = [[none()] * M for _ in range(M)]
    for a in range(M):
        for b in range(M):
            pr[a][b] = same[a] if a == b else cross[a][b]
    return HeadConfig.two_d(pr)


def search_head(pb: Problem, q_h: np.ndarray, k_g: np.ndarray, v_g: np.ndarray, labels: np.ndarray,
                space: Dict, cost: Callable[[HeadConfig], float], budget: float) -> Tuple[HeadConfig, Dict]:
    """Alg.4 for one head (fp64 oracle outputs); `cost(cfg)` = the kernel-measured tiles table."""
    M = pb.n_modalities
    present = [m for m in range(M) if (labels == m).any()]
    rows_of = {m: np.nonzero(labels == m)[0] for m in range(M)}
    all_rows = np.arange(labels.shape[0])
    O_ref, _, _ = dense_causal_attention(q_h, k_g, v_g, pb.tau)

    def out(cfg):
        return run_head(pb, cfg, q_h, k_g, v_g, labels)["O"]

    rep: Dict = {}
    intra = space["intra"]
    # global (No-boundary) pick
    outs_g = [out(HeadConfig.no_boundary(c)) for c in intra]
    d_g = [distance(o, O_ref, all_rows) for o in outs_g]
    c_g = [cost(HeadConfig.no_boundary(c)) for c in intra]
    p_global = intra[select(d_g, c_g, budget)]
    rep["global"] = dict(dist=d_g, cost=c_g)
    if len(present) <= 1:
        return HeadConfig.no_boundary(p_global), rep
    # phase 1: intra-modality (Q-boundary runs, scored per query modality)
    outs_q = [out(q_config([c] * M, M)) for c in intra]
    c_q = [cost(q_config([c] * M, M)) for c in intra]
    p_intra = []
    for m in range(M):
        if m not in present:
            p_intra.append(full())
            continue
        d = [distance(o, O_ref, rows_of[m]) for o in outs_q]
        p_intra.append(intra[select(d, c_q, budget)])
        rep[f"intra{m}"] = dict(dist=d, cost=c_q)
    # phase 2: cross-modality (2D runs): same-modality pairs with cross FULL, then the cross pairs
    fullx = [[full()] * M for _ in range(M)]
    outs_s = [out(twod_config([c] * M, fullx, M)) for c in intra]
    c_s = [cost(twod_config([c] * M, fullx, M)) for c in intra]
    p_same = []
    for a in range(M):
        if a not in present:
            p_same.append(full())
            continue
        d = [distance(o, O_ref, rows_of[a]) for o in outs_s]
        p_same.append(intra[select(d, c_s, budget)])
        rep[f"same{a}"] = dict(dist=d, cost=c_s)
    cross = space["cross"]
    cfgs_x = [twod_config(p_same, [[c] * M for _ in range(M)], M) for c in cross]
    outs_x = [out(cfg) for cfg in cfgs_x]
    c_x = [cost(cfg) for cfg in cfgs_x]
    p_cross = [[full()] * M for _ in range(M)]
    for a in range(M):
        if a not in present:
            continue
        d = [distance(o, O_ref, rows_of[a]) for o in outs_x]
        pick = cross[select(d, c_x, budget)]
        rep[f"cross{a}"] = dict(dist=d, cost=c_x)
        for b in range(M):
            if b != a:
                p_cross[a][b] = pick
    # phase 3: inter-modality (boundary type)
    cands = [HeadConfig.no_boundary(p_global), q_config(p_intra, M), twod_config(p_same, p_cross, M)]
    d3 = [distance(out(c), O_ref, all_rows) for c in cands]
    c3 = [cost(c) for c in cands]
    rep["inter"] = dict(dist=d3, cost=c3)
    return cands[select(d3, c3, budget)], rep
