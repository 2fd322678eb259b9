"""Offline modality-aware sparse-attention pattern search on the GPU (Alg.4,
P:578-614; App. A; search space tab:search_space P:749-785).

Every candidate is evaluated for ALL heads of the layer at once by the library's own hot path
(mmi_estimate_index -> mmi_permute -> mmi_sparse_prefill -> mmi_unpermute) and compared with the
same-build dense causal kernel (mmi_dense_prefill).  The cost of a candidate is "kernel-aware"
(App. A: "comparable real-world FLOPs based on GPU kernel measurements"): the computed 128x128
tiles of its sparse index per head, read back from the index; the budget is the cost of
A-shape(1024, 4096).  Distances ||O - O_ref|| / ||O_ref|| per head and query-modality
region are offline bookkeeping (torch reductions on the outputs; not part of the hot path).
The selection rule is written out in oracle/search.py (fp64) and the GPU parity test feeds that
oracle this module's cost table (tests/test_gpu_search.py).

    python -m paper_2504_16083_b200.search --workload 0 --out heads.json [--bench]
"""
from __future__ import annotations

import argparse
import json
import time
from typing import Dict, List, Optional, Sequence, Tuple

import torch

from synth.config import (HeadConfig, Pattern, Problem, MAX_MOD, grid, ashape, vslash, full, none,
                          save_head_configs)
from .mmi import SparsePrefill, dense_prefill


def search_space(frame_stride: int = 256) -> Dict:
    """tab:search_space: 12 Grid (frame_stride / searched stride x the six line-flag
    combinations, max stride 1024), 3 A-shape, 9 Vertical-Slash intra candidates; cross-pair
    candidates: NONE, FULL, A-shape, vertical-only VS (reading C13)."""
    flags = [(True, False, False), (False, True, False), (False, False, True),
             (True, True, False), (False, True, True), (True, True, True)]
    intra = [grid(frame_stride, *f) for f in flags] + [grid(0, *f, stride_min=2, stride_max=1024) for f in flags]
    intra += [ashape(128, l) for l in (1024, 2048, 4096)]
    intra += [vslash(a, b) for a, b in ((1000, 1024), (1000, 2048), (2000, 2048), (1000, 3096), (2000, 3096),
                                        (1000, 4096), (2000, 4096), (3500, 200), (1000, 2500))]
    cross = [none(), full()] + [ashape(128, l) for l in (1024, 2048, 4096)] + [vslash(n, 0) for n in (1000, 2000, 3500)]
    return dict(intra=intra, cross=cross)


def _q(pats, M):
    return HeadConfig.q_boundary(list(pats[:M]))


def _twod(same, cross, M):
    pr = [[none()] * M for _ in range(M)]
    for a in range(M):
        for b in range(M):
            pr[a][b] = same[a] if a == b else cross[a][b]
    return HeadConfig.two_d(pr)


def _select(dists: Sequence[float], costs: Sequence[float], budget: float) -> int:
    best = -1
    for i, (d, c) in enumerate(zip(dists, costs)):
        if c <= budget and (best < 0 or d < dists[best]):
            best = i
    if best < 0:
        raise ValueError(f"no candidate within the budget {budget} (cheapest {min(costs)})")
    return best


class PatternSearch:
    """Alg.4 over one layer's calibration sample (q [H,S,D], k/v [Hkv,S,D] bf16, labels u8 [S],
    all on the GPU).  `run()` returns per-head configs and a report with every distance / cost."""

    def __init__(self, pb: Problem, q, k, v, labels, space: Optional[Dict] = None,
                 budget_pattern: Pattern = None, frame_stride: int = 256):
        self.pb, self.q, self.k, self.v, self.labels = pb, q, k, v, labels
        self.space = space or search_space(frame_stride)
        self.budget_pattern = budget_pattern or ashape(1024, 4096)
        self.M = pb.n_modalities
        H, S = pb.n_heads, pb.seq_len
        self.o_ref = dense_prefill(pb, q, k, v).float()
        self.rows = {m: (labels == m) for m in range(self.M)}
        self.present = [m for m in range(self.M) if bool(self.rows[m].any())]
        self.ref_norm = {m: self.o_ref[:, self.rows[m]].norm(dim=(1, 2)) for m in self.present}
        self.ref_norm_all = self.o_ref.norm(dim=(1, 2))
        self.n_runs = 0
        self.cost_table: Dict[str, List[int]] = {}

    def _run(self, cfgs: List[HeadConfig]):
        """One pass of the hot path for per-head configs: (O fp32 [H,S,D], tiles per head)."""
        sp = SparsePrefill(self.pb, cfgs, device=self.q.device)
        o = sp(self.q, self.k, self.v, self.labels)
        tiles = sp.head_tiles()
        self.n_runs += 1
        for cfg, t in zip(cfgs, tiles):
            self.cost_table.setdefault(cfg.describe(), [None] * len(cfgs))
        for h, (cfg, t) in enumerate(zip(cfgs, tiles)):
            self.cost_table[cfg.describe()][h] = int(t)
        return o.float(), tiles

    def _dist(self, o, region: Optional[int]):
        """[H] normalised L2 distance of the output rows of a query modality (None: all rows)."""
        if region is None:
            return ((o - self.o_ref).norm(dim=(1, 2)) / self.ref_norm_all.clamp_min(1e-30)).tolist()
        r = self.rows[region]
        return ((o[:, r] - self.o_ref[:, r]).norm(dim=(1, 2)) / self.ref_norm[region].clamp_min(1e-30)).tolist()

    def run(self) -> Tuple[List[HeadConfig], Dict]:
        pb, M, H = self.pb, self.M, self.pb.n_heads
        intra, cross = self.space["intra"], self.space["cross"]
        _, budget = self._run([HeadConfig.no_boundary(self.budget_pattern)] * H)
        rep: Dict = {"budget_tiles": [int(b) for b in budget]}
        # global (No-boundary) candidates
        res_g = [self._run([HeadConfig.no_boundary(c)] * H) for c in intra]
        d_g = [self._dist(o, None) for o, _ in res_g]
        p_global = [intra[_select([d[h] for d in d_g], [t[h] for _, t in res_g], budget[h])] for h in range(H)]
        rep["global"] = dict(dist=d_g, cost=[[int(x) for x in t] for _, t in res_g])
        if len(self.present) <= 1:
            return [HeadConfig.no_boundary(p) for p in p_global], rep
        # phase 1: intra-modality (Q-boundary runs, scored per query modality)
        res_q = [self._run([_q([c] * M, M)] * H) for c in intra]
        p_intra = [[full()] * M for _ in range(H)]
        for m in self.present:
            d = [self._dist(o, m) for o, _ in res_q]
            for h in range(H):
                p_intra[h][m] = intra[_select([x[h] for x in d], [t[h] for _, t in res_q], budget[h])]
            rep[f"intra{m}"] = dict(dist=d)
        # phase 2: cross-modality (2D): same-modality pairs with cross FULL, then the cross pairs
        fullx = [[full()] * M for _ in range(M)]
        res_s = [self._run([_twod([c] * M, fullx, M)] * H) for c in intra]
        p_same = [[full()] * M for _ in range(H)]
        for a in self.present:
            d = [self._dist(o, a) for o, _ in res_s]
            for h in range(H):
                p_same[h][a] = intra[_select([x[h] for x in d], [t[h] for _, t in res_s], budget[h])]
            rep[f"same{a}"] = dict(dist=d)
        res_x = [self._run([_twod(p_same[h], [[c] * M for _ in range(M)], M) for h in range(H)]) for c in cross]
        p_cross = [[[full()] * M for _ in range(M)] for _ in range(H)]
        for a in self.present:
            d = [self._dist(o, a) for o, _ in res_x]
            for h in range(H):
                pick = cross[_select([x[h] for x in d], [t[h] for _, t in res_x], budget[h])]
                for b in range(M):
                    if b != a:
                        p_cross[h][a][b] = pick
            rep[f"cross{a}"] = dict(dist=d)
        # phase 3: inter-modality boundary type, per head end to end
        cands = [[HeadConfig.no_boundary(p_global[h]), _q(p_intra[h], M), _twod(p_same[h], p_cross[h], M)]
                 for h in range(H)]
        res3 = [self._run([cands[h][i] for h in range(H)]) for i in range(3)]
        d3 = [self._dist(o, None) for o, _ in res3]
        out = []
        for h in range(H):
            i = _select([d[h] for d in d3], [t[h] for _, t in res3], budget[h])
            out.append(cands[h][i])
        rep["inter"] = dict(dist=d3, cost=[[int(x) for x in t] for _, t in res3])
        rep["n_runs"] = self.n_runs
        return out, rep


def main():
    import os
    import sys
    import numpy as np
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from synth.workloads import build_workload, small_workload
    from synth.gen import gen_qkv
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", type=int, default=-1, help="-1: a 25K-token LongVILA-shaped calibration sample")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    if args.workload >= 0:
        wl = build_workload(args.workload)
    else:   # calibration sample <= 25K tokens: 96 frames of 256 tokens + text, LongVILA-shaped heads
        wl = build_workload(1)
        from synth.workloads import _segments
        seg = _segments([("T", 64), ("F", 96), ("T", 192)])
        wl.segments = seg
        wl.problem = Problem(28, 4, sum(n for _, n in seg), 128, n_modalities=2)
    d = gen_qkv(wl, seed=0)
    pb = wl.problem
    q, k, v = d["q"].cuda(), d["k"].cuda(), d["v"].cuda()
    lab = torch.from_numpy(np.ascontiguousarray(d["labels"])).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ps = PatternSearch(pb, q, k, v, lab)
    cfgs, rep = ps.run()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if args.out:
        save_head_configs(args.out, cfgs, meta={"workload": wl.name, "seq_len": pb.seq_len, "search_s": wall,
                                                "budget": "ashape(1024,4096) tiles"})
    print(json.dumps({"search": "Alg.4 kernel-aware", "workload": wl.name, "seq_len": pb.seq_len, "heads": pb.n_heads,
                      "runs": rep["n_runs"], "wall_s": wall, "paper_A100_s": 900,
                      "picked": [c.describe() for c in cfgs]}))


if __name__ == "__main__":
    main()
