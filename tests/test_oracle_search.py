"""Pins for the oracle of the offline search (Alg.4; oracle/search.py) -- CPU only.

The rule is pinned by special cases and properties: with an unlimited budget and FULL among the
candidates FULL wins with distance 0; the selection is the exhaustive in-budget argmin with
first-candidate tie-break; enlarging the budget never increases the winner's distance; on a
planted grid head the grid candidate beats A-shape / vertical-slash at equal budget."""
import numpy as np
import pytest

from synth.config import HeadConfig, full, grid, ashape, vslash, none, KIND_GRID, KIND_FULL
from synth.workloads import small_workload
from synth.gen import gen_qkv
from oracle.search import select, distance, search_head, search_space


def test_select_rule_properties():
    rng = np.random.default_rng(0)
    for _ in range(300):
        n = int(rng.integers(1, 12))
        d = list(np.round(rng.random(n), 1))          # many exact ties
        c = list(rng.integers(0, 10, n))
        b = int(rng.integers(min(c), 12))
        i = select(d, c, b)
        ok = [j for j in range(n) if c[j] <= b]
        assert c[i] <= b and d[i] == min(d[j] for j in ok) and i == min(j for j in ok if d[j] == d[i])
        if b + 1 <= 12:                               # monotone in the budget
            assert d[select(d, c, b + 1)] <= d[i]
    with pytest.raises(ValueError):
        select([0.1, 0.2], [5, 6], 4)


def test_distance_closed_forms():
    O = np.ones((4, 3))
    assert distance(O, O, np.arange(4)) == 0.0
    assert abs(distance(2 * O, O, np.arange(4)) - 1.0) < 1e-15
    assert distance(O, O, np.array([], dtype=np.int64)) == 0.0


def _wl(heads, S_frames=4, text=64):
    return small_workload(S_frames=S_frames, text=text, H=len(heads), Hkv=1, D=32, heads=heads)


def test_full_candidate_wins_unlimited_budget():
    wl = _wl([HeadConfig.no_boundary(grid(256, True, True, False))])
    d = gen_qkv(wl, seed=0)
    q, k, v = (d[x][0].double().numpy() for x in ("q", "k", "v"))
    space = dict(intra=[ashape(16, 64), grid(256, True, True, False), full()], cross=[none(), full()])
    lab = np.zeros_like(d["labels"])                    # one modality -> No-boundary forced
    wl.problem.__class__  # noqa: B018
    cfg, rep = search_head(wl.problem, q, k, v, lab, space, cost=lambda c: 0, budget=1)
    assert cfg.intra[0].kind == KIND_FULL and min(rep["global"]["dist"]) < 1e-12


def test_planted_grid_head_picks_grid():
    """Planted frame-stride grid head (synth generator): at equal cost the grid candidate has the
    smallest output distance among A-shape / vertical-slash / grid."""
    wl = _wl([HeadConfig.no_boundary(grid(256, True, True, False))], S_frames=6)
    d = gen_qkv(wl, seed=1)
    q, k, v = (d[x][0].double().numpy() for x in ("q", "k", "v"))
    lab = np.zeros_like(d["labels"])
    space = dict(intra=[ashape(16, 64), vslash(40, 40), grid(256, True, True, False)], cross=[none()])
    cfg, rep = search_head(wl.problem, q, k, v, lab, space, cost=lambda c: 1, budget=1)
    assert cfg.intra[0].kind == KIND_GRID, rep["global"]["dist"]


def test_search_space_matches_table():
    sp = search_space(256)
    assert len(sp["intra"]) == 12 + 3 + 9                     # tab:search_space P:755-781
    assert sum(p.kind == KIND_GRID and p.stride == 256 for p in sp["intra"]) == 6
    assert sum(p.kind == KIND_GRID and p.stride == 0 and p.stride_max == 1024 for p in sp["intra"]) == 6
