"""Pins for oracle O1/O4 (masks, modality permutation) — CPU only."""
import json
import os

import numpy as np
import pytest

from synth.config import (KIND_NONE, KIND_FULL, KIND_ASHAPE, KIND_VSLASH, KIND_GRID,
                          BND_NONE, BND_Q, BND_2D)
from oracle.masks import head_mask_rows, brute_force_mask, pattern_pred
from oracle.modality import modality_groups, inverse_permutation, residue_permutation
from oracle.attention import fingerprint, masked_attention, dense_causal_attention

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mask_fixtures.json")))
from synth.config import KIND_TRISHAPE, KIND_SF_FIXED, KIND_SF_STRIDED
KINDS = {"none": KIND_NONE, "full": KIND_FULL, "ashape": KIND_ASHAPE, "vslash": KIND_VSLASH, "grid": KIND_GRID,
         "trishape": KIND_TRISHAPE, "sf_fixed": KIND_SF_FIXED, "sf_strided": KIND_SF_STRIDED}


def _inst(d):
    d = dict(d)
    d["kind"] = KINDS[d["kind"]]
    for key in ("V", "Sl"):
        if key in d:
            d[key] = np.array(sorted(d[key]), dtype=np.int64)
    return d


@pytest.mark.parametrize("fx", GOLD["masks"], ids=[f["name"] for f in GOLD["masks"]])
def test_golden_fingerprints(fx):
    S = fx["S"]
    if fx["boundary"] == "none":
        labels = np.zeros(S, dtype=np.uint8)
        index = dict(intra=[_inst(fx["pattern"])])
        bnd, nm = BND_NONE, 1
    elif fx["boundary"] == "q":
        labels = np.array(fx["labels"], dtype=np.uint8)
        index = dict(intra=[_inst(p) for p in fx["intra"]])
        bnd, nm = BND_Q, 2
    else:
        labels = np.array(fx["labels"], dtype=np.uint8)
        index = dict(pair=[[_inst(p) for p in row] for row in fx["pair"]])
        bnd, nm = BND_2D, 2
    _, rho, _ = modality_groups(labels, nm)
    M = head_mask_rows(bnd, index, labels, rho, np.arange(S), S)
    cnt, sj, sj2 = fingerprint(M)
    assert cnt.tolist() == fx["count"]
    assert [int(x) for x in sj] == fx["sumj"]
    if "sumj2" in fx:
        assert [int(x) for x in sj2] == fx["sumj2"]
    # the vectorised builder agrees with the per-element loop
    assert (brute_force_mask(bnd, index, labels, rho, S) == M).all()


def test_golden_permutations():
    for fx in GOLD["permutations"]:
        if "labels" in fx:
            _, _, perm = modality_groups(np.array(fx["labels"]), 2)
        else:
            perm = residue_permutation(fx["S"], fx["s"])
        assert perm.tolist() == fx["perm"]
        inv = inverse_permutation(perm)
        x = np.arange(len(perm)) * 7 + 3
        assert (x[perm][inv] == x).all()      # permute then unpermute = identity


def _causal(S):
    return np.tril(np.ones((S, S), dtype=bool))


@pytest.mark.parametrize("S", [1, 7, 40])
def test_special_cases_reduce_to_full(S):
    """stride 1 -> full causal; sink >= S -> full; VS with
    V = all columns -> full."""
    lab = np.zeros(S, dtype=np.uint8)
    _, rho, _ = modality_groups(lab, 1)
    full = _causal(S)
    for inst in [dict(kind=KIND_GRID, s=1, p=0, h=False, v=True, sl=False, sink=0, local=1),
                 dict(kind=KIND_GRID, s=1, p=0, h=False, v=False, sl=True, sink=0, local=1),
                 dict(kind=KIND_ASHAPE, sink=S, local=1),
                 dict(kind=KIND_ASHAPE, sink=0, local=S),
                 dict(kind=KIND_VSLASH, V=np.arange(S), Sl=np.array([0])),
                 dict(kind=KIND_FULL)]:
        M = head_mask_rows(BND_NONE, dict(intra=[inst]), lab, rho, np.arange(S), S)
        assert (M == full).all(), inst


def test_grid_lines_bruteforce_enumeration():
    """Grid masks match an independent enumeration of stride/phase LINES
    (north_star: 'Grid masks must match a brute-force enumeration of
    stride/phase lines'): build the admitted set as a union of explicit line
    sets, not via the predicate."""
    rng = np.random.default_rng(1)
    for _ in range(30):
        S = int(rng.integers(5, 60))
        s = int(rng.integers(1, 9))
        p = int(rng.integers(0, s))
        h, v, sl = (bool(b) for b in rng.integers(0, 2, 3))
        sink, local = int(rng.integers(0, 4)), int(rng.integers(1, 5))
        want = np.zeros((S, S), dtype=bool)
        for i in range(S):
            for j in range(min(sink, i + 1)):
                want[i, j] = True                              # sink columns
            for j in range(max(0, i - local + 1), i + 1):
                want[i, j] = True                              # local band
        if h:
            for i in range(p, S, s):
                want[i, :i + 1] = True                         # horizontal line rows
        if v:
            for j in range(p, S, s):
                want[j:, j] = True                             # vertical line columns
        if sl:
            for o in range(0, S, s):
                for i in range(o, S):
                    want[i, i - o] = True                      # slash diagonals
        lab = np.zeros(S, dtype=np.uint8)
        _, rho, _ = modality_groups(lab, 1)
        inst = dict(kind=KIND_GRID, s=s, p=p, h=h, v=v, sl=sl, sink=sink, local=local)
        M = head_mask_rows(BND_NONE, dict(intra=[inst]), lab, rho, np.arange(S), S)
        assert (M == want).all()


def test_2d_reduces_to_per_modality_blocks():
    """2D with intra FULL and cross NONE: each modality's rows equal dense causal
    attention on that modality's subsequence alone (north_star 'boundary
    patterns must reduce to per-modality blocks')."""
    rng = np.random.default_rng(2)
    S, D = 50, 8
    lab = (rng.random(S) < 0.4).astype(np.uint8)
    q, k, v = (rng.standard_normal((S, D)) for _ in range(3))
    P, rho, _ = modality_groups(lab, 2)
    index = dict(pair=[[dict(kind=KIND_FULL), dict(kind=KIND_NONE)],
                       [dict(kind=KIND_NONE), dict(kind=KIND_FULL)]])
    M = head_mask_rows(BND_2D, index, lab, rho, np.arange(S), S)
    O, _, _ = masked_attention(q, k, v, M, 0.3)
    for m in range(2):
        Pm = P[m]
        Od, _, _ = dense_causal_attention(q[Pm], k[Pm], v[Pm], 0.3)
        np.testing.assert_allclose(O[Pm], Od, rtol=1e-12, atol=1e-12)


def test_boundary_all_full_equals_dense():
    """Q- or 2D-boundary with all FULL patterns = dense."""
    rng = np.random.default_rng(3)
    S, D = 40, 8
    lab = (rng.random(S) < 0.5).astype(np.uint8)
    _, rho, _ = modality_groups(lab, 2)
    full = _causal(S)
    Mq = head_mask_rows(BND_Q, dict(intra=[dict(kind=KIND_FULL)] * 2), lab, rho, np.arange(S), S)
    M2 = head_mask_rows(BND_2D, dict(pair=[[dict(kind=KIND_FULL)] * 2] * 2), lab, rho, np.arange(S), S)
    assert (Mq == full).all() and (M2 == full).all()


def test_single_modality_2d_equals_no_boundary():
    S = 30
    lab = np.zeros(S, dtype=np.uint8)
    _, rho, _ = modality_groups(lab, 1)
    inst = dict(kind=KIND_GRID, s=5, p=2, h=True, v=True, sl=True, sink=2, local=3)
    a = head_mask_rows(BND_NONE, dict(intra=[inst]), lab, rho, np.arange(S), S)
    b = head_mask_rows(BND_2D, dict(pair=[[inst]]), lab, rho, np.arange(S), S)
    assert (a == b).all()


def test_residue_causality_rule():
    """Residue permutation causality: with i = r_q + s t_q and
    j = r_k + s t_k, j <= i  <=>  t_k <= t_q - [r_k > r_q]."""
    for s in (1, 2, 3, 5, 8):
        for i in range(40):
            for j in range(40):
                rq, tq, rk, tk = i % s, i // s, j % s, j // s
                assert (j <= i) == (tk <= tq - (1 if rk > rq else 0))


def test_static_baseline_patterns_lines_and_special_cases():
    """f3 patterns: vectorised masks == an explicit union of their line / block sets,
    and the degenerate parameters reduce to full causal attention."""
    rng = np.random.default_rng(5)
    for _ in range(40):
        S = int(rng.integers(3, 50))
        lab = np.zeros(S, dtype=np.uint8)
        _, rho, _ = modality_groups(lab, 1)
        l, st, sink, b = int(rng.integers(1, 9)), int(rng.integers(1, 9)), int(rng.integers(0, 4)), int(rng.integers(0, 6))
        want = {k: np.zeros((S, S), dtype=bool) for k in ("tri", "fix", "str")}
        for i in range(S):
            for j in range(i + 1):
                want["tri"][i, j] = j < sink or i - j < l or i >= S - b
        for i in range(S):                       # segments of l keys + every segment's initial key
            want["fix"][i, (i // l) * l:i + 1] = True
            want["fix"][i, 0:i + 1:st] = True
        for i in range(S):                       # local window + dilated diagonals
            want["str"][i, max(0, i - l + 1):i + 1] = True
            for o in range(0, i + 1, st):
                want["str"][i, i - o] = True
        insts = {"tri": dict(kind=KIND_TRISHAPE, sink=sink, local=l, bottom=b, n=S),
                 "fix": dict(kind=KIND_SF_FIXED, local=l, stride=st),
                 "str": dict(kind=KIND_SF_STRIDED, local=l, stride=st)}
        for k, inst in insts.items():
            M = head_mask_rows(BND_NONE, dict(intra=[inst]), lab, rho, np.arange(S), S)
            assert (M == want[k]).all(), (k, S, l, st)
    S = 20
    lab = np.zeros(S, dtype=np.uint8)
    _, rho, _ = modality_groups(lab, 1)
    for inst in [dict(kind=KIND_TRISHAPE, sink=0, local=1, bottom=S, n=S), dict(kind=KIND_SF_FIXED, local=S, stride=7),
                 dict(kind=KIND_SF_STRIDED, local=1, stride=1), dict(kind=KIND_SF_FIXED, local=1, stride=1)]:
        M = head_mask_rows(BND_NONE, dict(intra=[inst]), lab, rho, np.arange(S), S)
        assert (M == _causal(S)).all(), inst
