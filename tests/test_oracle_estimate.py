"""Pins for oracle O2/O3 (slab estimate, VS top-k, grid fold) — CPU only.

The selection RULE itself (readings C5-C7, C15) is "parity unpinned" by the
paper; what is pinned here: the slab equals the last rows of the dense
attention matrix (library softmax), the reductions equal explicit loops, the
selections equal brute-force enumeration of the stated rule, and planted
structure is recovered (SPEC S:237, S:246-247, S:261, S:611 analogues).
"""
import numpy as np
import pytest
import torch

from synth.config import HeadConfig, Problem, grid, vslash
from synth.workloads import small_workload, build_workload
from synth.gen import gen_qkv
from oracle.estimate import (slab_attention, column_mass, diagonal_mass, diagonal_mass_ranked,
                             select_vs, grid_search, estimate_head, slab_rows)
from oracle.modality import modality_groups


def test_slab_is_last_rows_of_dense_attention():
    rng = np.random.default_rng(0)
    S, D = 90, 16
    q, k = rng.standard_normal((S, D)), rng.standard_normal((S, D))
    R = slab_rows(np.arange(S), 64)
    A = slab_attention(q[R], k, R, 0.25)
    z = torch.from_numpy(q @ k.T * 0.25)
    z = z.masked_fill(torch.triu(torch.ones(S, S, dtype=torch.bool), 1), float("-inf"))
    full = torch.softmax(z, dim=-1).numpy()
    np.testing.assert_allclose(A, full[R], rtol=1e-13, atol=1e-15)
    # last_q = S -> whole matrix
    A2 = slab_attention(q, k, np.arange(S), 0.25)
    np.testing.assert_allclose(A2, full, rtol=1e-13, atol=1e-15)


def test_column_and_diagonal_mass_loops():
    rng = np.random.default_rng(1)
    S = 40
    rows = np.array([3, 10, 11, 12, 30, 39])
    A = rng.random((rows.size, S))
    c = column_mass(A)
    dg = diagonal_mass(A, rows)
    for j in range(S):
        assert abs(c[j] - sum(A[r, j] for r in range(rows.size))) < 1e-12
    for o in range(S):
        want = sum(A[r, rows[r] - o] for r in range(rows.size) if rows[r] - o >= 0)
        assert abs(dg[o] - want) < 1e-12
    # rank coordinates (2D same-modality pair)
    lab = (rng.random(S) < 0.5).astype(np.uint8)
    P, rho, _ = modality_groups(lab, 2)
    Pa = P[0]
    rows_a = Pa[-5:]
    Aa = rng.random((rows_a.size, S))
    dga = diagonal_mass_ranked(Aa, rows_a, Pa, rho)
    for o in range(Pa.size):
        want = sum(Aa[r, Pa[rho[rows_a[r]] - o]] for r in range(rows_a.size) if rho[rows_a[r]] - o >= 0)
        assert abs(dga[o] - want) < 1e-12


def test_topk_bruteforce_and_planted():
    rng = np.random.default_rng(2)
    for _ in range(20):
        S = int(rng.integers(5, 200))
        c = np.round(rng.random(S), 2)           # many exact ties
        dg = np.round(rng.random(S), 2)
        nv, ns = int(rng.integers(1, 12)), int(rng.integers(1, 12))
        jmax = int(rng.integers(0, S))
        out = select_vs(c, dg, nv, ns, jmax, jmax)
        cand = [j for j in range(jmax + 1) if j != 0]
        want_v = sorted({0} | set(sorted(cand, key=lambda j: (-c[j], j))[:nv - 1]))
        want_s = sorted({0} | set(sorted(cand, key=lambda o: (-dg[o], o))[:ns - 1]))
        assert out["V"].tolist() == want_v
        assert out["Sl"].tolist() == want_s
    # planted: attention one-hot on column 5 / offset 7 ranks them first
    S = 64
    rows = np.arange(48, 64)
    A = np.full((rows.size, S), 1e-4)
    A[:, 5] = 1.0
    for r, pr in enumerate(rows):
        A[r, pr - 7] += 0.5
    out = select_vs(column_mass(A), diagonal_mass(A, rows), 2, 2, 63, 63)
    assert out["V"].tolist() == [0, 5] and out["Sl"].tolist() == [0, 7]


def test_grid_fold_bruteforce():
    rng = np.random.default_rng(3)
    for _ in range(10):
        n = int(rng.integers(50, 300))
        c = rng.random(n)
        lo, hi = int(rng.integers(0, 10)), int(rng.integers(40, n))
        cands = list(range(2, 25))
        g = grid_search(c, lo, hi, cands)
        N = hi - lo
        T = sum(c[lo:hi])
        best = None
        for s in cands:
            if N < s:
                continue
            for p in range(s):
                m = sum(c[j] for j in range(lo, hi) if j % s == p)
                cnt = sum(1 for j in range(lo, hi) if j % s == p)
                J = m - cnt * T / N
                if best is None or J > best[2] + 1e-12:
                    best = (s, p, J)
        assert (g["s"], g["p"]) == best[:2]
        assert abs(g["J"] - best[2]) < 1e-9


def test_grid_fold_degenerate_and_ties():
    c = np.ones(500)
    g = grid_search(c, 0, 500, [2, 3, 4])          # uniform: all J = 0 -> smaller stride, phase 0
    assert (g["s"], g["p"]) == (2, 0)
    g = grid_search(np.random.default_rng(4).random(100), 0, 100, [1])
    assert (g["s"], g["p"]) == (1, 0)


@pytest.mark.parametrize("s", [2, 3, 7, 16, 64, 255, 256, 512])
def test_grid_planted_column_recovery(s):
    """Planted vertical lines j = p (mod s) with SNR >= 5 are recovered over
    seeds (SPEC S:261 analogue) against candidates [2, 1024].  Under reading C5
    (excess mass over uniform) a divisor s' of s with the same phase class
    captures the same line mass plus zero-mean noise classes, so it can tie
    with s up to noise ("a divisor ... at the weakest gain"):
    every result must be s or such a divisor (the planted lines are always
    covered); prime strides (no divisor candidate) must be recovered exactly.
    Observed exact rates for composite s are recorded in DESIGN.md."""
    ok = 0
    for seed in range(20):
        rng = np.random.default_rng(seed)
        n = 16 * max(s, 64) + 400
        p = int(rng.integers(0, s))
        c = rng.random(n) * 0.2
        c[p::s] += 1.0 + rng.random(c[p::s].size)
        g = grid_search(c, 128, n - 128, list(range(2, 1025)))
        ok += (g["s"], g["p"]) == (s, p)
        assert s % g["s"] == 0 and g["p"] == p % g["s"], (g["s"], g["p"], s, p)
    if all(s % d for d in range(2, s)):
        assert ok == 20


def test_grid_planted_recovery_from_qkv():
    """End to end from planted Q/K geometry (synth generator): the oracle
    recovers the planted (stride, phase) for frame-stride and searched heads."""
    heads = [HeadConfig.no_boundary(grid(256, True, True, False)),
             HeadConfig.no_boundary(grid(0, False, True, False))]
    wl = small_workload(S_frames=24, text=64, H=2, Hkv=1, D=64, heads=heads)
    for seed in range(3):
        d = gen_qkv(wl, seed=seed)
        q = d["q"].double().numpy(); k = d["k"].double().numpy()
        for h in range(2):
            idx = estimate_head(wl.problem, wl.heads[h], q[h], k[0], d["labels"])
            inst = idx["intra"][0]
            assert (inst["s"], inst["p"]) == d["planted"][h][0], (seed, h, inst["s"], inst["p"], d["planted"][h])


def test_tiny_workload_estimate():
    """configs[0] (tiny): one Grid head with frame_stride 256 recovers the planted phase."""
    wl = build_workload(0)
    d = gen_qkv(wl, seed=0)
    idx = estimate_head(wl.problem, wl.heads[0], d["q"][0].double().numpy(),
                        d["k"][0].double().numpy(), d["labels"])
    assert (idx["intra"][0]["s"], idx["intra"][0]["p"]) == d["planted"][0][0]


def test_boundary_heads_planted_recovery():
    """Q-boundary (vision Grid in original coordinates, reading C12) and
    2D-boundary (V->V Grid in vision-rank coordinates, C13) recover the planted
    phase on an interleaved [3 frames][256 text] layout (SURVEY §8d.1 512K
    layout, scaled down)."""
    from synth.workloads import _qwen_heads
    wl = small_workload(S_frames=3, interleave=8, H=2, Hkv=1, D=64, heads=_qwen_heads(2))
    d = gen_qkv(wl, seed=0)
    q = d["q"].double().numpy(); k = d["k"].double().numpy()
    iq = estimate_head(wl.problem, wl.heads[0], q[0], k[0], d["labels"])
    i2 = estimate_head(wl.problem, wl.heads[1], q[1], k[0], d["labels"])
    assert (iq["intra"][0]["s"], iq["intra"][0]["p"]) == d["planted"][0][0]
    assert (i2["pair"][0][0]["s"], i2["pair"][0][0]["p"]) == d["planted"][1][0]
    assert iq["intra"][1]["V"].size == 1000 and iq["intra"][1]["Sl"].size == 2048
    # text rows' VS index only uses columns / offsets up to the text slab's last row
    assert iq["intra"][1]["V"].max() <= iq["slab"][1].max()
