"""Oracle end-to-end pins: all-FULL configs reduce to dense attention; the
fingerprints of a FULL head are the closed forms count = i+1, sum j = i(i+1)/2."""
import numpy as np

from synth.config import HeadConfig, full, grid
from synth.workloads import small_workload
from synth.gen import gen_qkv
from oracle.pipeline import run_head, sample_rows
from oracle.attention import dense_causal_attention


def test_full_head_equals_dense_and_closed_form_fingerprints():
    wl = small_workload(S_frames=2, text=32, H=1, Hkv=1, D=32, heads=[HeadConfig.no_boundary(full())])
    d = gen_qkv(wl, seed=0)
    q, k, v = (d[x][0].double().numpy() for x in ("q", "k", "v"))
    r = run_head(wl.problem, wl.heads[0], q, k, v, d["labels"])
    O, lse, _ = dense_causal_attention(q, k, v, wl.problem.tau)
    np.testing.assert_allclose(r["O"], O, rtol=1e-10, atol=1e-12)
    i = np.arange(q.shape[0])
    assert (r["count"] == i + 1).all()
    assert (r["sumj"].astype(np.int64) == i * (i + 1) // 2).all()
    assert (r["sumj2"].astype(np.int64) == i * (i + 1) * (2 * i + 1) // 6).all()   # sum_{j<=i} j^2


def test_sampled_rows_match_full_rows():
    wl = small_workload(S_frames=4, text=64, H=1, Hkv=1, D=32)
    d = gen_qkv(wl, seed=1)
    q, k, v = (d[x][0].double().numpy() for x in ("q", "k", "v"))
    full_r = run_head(wl.problem, wl.heads[0], q, k, v, d["labels"])
    rows = sample_rows(wl.problem, d["labels"], full_r["index"], n_random=50)
    part = run_head(wl.problem, wl.heads[0], q, k, v, d["labels"], rows=rows, index=full_r["index"])
    np.testing.assert_allclose(part["O"], full_r["O"][rows], rtol=1e-12, atol=1e-14)
    assert (part["count"] == full_r["count"][rows]).all()


def test_hline_rows_are_the_full_rows():
    """hline_rows (SURVEY §8c O6 sample) = exactly the rows whose admitted set is the whole
    causal row of the pattern's coordinate system (grid h only, no sink, local 1):
    No-boundary count = i + 1; 2D rank coordinates count = rho(i) + 1 (cross pairs NONE)."""
    from oracle.pipeline import hline_rows
    from oracle.masks import head_mask_rows
    from oracle.modality import modality_groups
    from synth.config import KIND_GRID, KIND_NONE, BND_NONE, BND_2D
    rng = np.random.default_rng(0)
    S = 90
    lab = (rng.random(S) < 0.4).astype(np.uint8)
    _, rho, _ = modality_groups(lab, 2)
    g = dict(kind=KIND_GRID, s=7, p=3, h=True, v=False, sl=False, sink=0, local=1)
    M = head_mask_rows(BND_NONE, dict(intra=[g]), lab, rho, np.arange(S), S)
    full = np.nonzero(M.sum(1) == np.arange(S) + 1)[0]
    assert sorted(set(full.tolist()) - {0}) == sorted(set(hline_rows(BND_NONE, dict(intra=[g]), lab, rho).tolist()) - {0})
    idx = dict(pair=[[g, dict(kind=KIND_NONE)], [dict(kind=KIND_NONE), dict(g, s=5, p=1)]])
    M = head_mask_rows(BND_2D, idx, lab, rho, np.arange(S), S)
    full = np.nonzero((M.sum(1) == rho + 1) & (rho > 0))[0]
    want = hline_rows(BND_2D, idx, lab, rho)
    assert sorted(full.tolist()) == sorted(x for x in want.tolist() if rho[x] > 0)
    assert all(rho[x] % (7 if lab[x] == 0 else 5) == (3 if lab[x] == 0 else 1) for x in want)
