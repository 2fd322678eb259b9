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


def test_sampled_rows_match_full_rows():
    wl = small_workload(S_frames=4, text=64, H=1, Hkv=1, D=32)
    d = gen_qkv(wl, seed=1)
    q, k, v = (d[x][0].double().numpy() for x in ("q", "k", "v"))
    full_r = run_head(wl.problem, wl.heads[0], q, k, v, d["labels"])
    rows = sample_rows(wl.problem, d["labels"], full_r["index"], n_random=50)
    part = run_head(wl.problem, wl.heads[0], q, k, v, d["labels"], rows=rows, index=full_r["index"])
    np.testing.assert_allclose(part["O"], full_r["O"][rows], rtol=1e-12, atol=1e-14)
    assert (part["count"] == full_r["count"][rows]).all()
