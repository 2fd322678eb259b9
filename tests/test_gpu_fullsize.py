"""Full-size GPU parity at BASELINE.json sizes, in the launch configuration
bench.py times (whole layer, all heads, one SparsePrefill call).

Per head: index sets bit-exact vs the oracle (near-ties reported), and on a
seeded row sample (first/last rows, modality boundaries, random rows, hline
rows) the admitted-key fingerprints are exact and the attention output is
within the north_star tolerance of the fp64 oracle run with the GPU's index."""
import numpy as np
import pytest

from synth.workloads import build_workload
from synth.gen import gen_qkv
from oracle.pipeline import sample_rows
from gpu_harness import run_gpu, check_head, gpu_index_as_oracle, TOL_MAX, TOL_MEAN

pytestmark = pytest.mark.gpu


def _sample(wl, d, g, h, n_random):
    idx = gpu_index_as_oracle(wl.heads[h], g["exp"][h], wl.problem.n_modalities)
    rows = sample_rows(wl.problem, d["labels"], idx, seed=h, n_random=n_random)
    if rows.size > 512:
        rng = np.random.default_rng(h)
        keep = np.concatenate([rows[:64], rows[-64:], rng.choice(rows[64:-64], 384, replace=False)])
        rows = np.unique(keep)
    return rows


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_fullsize_config(cfg):
    wl = build_workload(cfg)
    d = gen_qkv(wl, seed=cfg)
    g = run_gpu(wl, d)
    H = wl.problem.n_heads
    heads = list(range(H)) if cfg == 1 else list(range(0, H, 3))
    report = []
    for h in heads:
        rows = _sample(wl, d, g, h, n_random=128)
        res = check_head(wl, d, g, h, rows=rows)
        report.append(res)
        assert not res["index"]["mismatch"], res
        assert res["fp_count_ok"] and res["fp_sum_ok"] and res["fp_sum2_ok"], res
        assert res["max_err"] <= TOL_MAX and res["mean_err"] <= TOL_MEAN, res
    near = sum(r["index"]["near"] for r in report)
    print(f"config {cfg}: {len(report)} heads checked, near-ties {near}, "
          f"max err {max(r['max_err'] for r in report):.4f}")


@pytest.mark.slow
def test_fullsize_1m_sampled():
    """BASELINE configs[4] (LongVILA-shaped, 1M tokens) in the bench's launch
    configuration: one head of each pattern type (fixed-stride grid, searched grid,
    grid with slash lines, A-shape), exact index + fingerprints + tolerance on sampled rows."""
    wl = build_workload(4)
    d = gen_qkv(wl, seed=4)
    g = run_gpu(wl, d)
    for h in (0, 1, 2, 3):
        rows = _sample(wl, d, g, h, n_random=64)
        if rows.size > 192:
            rng = np.random.default_rng(h)
            rows = np.unique(np.concatenate([rows[:32], rows[-32:], rng.choice(rows[32:-32], 128, replace=False)]))
        res = check_head(wl, d, g, h, rows=rows)
        assert not res["index"]["mismatch"], res
        assert res["fp_count_ok"] and res["fp_sum_ok"] and res["fp_sum2_ok"], res
        assert res["max_err"] <= TOL_MAX and res["mean_err"] <= TOL_MEAN, res
