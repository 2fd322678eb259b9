"""Full-size GPU parity at BASELINE.json sizes, in the launch configuration
bench.py times (whole layer, all heads, one SparsePrefill call).

EVERY head of every config is checked: index sets bit-exact vs the oracle's own
estimate (near-ties reported), and on a seeded row sample the admitted-key
fingerprints are exact and O / LSE are within the north_star tolerance of the
fp64 oracle (run with its own index; gpu_harness.check_head).  One head per
boundary / pattern type additionally gets the full SURVEY §8c O6 sample: every
modality boundary +- 8 rows and every horizontal-line row."""
import numpy as np
import pytest

from synth.config import KIND_GRID, BND_Q, BND_2D
from synth.workloads import build_workload
from synth.gen import gen_qkv
from oracle.pipeline import sample_rows
from gpu_harness import run_gpu, check_head, gpu_index_as_oracle, assert_head

pytestmark = pytest.mark.gpu


def _light_rows(S, h, n_random):
    rng = np.random.default_rng(1000 + h)
    return np.unique(np.concatenate([np.arange(64), np.arange(S - 64, S), rng.integers(0, S, n_random)]))


def _full_rows(wl, d, g, h, n_random=128, thin=1):
    """SURVEY §8c O6 sample; thin > 1 keeps every thin-th boundary window / h-line row (oracle time
    at 512K-1M)."""
    idx = gpu_index_as_oracle(wl.heads[h], g["exp"][h], wl.problem.n_modalities, wl.problem.seq_len)
    rows = sample_rows(wl.problem, d["labels"], idx, seed=h, n_random=n_random, boundary=wl.heads[h].boundary)
    if thin > 1:
        light = _light_rows(wl.problem.seq_len, h, n_random)
        rows = np.union1d(rows[::thin], light)
    return rows


def _designated(wl):
    """First head of each distinct boundary type / pattern description."""
    seen, out = set(), []
    for h, c in enumerate(wl.heads):
        key = c.describe().split(",sink")[0]
        if key not in seen:
            seen.add(key)
            out.append(h)
    return out


def _run_config(cfg, n_random, full_heads, thin=None):
    wl = build_workload(cfg)
    d = gen_qkv(wl, seed=cfg)
    g = run_gpu(wl, d)
    S = wl.problem.seq_len
    report = []
    for h in range(wl.problem.n_heads):
        rows = _full_rows(wl, d, g, h, thin=(thin or {}).get(h, 1)) if h in full_heads else _light_rows(S, h, n_random)
        res = check_head(wl, d, g, h, rows=rows)
        report.append(res)
        assert_head(res)
    near = sum(r["index"]["near"] for r in report)
    print(f"config {cfg}: {len(report)} heads, {sum(r['rows_checked'] for r in report)} rows, near-ties {near}, "
          f"max err {max(r['max_err'] for r in report):.4f}, max lse err {max(r['lse_err'] for r in report):.2e}")


@pytest.mark.parametrize("cfg", [1, 2, 3])
def test_fullsize_config(cfg):
    wl = build_workload(cfg)
    full = _designated(wl)
    thin = None
    if cfg == 3:
        # one Q-boundary head with every one of the 1024 modality boundaries (+-8 rows) and one
        # 2D-boundary head with every 4th row of that sample (oracle time)
        full = full[:2]
        thin = {full[1]: 4}
    _run_config(cfg, n_random=64, full_heads=set(full), thin=thin)


@pytest.mark.slow
def test_fullsize_1m_sampled():
    """BASELINE configs[4] (LongVILA-shaped, 1M tokens) in the bench's launch configuration:
    every head on sampled rows; the grid head with h-lines (head 0) on every 4th of its 4096
    h-line rows (each a whole causal row of up to 1M keys: oracle time)."""
    _run_config(4, n_random=32, full_heads={0}, thin={0: 4})
