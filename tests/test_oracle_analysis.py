"""Pins for the analysis-metric oracle (oracle/analysis.py) -- CPU only:
closed forms (uniform attention -> ceil(target * n) keys; a one-hot row -> 1 key), brute force over
subsets on tiny rows, and recall = exp(LSE_sparse - LSE_dense) (masked-attention oracle)."""
import itertools

import numpy as np

from oracle.analysis import topk_coverage, attention_recall, causal_probs
from oracle.attention import masked_attention


def test_uniform_and_one_hot_closed_forms():
    S, D = 40, 8
    q = np.zeros((S, D))
    k = np.random.default_rng(0).standard_normal((S, D))
    fr, cnt = topk_coverage(q, k, [9, 39], 0.5, target=0.95)      # q = 0: uniform over i + 1 keys
    assert cnt.tolist() == [int(np.ceil(0.95 * 10)), int(np.ceil(0.95 * 40))]
    k2 = np.zeros((S, D)); k2[7, 0] = 1.0
    q2 = np.zeros((S, D)); q2[:, 0] = 100.0
    _, c2 = topk_coverage(q2, k2, [20], 1.0, target=0.95)           # one dominant key
    assert c2.tolist() == [1]


def test_bruteforce_minimal_subset():
    rng = np.random.default_rng(1)
    for _ in range(30):
        S, D = int(rng.integers(2, 11)), 4
        q, k = rng.standard_normal((S, D)), rng.standard_normal((S, D))
        i = S - 1
        t = float(rng.uniform(0.3, 0.99))
        _, c = topk_coverage(q, k, [i], 0.7, target=t)
        p = causal_probs(q[i], k, i, 0.7)
        best = min(len(sub) for r in range(1, S + 1) for sub in itertools.combinations(range(S), r)
                   if p[list(sub)].sum() >= t - 1e-15)
        assert c[0] == best


def test_recall_equals_lse_difference():
    rng = np.random.default_rng(2)
    S, D = 30, 8
    q, k, v = (rng.standard_normal((S, D)) for _ in range(3))
    causal = np.tril(np.ones((S, S), dtype=bool))
    M = causal & (rng.random((S, S)) < 0.4)
    M[np.arange(S), np.arange(S)] = True
    _, lse_s, _ = masked_attention(q, k, v, M, 0.3)
    _, lse_d, _ = masked_attention(q, k, v, causal, 0.3)
    rec = attention_recall(q, k, M, np.arange(S), 0.3)
    np.testing.assert_allclose(rec, np.exp(lse_s - lse_d), rtol=1e-12)
