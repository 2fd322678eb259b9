"""Pins for oracle O5/O6 (masked attention, LSE merge) — CPU only."""
import numpy as np
import pytest
import torch

from oracle.attention import masked_attention, dense_causal_attention, merge_partials


def test_dense_matches_torch_sdpa_fp64():
    """Library pin: torch scaled_dot_product_attention(is_causal=True) in fp64."""
    rng = np.random.default_rng(0)
    for S, D in [(1, 4), (37, 16), (130, 64)]:
        q, k, v = (rng.standard_normal((S, D)) for _ in range(3))
        O, lse, _ = dense_causal_attention(q, k, v, 1 / np.sqrt(D))
        ref = torch.nn.functional.scaled_dot_product_attention(
            torch.from_numpy(q)[None], torch.from_numpy(k)[None], torch.from_numpy(v)[None],
            is_causal=True)[0].numpy()
        np.testing.assert_allclose(O, ref, rtol=1e-11, atol=1e-12)
        z = (q @ k.T) / np.sqrt(D)
        z[np.triu_indices(S, 1)] = -np.inf
        np.testing.assert_allclose(lse, np.log(np.exp(z).sum(1)), rtol=1e-12)


def test_closed_forms():
    """S=1 -> v0; q = 0 -> prefix means; diagonal mask -> v."""
    rng = np.random.default_rng(1)
    v = rng.standard_normal((5, 3))
    k = rng.standard_normal((5, 3))
    O, _, _ = dense_causal_attention(np.ones((1, 3)), k[:1], v[:1], 0.5)
    np.testing.assert_array_equal(O[0], v[0])
    O, lse, _ = dense_causal_attention(np.zeros((5, 3)), k, v, 0.5)
    for i in range(5):
        np.testing.assert_allclose(O[i], v[:i + 1].mean(0), rtol=1e-14)
        np.testing.assert_allclose(lse[i], np.log(i + 1), rtol=1e-14)
    O, _, _ = masked_attention(rng.standard_normal((5, 3)), k, v, np.eye(5, dtype=bool), 0.5)
    np.testing.assert_allclose(O, v, rtol=1e-14)


def test_empty_row_zero_flag():
    rng = np.random.default_rng(2)
    q, k, v = (rng.standard_normal((4, 3)) for _ in range(3))
    M = np.tril(np.ones((4, 4), dtype=bool)); M[2] = False
    O, lse, empty = masked_attention(q, k, v, M, 1.0)
    assert empty.tolist() == [False, False, True, False]
    assert (O[2] == 0).all() and np.isneginf(lse[2])


@pytest.mark.parametrize("seed", range(20))
def test_merge_partials_equals_single_pass(seed):
    """merged partials over a random partition of the key range = single pass
    within 1e-10; merge is symmetric; empty is identity."""
    rng = np.random.default_rng(seed)
    S, D = int(rng.integers(2, 80)), 8
    q, k, v = (rng.uniform(-3, 3, (S, D)) for _ in range(3))
    causal = np.tril(np.ones((S, S), dtype=bool))
    part = rng.random((S, S)) < 0.5
    O, lse, _ = masked_attention(q, k, v, causal, 0.4)
    O1, l1, _ = masked_attention(q, k, v, causal & part, 0.4)
    O2, l2, _ = masked_attention(q, k, v, causal & ~part, 0.4)
    Om, lm = merge_partials(O1, l1, O2, l2)
    np.testing.assert_allclose(Om, O, rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(lm, lse, rtol=1e-12)
    Om2, _ = merge_partials(O2, l2, O1, l1)
    np.testing.assert_allclose(Om2, Om, rtol=1e-12, atol=1e-12)
    Oe, le = merge_partials(O, lse, np.zeros_like(O), np.full(S, -np.inf))
    np.testing.assert_allclose(Oe, O, rtol=1e-14, atol=1e-14)
