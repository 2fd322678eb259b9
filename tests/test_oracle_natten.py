"""Pins for the NATTEN oracle (oracle/natten.py) -- CPU only."""
import itertools

import numpy as np
import torch

from synth.config import NattenConfig
from oracle.natten import natten_mask_rows, natten_attention
from oracle.attention import fingerprint


def test_hand_fixture_1d():
    """T = Hh = 1, Ww = 6, kw = 3 (clamped windows): x=0,1 -> {0,1,2}; x=2 -> {1,2,3};
    x=3 -> {2,3,4}; x=4,5 -> {3,4,5}."""
    cfg = NattenConfig(1, 1, 6, 1, 1, 3)
    M = natten_mask_rows(cfg, np.arange(6))
    cnt, sj, sj2 = fingerprint(M)
    assert cnt.tolist() == [3] * 6
    assert [int(x) for x in sj] == [3, 3, 6, 9, 12, 12]
    assert [int(x) for x in sj2] == [5, 5, 14, 29, 50, 50]


def test_bruteforce_3d_windows():
    rng = np.random.default_rng(0)
    for _ in range(20):
        T, H, W = (int(x) for x in rng.integers(1, 6, 3))
        kt, kh, kw = int(rng.integers(1, T + 1)), int(rng.integers(1, H + 1)), int(rng.integers(1, W + 1))
        cfg = NattenConfig(T, H, W, kt, kh, kw)
        M = natten_mask_rows(cfg, np.arange(cfg.seq_len))
        want = np.zeros_like(M)
        for (t, y, x) in itertools.product(range(T), range(H), range(W)):
            i = (t * H + y) * W + x
            st = [min(max(c - k // 2, 0), L - k) for c, k, L in ((t, kt, T), (y, kh, H), (x, kw, W))]
            for (a, b, c) in itertools.product(range(st[0], st[0] + kt), range(st[1], st[1] + kh), range(st[2], st[2] + kw)):
                want[i, (a * H + b) * W + c] = True
        assert (M == want).all()
        assert (M.sum(1) == kt * kh * kw).all()            # clamped windows: constant key count


def test_full_window_is_dense_bidirectional_sdpa():
    rng = np.random.default_rng(1)
    cfg = NattenConfig(2, 3, 4, 2, 3, 4)
    S, D = cfg.seq_len, 8
    q, k, v = (rng.standard_normal((S, D)) for _ in range(3))
    O, _, M = natten_attention(cfg, q, k, v, 0.3)
    assert M.all()
    ref = torch.nn.functional.scaled_dot_product_attention(torch.from_numpy(q)[None], torch.from_numpy(k)[None],
                                                           torch.from_numpy(v)[None], scale=0.3)[0].numpy()
    np.testing.assert_allclose(O, ref, rtol=1e-11, atol=1e-12)
