"""GPU parity of permuted NATTEN / DiT neighborhood attention (App. F)
against the fp64 oracle (oracle/natten.py): per-row admitted-key fingerprints exact (the kernel
applies exactly the clamped 3D windows, reading C25), O within the north_star tolerance and LSE
within 2e-3, on ragged grids (extents not multiples of the tile) and several tile shapes."""
import numpy as np
import pytest
import torch

from synth.config import NattenConfig, Problem
from oracle.natten import natten_attention
from oracle.attention import fingerprint
from gpu_harness import TOL_MAX, TOL_MEAN, TOL_LSE

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("nc,H,Hkv,D", [
    (NattenConfig(4, 12, 20, 3, 5, 7, 2, 8, 8), 2, 1, 64),
    (NattenConfig(3, 16, 24, 3, 7, 9, 1, 8, 16), 4, 2, 128),
    (NattenConfig(5, 9, 13, 5, 9, 13, 2, 8, 8), 2, 2, 64),     # window = whole grid: dense bidirectional
    (NattenConfig(1, 40, 40, 1, 11, 11, 1, 8, 16), 2, 1, 128),  # 2D (image) neighborhood
])
def test_natten_vs_oracle(nc, H, Hkv, D):
    from paper_2504_16083_b200 import NattenPrefill
    S = nc.seq_len
    g = torch.Generator().manual_seed(7)
    q = torch.randn(H, S, D, generator=g).to(torch.bfloat16)
    k = torch.randn(Hkv, S, D, generator=g).to(torch.bfloat16)
    v = torch.randn(Hkv, S, D, generator=g).to(torch.bfloat16)
    pb = Problem(H, Hkv, S, D)
    npf = NattenPrefill(pb, nc)
    lse = torch.full((H, S), float("nan"), device="cuda")
    o = npf(q.cuda(), k.cuda(), v.cuda(), lse=lse)
    fp = torch.zeros((H, S, 3), dtype=torch.int64, device="cuda")
    npf.fingerprint(q.cuda(), k.cuda(), v.cuda(), fp)
    torch.cuda.synchronize()
    G = H // Hkv
    for h in range(H):
        O, L, M = natten_attention(nc, q[h].double().numpy(), k[h // G].double().numpy(), v[h // G].double().numpy(),
                                   pb.tau)
        cnt, sj, sj2 = fingerprint(M)
        f = fp[h].cpu().numpy()
        assert (f[:, 0] == cnt).all() and (f[:, 1].astype(np.uint64) == sj).all() and (f[:, 2].astype(np.uint64) == sj2).all()
        err = np.abs(o[h].float().cpu().numpy() - O)
        assert err.max() <= TOL_MAX and err.mean() <= TOL_MEAN, (h, err.max(), err.mean())
        assert np.abs(lse[h].cpu().numpy() - L).max() <= TOL_LSE
