"""GPU parity of the analysis metrics against oracle/analysis.py: top-k coverage
counts within one key of the fp64 oracle (the fp32 probabilities may move the crossing of the
target by one key), attention recall of the sparse index within 2e-3 (LSE tolerance), and index
reuse (estimate on one input, attend on another) lowers the recall of a planted grid head."""
import numpy as np
import pytest
import torch

from synth.config import HeadConfig, grid, ashape, vslash
from synth.workloads import small_workload
from synth.gen import gen_qkv
from oracle.analysis import topk_coverage as o_cov, attention_recall as o_rec
from oracle.estimate import estimate_head
from oracle.masks import head_mask_rows
from oracle.modality import modality_groups

pytestmark = pytest.mark.gpu


def test_topk_coverage_matches_oracle():
    from paper_2504_16083_b200.analysis import topk_coverage
    heads = [HeadConfig.no_boundary(grid(256, True, True, False)), HeadConfig.no_boundary(ashape(64, 256))]
    wl = small_workload(S_frames=10, text=100, H=2, Hkv=1, D=64, heads=heads)
    d = gen_qkv(wl, seed=4)
    pb = wl.problem
    rows = np.array([0, 1, 5, 130, 777, 1500, pb.seq_len - 1])
    fr = topk_coverage(pb, d["q"].cuda(), d["k"].cuda(), torch.from_numpy(rows), 0.95).cpu().numpy()
    for h in range(2):
        ofr, ocnt = o_cov(d["q"][h].double().numpy(), d["k"][0].double().numpy(), rows, pb.tau, 0.95)
        cnt = np.rint(fr[h] * (rows + 1)).astype(int)
        assert (np.abs(cnt - ocnt) <= 1).all(), (h, cnt, ocnt)


def test_recall_and_index_reuse():
    from paper_2504_16083_b200.analysis import attention_recall
    heads = [HeadConfig.no_boundary(grid(256, True, True, False)), HeadConfig.no_boundary(vslash(100, 64))]
    wl = small_workload(S_frames=10, text=100, H=2, Hkv=1, D=64, heads=heads)
    da, db = gen_qkv(wl, seed=5), gen_qkv(wl, seed=6)
    pb = wl.problem
    lab = torch.from_numpy(np.ascontiguousarray(da["labels"])).cuda()
    qa, ka, va = da["q"].cuda(), da["k"].cuda(), da["v"].cuda()
    rec = attention_recall(pb, wl.heads, qa, ka, va, lab).cpu().numpy()
    _, rho, _ = modality_groups(da["labels"], pb.n_modalities)
    rows = np.arange(0, pb.seq_len, 7)
    for h in range(2):
        q, k = da["q"][h].double().numpy(), da["k"][0].double().numpy()
        idx = estimate_head(pb, wl.heads[h], q, k, da["labels"])
        M = head_mask_rows(wl.heads[h].boundary, idx, da["labels"], rho, rows, pb.seq_len)
        orec = o_rec(q, k, M, rows, pb.tau)
        assert np.abs(rec[h, rows] - orec).max() <= 2e-3, (h, np.abs(rec[h, rows] - orec).max())
    # reuse: B attended with A's index
    qb, kb, vb = db["q"].cuda(), db["k"].cuda(), db["v"].cuda()
    own = attention_recall(pb, wl.heads, qb, kb, vb, lab).mean(dim=1)
    reuse = attention_recall(pb, wl.heads, qb, kb, vb, lab, index_from=(qa, ka, lab)).mean(dim=1)
    assert torch.isfinite(reuse).all() and float(reuse[0]) < float(own[0]), (own, reuse)   # planted grid head
