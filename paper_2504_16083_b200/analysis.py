"""Attention-sparsity analysis on the GPU: offline
measurement tooling around the C ABI, not part of the hot path.

  * top-k coverage    mmi_topk_coverage (C ABI kernel): fraction of keys carrying `target` of the
                      causal attention mass per sampled row (5.78 % for 95 % in VLMs);
  * attention recall  of a sparse index: exp(LSE_sparse - LSE_dense) per row, the attention mass
                      its admitted keys carry (LSEs from mmi_sparse_prefill / mmi_dense_prefill);
  * index reuse       the recall on input B of the index estimated on input A ("reusing
                      top-k indices ... across different contexts leads to a significant drop").
"""
from __future__ import annotations

from typing import List, Optional

import torch

from synth.config import HeadConfig, Problem
from .mmi import SparsePrefill, dense_prefill, mmi_topk_coverage


def topk_coverage(pb: Problem, q, k, rows, target: float = 0.95) -> torch.Tensor:
    rows = rows.to(device=q.device, dtype=torch.int32).contiguous()
    return mmi_topk_coverage(pb, q, k, rows, target)


def attention_recall(pb: Problem, cfgs: List[HeadConfig], q, k, v, labels,
                     index_from: Optional[tuple] = None) -> torch.Tensor:
    """[H, S] recall of the sparse index of `cfgs` on (q, k, v).  index_from = (q_a, k_a, labels_a):
    estimate the index on another input first and reuse it on (q, k, v) (index reuse)."""
    sp = SparsePrefill(pb, cfgs, device=q.device)
    lse_s = torch.empty((pb.n_heads, pb.seq_len), dtype=torch.float32, device=q.device)
    o = torch.empty((pb.n_heads, pb.seq_len, pb.head_dim), dtype=torch.bfloat16, device=q.device)
    if index_from is None:
        sp.estimate(q, k, labels)
    else:
        sp.estimate(*index_from)
    sp.permute(q, k, v)
    sp.sparse(q, k, v, o, lse_s)
    sp.unpermute(o, lse_s)
    lse_d = torch.empty_like(lse_s)
    dense_prefill(pb, q, k, v, lse=lse_d)
    return torch.exp(lse_s - lse_d)
