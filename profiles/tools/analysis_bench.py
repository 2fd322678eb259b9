"""f1 / f3 measurement lines: the offline pattern search on a <= 25K-token calibration
sample (P:747 reports ~15 min on one A100), and the sparsity metrics on the LongVILA-shaped 128K
layer: top-k coverage for 95 % recall on sampled rows, attention recall of each head's
index and of an index reused from another input.  Prints one JSON line per measurement."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from synth.config import Problem
from synth.workloads import build_workload, _segments
from synth.gen import gen_qkv
import paper_2504_16083_b200 as mmi
from paper_2504_16083_b200.search import PatternSearch
from paper_2504_16083_b200.analysis import topk_coverage, attention_recall

# ---- f1: search on a 25K-token calibration sample (LongVILA-shaped heads, 96 frames + text)
wl = build_workload(1)
wl.segments = _segments([("T", 64), ("F", 96), ("T", 192)])
wl.problem = Problem(28, 4, sum(n for _, n in wl.segments), 128, n_modalities=2)
d = gen_qkv(wl, seed=0)
pb = wl.problem
q, k, v = d["q"].cuda(), d["k"].cuda(), d["v"].cuda()
lab = torch.from_numpy(np.ascontiguousarray(d["labels"])).cuda()
ps = PatternSearch(pb, q, k, v, lab)   # warm-up (kernels, plan cache)
torch.cuda.synchronize()
t0 = time.perf_counter()
ps = PatternSearch(pb, q, k, v, lab)
cfgs, rep = ps.run()
torch.cuda.synchronize()
wall = time.perf_counter() - t0
planted = [c.describe() for c in wl.heads]
print(json.dumps({"measurement": "f1 offline pattern search (Alg.4, kernel-aware budget)", "seq_len": pb.seq_len,
                  "heads": pb.n_heads, "candidate_runs": rep["n_runs"], "wall_s": wall, "paper_A100_s": 900,
                  "picked": [c.describe() for c in cfgs], "generator_heads": planted}), flush=True)
del q, k, v, ps
torch.cuda.empty_cache()

# ---- f3: sparsity metrics at 128K
wl = build_workload(1)
d = gen_qkv(wl, seed=1)
d2 = gen_qkv(wl, seed=2)
pb = wl.problem
q, k, v = d["q"].cuda(), d["k"].cuda(), d["v"].cuda()
lab = torch.from_numpy(np.ascontiguousarray(d["labels"])).cuda()
rows = torch.from_numpy(np.sort(np.random.default_rng(0).choice(pb.seq_len, 64, replace=False)).astype(np.int32))
torch.cuda.synchronize()
t0 = time.perf_counter()
cov = topk_coverage(pb, q, k, rows, 0.95)
torch.cuda.synchronize()
t_cov = time.perf_counter() - t0
rec = attention_recall(pb, wl.heads, q, k, v, lab)
q2, k2, v2 = d2["q"].cuda(), d2["k"].cuda(), d2["v"].cuda()
own2 = attention_recall(pb, wl.heads, q2, k2, v2, lab)
reuse = attention_recall(pb, wl.heads, q2, k2, v2, lab, index_from=(q, k, lab))
print(json.dumps({"measurement": "f3 sparsity metrics", "workload": wl.name, "rows_sampled": int(rows.numel()),
                  "topk95_fraction_mean": float(cov.mean()), "topk95_fraction_per_head": cov.mean(1).tolist(),
                  "topk_wall_s": t_cov, "paper_topk95_fraction_VLM": 0.0578,
                  "recall_own_index_mean": float(rec.mean()), "recall_per_head": rec.mean(1).tolist(),
                  "recall_input2_own": float(own2.mean()), "recall_input2_reused_index": float(reuse.mean())}),
      flush=True)
