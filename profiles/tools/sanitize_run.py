"""Small end-to-end runs of the hot path for compute-sanitizer (tiny config + a ragged 3.3K mixed
config with every pattern kind and boundary type, D = 64 and 128)."""
import os
import sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_2504_16083_b200 as mmi
from synth.config import HeadConfig, grid, ashape, vslash, full, none, trishape, sf_fixed, sf_strided
from synth.workloads import build_workload, small_workload, _qwen_heads
from synth.gen import gen_qkv


def run(wl, seed):
    d = gen_qkv(wl, seed=seed)
    pb = wl.problem
    q, k, v = d["q"].cuda(), d["k"].cuda(), d["v"].cuda()
    lab = torch.from_numpy(np.ascontiguousarray(d["labels"])).cuda()
    sp = mmi.SparsePrefill(pb, wl.heads)
    lse = torch.empty(pb.n_heads, pb.seq_len, device="cuda")
    o = sp(q, k, v, lab, lse=lse)
    fp = torch.zeros((pb.n_heads, pb.seq_len, 3), dtype=torch.int64, device="cuda")
    mmi.mmi_sparse_fingerprint(pb, wl.heads, sp.ws, q, k, v, fp)
    od = mmi.dense_prefill(pb, q, k, v)
    torch.cuda.synchronize()
    assert sp.flags() == 0
    print(wl.name, pb.seq_len, "finite", bool(torch.isfinite(o.float()).all()), bool(torch.isfinite(od.float()).all()))


run(build_workload(0), 0)
if len(sys.argv) > 1 and sys.argv[1] == "tiny":
    print("sanitize run ok (tiny)")
    sys.exit(0)
heads = [HeadConfig.no_boundary(grid(256, True, True, True)), HeadConfig.no_boundary(grid(0, True, True, True)),
         HeadConfig.no_boundary(ashape(64, 300)), HeadConfig.no_boundary(vslash(100, 64)),
         HeadConfig.no_boundary(trishape(16, 128, 200)), HeadConfig.no_boundary(sf_fixed(256, 256)),
         HeadConfig.no_boundary(sf_strided(64, 7)), HeadConfig.no_boundary(full())]
for D in (64, 128):
    run(small_workload(S_frames=12, text=100, H=len(heads), Hkv=2, D=D, heads=heads), 1)
run(small_workload(S_frames=3, interleave=3, text_len=200, H=4, Hkv=2, D=128, heads=_qwen_heads(4)), 2)
print("sanitize run ok")
