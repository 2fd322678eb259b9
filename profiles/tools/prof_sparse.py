import sys, os; sys.path.insert(0,'.')
import torch, numpy as np
from synth.workloads import build_workload
from synth.gen import gen_qkv
import paper_2504_16083_b200 as mmi
wl = build_workload(int(sys.argv[1]) if len(sys.argv)>1 else 1)
d = gen_qkv(wl, seed=0)
pb = wl.problem
q,k,v = d['q'].cuda(), d['k'].cuda(), d['v'].cuda()
lab = torch.from_numpy(np.ascontiguousarray(d['labels'])).cuda()
sp = mmi.SparsePrefill(pb, wl.heads)
o = torch.empty_like(q)
for _ in range(3): sp(q,k,v,lab,o=o)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
sp(q,k,v,lab,o=o)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", flush=True)
