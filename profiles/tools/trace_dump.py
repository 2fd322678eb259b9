"""Runs the sparse stage once with an MMI_TRACE build (MMI_LIB=...libmmi_trace.so) and dumps the
per-event SM-clock trace of CTA 0 (region 0 MMA issuer, 1 / 2 first softmax warp of half A / B)
as JSON.  usage: MMI_LIB=... python profiles/tools/trace_dump.py WORKLOAD OUT.json"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from synth.workloads import build_workload
from synth.gen import gen_qkv
import paper_2504_16083_b200 as mmi
from paper_2504_16083_b200.mmi import lib

w = int(sys.argv[1])
wl = build_workload(w)
d = gen_qkv(wl, seed=0)
pb = wl.problem
q, k, v = d['q'].cuda(), d['k'].cuda(), d['v'].cuda()
lab = torch.from_numpy(np.ascontiguousarray(d['labels'])).cuda()
sp = mmi.SparsePrefill(pb, wl.heads)
o = torch.empty_like(q)
for _ in range(2):
    sp(q, k, v, lab, o=o)
sp.sparse(q, k, v, o)
torch.cuda.synchronize()
L = lib()
N = 16384
buf = (ctypes.c_ulonglong * (3 * N))()
n = (ctypes.c_int * 3)()
L.mmi_debug_trace(buf, n)
out = {"workload": w, "n": list(n), "ev": [[int(buf[r * N + i]) for i in range(n[r])] for r in range(3)]}
json.dump(out, open(sys.argv[2], "w"))
print("trace", list(n))
