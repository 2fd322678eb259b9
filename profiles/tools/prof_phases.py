"""Times the sparse attention stage (and optionally the dense comparator) with the library named
by MMI_LIB; for MMI_PROF builds also prints the per-phase SM-clock counters of the MMA issuer and
softmax warps.  usage: MMI_LIB=... python profiles/tools/prof_phases.py WORKLOAD [dense]"""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from synth.workloads import build_workload
from synth.gen import gen_qkv
import paper_2504_16083_b200 as mmi
from paper_2504_16083_b200.mmi import lib

w = int(sys.argv[1]) if len(sys.argv) > 1 else 1
wl = build_workload(w)
d = gen_qkv(wl, seed=0)
pb = wl.problem
q, k, v = d['q'].cuda(), d['k'].cuda(), d['v'].cuda()
lab = torch.from_numpy(np.ascontiguousarray(d['labels'])).cuda()
sp = mmi.SparsePrefill(pb, wl.heads)
o = torch.empty_like(q)
for _ in range(3):
    sp(q, k, v, lab, o=o)
torch.cuda.synchronize()
L = lib()
prof = getattr(L, "mmi_debug_prof", None) if hasattr(L, "mmi_debug_prof") else None
buf = (ctypes.c_ulonglong * 32)()
if prof:
    prof(buf, 1)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sp.sparse(q, k, v, o); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
lab_ = lab
te = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); sp.estimate(q, k, lab_); e1.record(); torch.cuda.synchronize()
    te.append(e0.elapsed_time(e1))
tiles = sp.total_tiles()
import struct
from paper_2504_16083_b200.mmi import mmi_export_index
n_items = sum(mmi_export_index(pb, sp.cfgs, sp.ws, h).tolist()[-4] for h in range(pb.n_heads))
ms = float(np.median(ts))
out = {"lib": os.environ.get("MMI_LIB", "libmmi.so"), "workload": w, "sparse_ms": ms, "estimate_ms": float(np.median(te)), "tiles": tiles, "items": n_items,
       "tflops": tiles * 4 * 128 * 128 * pb.head_dim / ms / 1e9}
if prof:
    prof(buf, 1)
    names = ["mma_tot", "mma_wait_p", "mma_wait_k", "mma_wait_v", "mma_wait_q", "mma_wait_o", "mma_nt", "",
             "sm_tot", "sm_wait_s", "sm_ld", "sm_mask", "sm_softmax", "sm_rescale", "sm_pstore", "sm_epi",
             "sm_nsub", "sm_nresc", "sm_fetch", "sm_item", "sm_mword", "sm_epi_wait", "sm_epi_ld"]
    tot = {n: buf[i] for i, n in enumerate(names) if n}
    out["prof_frac"] = {n: round(tot[n] / max(tot["mma_tot" if n.startswith("mma") else "sm_tot"], 1), 4)
                        for n in tot if not n.endswith("tot") and n not in ("mma_nt", "sm_nsub", "sm_nresc")}
    out["prof_counts"] = {n: tot[n] for n in ("mma_nt", "sm_nsub", "sm_nresc")}
if len(sys.argv) > 2 and sys.argv[2] == "dense":
    od = torch.empty_like(q)
    for _ in range(2):
        mmi.dense_prefill(pb, q, k, v, o=od)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); mmi.dense_prefill(pb, q, k, v, o=od); e1.record(); torch.cuda.synchronize()
    dms = e0.elapsed_time(e1)
    S = pb.seq_len; nb = (S + 127) // 128
    out["dense_ms"] = dms
    out["dense_tflops"] = 4 * pb.head_dim * pb.n_heads * S * (S + 1) / 2 / dms / 1e9
print(json.dumps(out))
