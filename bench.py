#!/usr/bin/env python
"""Benchmark: one sparse pre-fill attention layer (MMInference hot path) on B200.

A step = one pass of the whole hot path over one layer of synthetic
video-shaped input (+ a9 output all-gather for N > 1):
mmi_estimate_index -> mmi_permute -> mmi_sparse_prefill -> mmi_unpermute.
Default workload: BASELINE.json configs[4] (LongVILA-7B-shaped layer, 1M
tokens, 28 Q / 4 KV heads, D = 128) -- the north_star configuration.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload I] [--impl mmi|reference]

N > 1: one process per GPU.  Launched by torchrun (RANK / WORLD_SIZE set), or
self-launched through torch.distributed.run when `--gpus N` is given without
a WORLD_SIZE.  The layer's heads are sharded by KV-head group;
when N > Hkv the ranks of one group split its heads by computed-tile cost.
Each rank runs the whole pipeline on its heads, then one NCCL
all_gather_into_tensor assembles O on every rank.  Scaling is strong (one
layer, fixed total work).
Timing: CUDA events on the launching stream, barrier + synchronize on both
sides of the K timed steps, max over ranks.  Inputs (Q: 7.5 GB at 1M) are
larger than L2 (126 MB), so no explicit flush between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth.config import KIND_GRID, KIND_VSLASH, KIND_NONE, BND_2D, BND_Q, Problem  # noqa: E402
from synth.workloads import build_workload  # noqa: E402
from synth.gen import gen_qkv  # noqa: E402
from paper_2504_16083_b200.dist import all_ranges, OutputExchange  # noqa: E402

METRIC = "sparse pre-fill attention ms/layer at 128K-1M tokens; speedup vs dense; TC util"
UNIT = "ms/layer"
DEFAULT_WORKLOAD = 4          # BASELINE.json configs[4]: LongVILA-7B-shaped, 1M tokens (north_star)
MUFU_PER_CLK_SM = 16          # ex2 results / clk / SM (measured)
ALU_PER_CLK_SM = 64           # 32-bit integer adds / clk / SM (alu pipe: rt 2 clk per warp per SMSP)
N_SM = 148


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0,
                "_fallback": True}


def _patterns(cfg, M=2):
    if cfg.boundary in (0, 1):
        out = [(cfg.intra[0], None)]
    elif cfg.boundary == BND_Q:
        out = [(cfg.intra[m], m) for m in range(M)]
    else:
        out = [(cfg.pair[a][b], a) for a in range(M) for b in range(M)]
    return [(p, m) for p, m in out if p.kind != KIND_NONE]


def count_launches(heads, fused: int = 1) -> int:
    """Kernels of libmmi.so launched per step (every one is this library's own kernel)."""
    from synth.config import KIND_TRISHAPE, KIND_SF_FIXED, KIND_SF_STRIDED
    pats = [p for c in heads for p, _ in _patterns(c)]
    static = [p for p in pats if p.kind in (KIND_TRISHAPE, KIND_SF_FIXED, KIND_SF_STRIDED)]
    n = 4                                   # modality count / scan / place / pad
    if any(p.kind in (KIND_GRID, KIND_VSLASH) for p in pats):
        n += 4                              # slab rows, pass 1, combine, pass 2
    if any(p.kind == KIND_GRID for p in pats) or static:
        n += 5                              # gather-rank, fold, derive, eval, pick
    if any(p.kind == KIND_VSLASH for p in pats):
        n += 1                              # vs select
    n += 1 + 2 + 1                          # view aliases, views (Q, K), inst params
    n += 1                                  # items fill (static per-slot segment regions: no count, no scan)
    n += 8                                  # LPT sort: 4 radix passes x (histogram, scatter)
    n += 1                                  # items gather
    n += 0 if fused == 3 else (1 if fused == 1 else 2)  # permute gathers (K/V; Q fused into the attention loads)
    n += 1                                  # sparse attention
    # kernel byte copies / fills (util.cu; not copy-engine operations): estimate: device tables,
    # labels; fills of flags, column mass, diagonal mass, VS bitmaps, VS counts, segment counts
    # (every region has at least one word); sparse: scheduler counter, + NaN fill of partial LSEs
    # when rows are merged
    n += 2 + 6
    merged = any((p.kind == KIND_GRID and (p.use_slash or p.use_hline)) or p.kind in (KIND_SF_STRIDED, KIND_TRISHAPE)
                 for p in pats)
    n += 1 + int(merged)
    n += int(any((p.kind == KIND_GRID and p.use_slash) or p.kind == KIND_SF_STRIDED for p in pats))  # LSE merge
    n += int(any((p.kind == KIND_GRID and p.use_hline) or p.kind == KIND_TRISHAPE for p in pats))   # h-row merge
    return n


def estimate_bound(wl, lheads, S, D, sm_mhz, peaks):
    """Algorithmic work of mmi_estimate_index and its time bound:
    slab scores = 2 passes x 2 L keys D FLOP (tensor), 2 passes x L keys exp2 (MUFU);
    grid fold = candidate strides x |W| adds (ALU).  Bound = max(MUFU, tensor) + ALU."""
    slabs = []
    folds = 0
    labels = None
    for c in lheads:
        seen = set()
        for p, m in _patterns(c):
            if p.kind not in (KIND_GRID, KIND_VSLASH):
                continue
            if m not in seen:
                seen.add(m)
                slabs.append(m)
            if p.kind == KIND_GRID:
                ncand = 1 if p.stride > 0 else p.stride_max - p.stride_min + 1
                folds += ncand * max(0, S - 256)
    L = 64
    exps = 2 * L * S * len(slabs)
    flops = 2 * 2 * L * S * D * len(slabs)
    clk = sm_mhz * 1e6
    t_mufu = exps / (MUFU_PER_CLK_SM * N_SM * clk)
    t_tc = flops / (float(peaks["bf16_tflops"]) * 1e12)
    t_alu = folds / (ALU_PER_CLK_SM * N_SM * clk)
    return {"slabs": len(slabs), "exp2": exps, "slab_flops": flops, "fold_adds": folds,
            "bound_ms": (max(t_mufu, t_tc) + t_alu) * 1e3,
            "parts_ms": {"mufu": t_mufu * 1e3, "tensor": t_tc * 1e3, "alu_fold": t_alu * 1e3},
            "clock_mhz": sm_mhz,
            "def": "max(MUFU ex2 at 16/clk/SM, tensor at measured bf16 burst) + fold adds at 64/clk/SM; 148 SMs"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev: int):
        self.dev, self.proc, self.f = dev, None, None

    def start(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.seek(0)
        rows = [r.strip().split(",") for r in self.f.read().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm = [float(r[0]) for r in rows if len(r) >= 6 and r[0].strip().replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 6 and r[1].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 6 for i in range(4) if r[2 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------------ oracle (CPU) timing
def _cores():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count()


def oracle_sample(wl, d, heads, n_rows, seed=0):
    """Times the fp64 oracle (as it stands) on a bounded sample of the workload: the full
    estimation (O2/O3) of each sampled head plus masked attention (O4/O5) on n_rows seeded
    rows; extrapolates to ms/layer = mean over sampled heads x H heads."""
    from oracle.estimate import estimate_head
    from oracle.pipeline import run_head
    pb = wl.problem
    G = pb.n_heads // pb.n_kv_heads
    rng = np.random.default_rng(seed)
    per_head = []
    t_all = time.perf_counter()
    for h in heads:
        qh = d["q"][h].double().numpy()
        kg = d["k"][h // G].double().numpy()
        vg = d["v"][h // G].double().numpy()
        t0 = time.perf_counter()
        idx = estimate_head(pb, wl.heads[h], qh, kg, d["labels"])
        t1 = time.perf_counter()
        rows = np.sort(rng.integers(0, pb.seq_len, size=n_rows))
        run_head(pb, wl.heads[h], qh, kg, vg, d["labels"], rows=rows, index=idx)
        t2 = time.perf_counter()
        per_head.append((t1 - t0) + (t2 - t1) / n_rows * pb.seq_len)
    wall = time.perf_counter() - t_all
    ms_layer = statistics.mean(per_head) * pb.n_heads * 1e3
    sample = (f"heads {list(heads)}: full last-64 estimation + {n_rows} seeded rows of masked fp64 attention each; "
              f"extrapolated to {pb.n_heads} heads x {pb.seq_len} rows")
    return ms_layer, wall, _cores(), sample


def _representative_heads(wl, k=3):
    kinds = {}
    for h, c in enumerate(wl.heads):
        kinds.setdefault(c.describe().split("(")[0] + str(c.intra[0].stride > 0), h)
    return sorted(kinds.values())[:k]


def _sdpa_sanity(q, k, v, G, stream):
    """SURVEY 8(d.3) sanity: the same dense causal layer through torch SDPA's cuDNN backend
    (a library kernel, timed beside the same-build comparator so it is not a strawman)."""
    from torch.nn.attention import sdpa_kernel, SDPBackend
    import torch.nn.functional as F
    out = {}
    qq = q.unsqueeze(0)
    kk = k.repeat_interleave(G, dim=0).unsqueeze(0)
    vv = v.repeat_interleave(G, dim=0).unsqueeze(0)
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION),):
        try:
            with sdpa_kernel([be]):
                if q.shape[1] <= 262144:  # warm-up call (skipped at >= 512K: one call is seconds)
                    F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                F.scaled_dot_product_attention(qq, kk, vv, is_causal=True)
                b.record(stream)
                torch.cuda.synchronize()
                out[name] = a.elapsed_time(b)
        except Exception as ex:  # library backend unavailable for this shape / arch
            out[name] = None
            out[name + "_error"] = str(ex).splitlines()[0][:120] if str(ex) else type(ex).__name__
    del kk, vv
    return out


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _self_launch(n: int) -> int:
    """`--gpus N` without torchrun: re-run this script under torch.distributed.run with N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def plan_ranks(pb, heads, N, dist=None, dev=None, d=None, kv_range=None):
    """Rank ranges.  N <= Hkv: whole KV groups.  N > Hkv: the ranks of a KV group
    split its heads by COMPUTED TILES: every rank of the group builds the group's index once
    (outside the timed region), reads the per-head tile counts, and the counts are max-reduced
    so every rank derives the same split (paper_2504_16083_b200.dist.split_by_cost)."""
    H, Hkv = pb.n_heads, pb.n_kv_heads
    if N <= Hkv:
        return all_ranges(H, Hkv, N), None
    import paper_2504_16083_b200 as mmi
    G = H // Hkv
    kv0, kv1 = kv_range
    gpb = Problem(G * (kv1 - kv0), kv1 - kv0, pb.seq_len, pb.head_dim, pb.n_modalities, pb.last_q, pb.block, pb.scale)
    gheads = heads[kv0 * G:kv1 * G]
    sp = mmi.SparsePrefill(gpb, gheads, device=dev)
    q = d["q"][kv0 * G:kv1 * G].to(dev)
    k = d["k"][kv0:kv1].contiguous().to(dev)
    lab = torch.from_numpy(np.ascontiguousarray(d["labels"])).to(dev)
    sp.estimate(q, k, lab)
    torch.cuda.synchronize()
    cost = torch.zeros(H, dtype=torch.float64, device=dev)
    for i, t in enumerate(sp.head_tiles()):
        cost[kv0 * G + i] = float(t)
    del sp, q, k
    if dist is not None:
        dist.all_reduce(cost, op=dist.ReduceOp.MAX)
    cost = cost.cpu().tolist()
    return all_ranges(H, Hkv, N, cost), cost


def bench_natten(args, rank, local, N):
    """f4 workload (--workload 6): one permuted-NATTEN DiT layer (mmi_natten_prefill), heads sharded
    across ranks (N > 1: each rank its head slice, no collective -- the output stays sharded)."""
    import paper_2504_16083_b200 as mmi
    from synth.workloads import natten_workload
    name, pb0, nc = natten_workload()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    h0, h1 = rank * pb0.n_heads // N, (rank + 1) * pb0.n_heads // N
    pb = Problem(h1 - h0, h1 - h0, pb0.seq_len, pb0.head_dim)
    g = torch.Generator().manual_seed(args.seed + rank)
    S, D = pb.seq_len, pb.head_dim
    q = torch.randn(pb.n_heads, S, D, generator=g).to(torch.bfloat16).to(dev)
    k = torch.randn(pb.n_kv_heads, S, D, generator=g).to(torch.bfloat16).to(dev)
    v = torch.randn(pb.n_kv_heads, S, D, generator=g).to(torch.bfloat16).to(dev)
    npf = mmi.NattenPrefill(pb, nc, device=dev)
    o = torch.empty_like(q)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        npf(q, k, v, o)
    torch.cuda.synchronize()
    fp = torch.zeros((pb.n_heads, S, 3), dtype=torch.int64, device=dev)
    npf.fingerprint(q, k, v, fp)
    admitted = int(fp[:, :, 0].sum().item())
    del fp
    clocks = ClockSampler(local)
    clocks.start()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        npf(q, k, v, o)
    b.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = a.elapsed_time(b) / args.steps
    if N > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    # same-build dense comparator: the same kernel with the window = the whole grid (every tile FULL)
    from synth.config import NattenConfig
    dn = mmi.NattenPrefill(pb, NattenConfig(nc.T, nc.Hh, nc.Ww, nc.T, nc.Hh, nc.Ww, nc.bt, nc.bh, nc.bw), device=dev)
    dn(q, k, v, o)
    torch.cuda.synchronize()
    a.record(stream)
    dn(q, k, v, o)
    b.record(stream)
    torch.cuda.synchronize()
    dense_ms = a.elapsed_time(b)
    peaks = _peaks()
    # computed tiles: live (tile, half) pairs of the index = admitted keys rounded up to whole tiles;
    # reported with the admitted-element FLOPs
    achieved_adm = 4 * D * admitted / (ms * 1e-3) / 1e12
    if rank == 0:
        print(json.dumps({
            "metric": "permuted NATTEN (DiT 3D neighborhood attention) ms/layer", "value": ms, "unit": UNIT,
            "n_gpus": N, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic (randn Q/K/V)",
            "config": {"workload": name, "seq_len": S, "heads": pb0.n_heads, "head_dim": D,
                       "grid": [nc.T, nc.Hh, nc.Ww], "window": [nc.kt, nc.kh, nc.kw], "tile": [nc.bt, nc.bh, nc.bw]},
            "dense_ms": dense_ms, "speedup_vs_dense": dense_ms / ms,
            "roofline": {"bound": "tensor", "achieved": achieved_adm, "peak": float(peaks["bf16_tflops"]),
                         "unit": "TFLOP/s", "frac": achieved_adm / float(peaks["bf16_tflops"]), "traffic": None,
                         "def": "admitted-element FLOPs 4*D*sum_i |window(i)| / mmi_natten_prefill time",
                         "admitted_elements": admitted},
            "gpu_launches": 4 * args.steps, "clocks": clk}), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", type=int, default=DEFAULT_WORKLOAD)
    ap.add_argument("--impl", default="mmi", choices=["mmi", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dense", type=int, default=1, help="time the same-build dense comparator once (0: skip)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _self_launch(args.gpus)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = max(world, 1)
    if args.workload == 6:
        return bench_natten(args, rank, local, N)
    if args.workload == 5:
        from synth.workloads import baselines_workload
        wl = baselines_workload()
    else:
        wl = build_workload(args.workload)
    pb = wl.problem

    if args.impl == "reference":
        # the oracle timed as it stands on the host cores: each step is a bounded sample (one head,
        # full estimation + 64 seeded rows), so the whole --steps/--warmup run ends in minutes
        if rank != 0:
            return 0
        reps = _representative_heads(wl)
        d = gen_qkv(wl, seed=args.seed, only_heads=reps)
        vals, walls = [], []
        for step in range(args.warmup + args.steps):
            h = reps[step % len(reps)]
            ms, wall, cores, sample = oracle_sample(wl, d, [h], n_rows=64, seed=step)
            if step >= args.warmup:
                vals.append(ms)
                walls.append(wall)
        v = statistics.median(vals)
        sample = (f"per step one head (cycling {reps}): full last-64 estimation + 64 seeded rows of masked fp64 "
                  f"attention, extrapolated to {pb.n_heads} heads x {pb.seq_len} rows; value = median over steps")
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": N, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": statistics.mean(walls) * 1e3, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": wl.name, "seq_len": pb.seq_len, "heads": pb.n_heads, "kv_heads": pb.n_kv_heads,
                           "head_dim": pb.head_dim},
                "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import paper_2504_16083_b200 as mmi
    torch.cuda.set_device(local)
    dist = None
    if N > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    H, Hkv, S, D = pb.n_heads, pb.n_kv_heads, pb.seq_len, pb.head_dim
    G = H // Hkv

    # this rank's KV range, then (N > Hkv) the cost-balanced head split inside it
    from paper_2504_16083_b200.dist import group_of_rank
    kv0, kv1, _ = group_of_rank(Hkv, N, rank)
    d = gen_qkv(wl, seed=args.seed, only_heads=list(range(kv0 * G, kv1 * G)))
    ranges, head_cost = plan_ranks(pb, wl.heads, N, dist, dev, d, (kv0, kv1))
    h0, h1, kv0, kv1 = ranges[rank]
    lpb = Problem(h1 - h0, kv1 - kv0, S, D, pb.n_modalities, pb.last_q, pb.block, pb.scale)
    lheads = wl.heads[h0:h1]
    q = d["q"][h0:h1].contiguous().to(dev)
    k = d["k"][kv0:kv1].contiguous().to(dev)
    v = d["v"][kv0:kv1].contiguous().to(dev)
    lab = torch.from_numpy(np.ascontiguousarray(d["labels"])).to(dev)
    O = torch.empty((H if N > 1 else h1 - h0, S, D), dtype=torch.bfloat16, device=dev)
    o = O[h0:h1] if N > 1 else O
    sp = mmi.SparsePrefill(lpb, lheads, device=dev)
    exch = OutputExchange(O, ranges, rank) if N > 1 else None

    stream = torch.cuda.current_stream()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    stage_ms = {"estimate": [], "permute": [], "sparse": [], "unpermute": [], "allgather": []}

    def step(record):
        e = [ev() for _ in range(6)] if record else None
        if e: e[0].record(stream)
        sp.estimate(q, k, lab)
        if e: e[1].record(stream)
        sp.permute(q, k, v)
        if e: e[2].record(stream)
        sp.sparse(q, k, v, o)
        if e: e[3].record(stream)
        sp.unpermute(o)
        if e: e[4].record(stream)
        if exch is not None:
            exch(dist)
        if e: e[5].record(stream)
        return e

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    # index statistics of this rank (outside the timed region)
    tiles = sp.total_tiles()                              # computed 128x128 tiles (per half)
    moved = mmi.mmi_traffic_stats(lpb, lheads, sp.ws)     # rows the permute step moves
    fp = torch.zeros((h1 - h0, S, 3), dtype=torch.int64, device=dev)
    mmi.mmi_sparse_fingerprint(lpb, lheads, sp.ws, q, k, v, fp)
    admitted = int(fp[:, :, 0].sum().item())               # sum_i |A(i)| over the rank's rows
    del fp
    if dist: dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t0, t1 = ev(), ev()
    t0.record(stream)
    evs = [step(True) for _ in range(args.steps)]
    t1.record(stream)
    torch.cuda.synchronize()
    if dist: dist.barrier()
    clk = clocks.stop()
    elapsed = t0.elapsed_time(t1)
    for e in evs:
        for i, k_ in enumerate(stage_ms):
            stage_ms[k_].append(e[i].elapsed_time(e[i + 1]))
    stage = {k_: statistics.mean(v_) for k_, v_ in stage_ms.items()}
    if dist:
        t = torch.tensor([elapsed] + [stage[k_] for k_ in stage_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t[0])
        stage = {k_: float(t[1 + i]) for i, k_ in enumerate(stage_ms)}
        tt = torch.tensor([tiles, admitted], device=dev, dtype=torch.float64)
        dist.all_reduce(tt)
        tiles_all, admitted_all = int(tt[0]), int(tt[1])
    else:
        tiles_all, admitted_all = tiles, admitted
    ms = elapsed / args.steps

    # roofline of the dominant kernel (sparse attention): computed-tile FLOPs / its event time
    peaks = _peaks()
    flops_tile = 4 * 128 * 128 * D
    sparse_ms = stage["sparse"]
    achieved = tiles * flops_tile / (sparse_ms * 1e-3) / 1e12
    peak = float(peaks["bf16_tflops"])
    traffic, tc_pct = None, None
    try:  # per-launch dram bytes + tensor-pipe % of this kernel, from the committed ncu capture of this workload
        tr = json.load(open(os.path.join(ROOT, "profiles", "attn_traffic.json")))["workloads"].get(wl.name)
        if tr and N == 1:
            traffic, tc_pct = tr["dram_bytes_per_launch"], tr.get("tensor_pipe_pct")
    except Exception:
        pass
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write, profiles/attn_traffic.json)",
            "kernel": "mmi::attn_kernel<%d>" % D,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if "_fallback" not in peaks else "fallback 1.59 PF",
            "computed_tiles": int(tiles), "flops_per_tile": flops_tile,
            "admitted_elements": admitted,
            "admitted_flops": 4 * D * admitted,
            "tile_efficiency": admitted / (tiles * 128 * 128) if tiles else None,
            "admitted_tflops": 4 * D * admitted / (sparse_ms * 1e-3) / 1e12,
            "ncu_tensor_pipe_pct": tc_pct,
            "def": "achieved = computed 128x128 tiles (both halves of every work item, after per-half dead-tile "
                   "skipping) x 4*128*128*D FLOP / sparse-stage CUDA-event time; admitted = 4*D*sum_i |A(i)| "
                   "(per-row admitted keys from the fingerprint pass)"}

    # memory-bound stages: algorithmic bytes per step / stage event time, vs the measured HBM peak
    st = mmi.mmi_plan_stats(lpb, lheads)
    hbm_peak = float(peaks["hbm_gbs"])
    alg = {
        # gathered Q-bar / K-bar / V-bar rows: read + write, bf16 (0: permutation fused into the attention loads)
        "permute": (((0 if st["fused"] & 1 else moved["qg_read"] + moved["qg_written"]) +
                     (0 if st["fused"] & 2 else 2 * (moved["kg_read"] + moved["kg_written"]))) * D * 2,
                    "(rows read + rows written) x D x 2 B of the materialised views (mmi_traffic_stats): "
                    + ("Kbar, Vbar (Q gathered in the attention kernel)" if st["fused"] == 1 else
                       "none (all gathered in the attention kernel)" if st["fused"] == 3 else "Qbar, Kbar, Vbar")),
        # LSE merge: two fp16 partial rows + two fp32 LSEs in, one bf16 row out, per token of a merged head
        "unpermute": (st["merge_heads"] * S * (2 * D * 2 + 2 * 4 + D * 2),
                      "merged heads x S x (2 fp16 partial rows + 2 fp32 LSE + 1 bf16 row)"),
    }
    hbm = {"peak_GBs": hbm_peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs", "stages": {}}
    for name, (nbytes, how) in alg.items():
        gbs = nbytes / (stage[name] * 1e-3) / 1e9 if stage[name] > 0 and nbytes > 0 else None
        hbm["stages"][name] = {"bytes": int(nbytes), "GBps": gbs, "frac": (gbs / hbm_peak) if gbs else None,
                               "bytes_def": how}
    est = estimate_bound(wl, lheads, S, D, float(peaks.get("sm_max_mhz", 1965.0)), peaks)
    est["measured_ms"] = stage["estimate"]
    est["frac"] = est["bound_ms"] / stage["estimate"] if stage["estimate"] > 0 else None

    # same-build dense comparator (a separate measurement, not in the timed steps): once at >= 512K
    dense_ms, dense_sota = None, None
    if args.dense:
        od = torch.empty_like(o)
        if S <= 262144:
            mmi.dense_prefill(lpb, q, k, v, od)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        mmi.dense_prefill(lpb, q, k, v, od)
        b.record(stream)
        torch.cuda.synchronize()
        dense_ms = a.elapsed_time(b)
        del od
        dense_sota = _sdpa_sanity(q, k, v, G, stream) if rank == 0 else None
        torch.cuda.empty_cache()

    # end to end through the public API with host buffers (pinned), per step: H2D of this rank's inputs,
    # the four calls, D2H of this rank's output heads
    e2e = None
    if not args.no_e2e:
        try:
            hp = mmi.HostSparsePrefill(lpb, lheads, device=dev)
            q_h = d["q"][h0:h1].contiguous().pin_memory()
            k_h = d["k"][kv0:kv1].contiguous().pin_memory()
            v_h = d["v"][kv0:kv1].contiguous().pin_memory()
            lab_h = torch.from_numpy(np.ascontiguousarray(d["labels"])).pin_memory()
            o_h = torch.empty(q_h.shape, dtype=torch.bfloat16).pin_memory()
            # warm-up: the first call also picks the chunking (HostSparsePrefill), the second
            # builds the chosen chunks' plans
            for _ in range(max(2, args.warmup // 2)):
                hp(q_h, k_h, v_h, lab_h, o_h)
            torch.cuda.synchronize()
            if dist: dist.barrier()
            a, b = ev(), ev()
            a.record(stream)
            for _ in range(args.steps):
                hp(q_h, k_h, v_h, lab_h, o_h)
            b.record(stream)
            torch.cuda.synchronize()
            et = a.elapsed_time(b)
            hb, db = hp.h2d_bytes(), hp.d2h_bytes()
            if dist:
                t = torch.tensor([et, hb, db], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                et = float(t[0])
                hb, db = hb * N, db * N
            e2e = {"value": et / args.steps, "unit": UNIT, "h2d_bytes_per_step": int(hb),
                   "d2h_bytes_per_step": int(db)}
            del hp, q_h, k_h, v_h, o_h
        except Exception as ex:  # pragma: no cover
            e2e = {"value": None, "unit": UNIT, "error": str(ex)[:200]}

    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu:
        reps = [h for h in _representative_heads(wl) if h0 <= h < h1]
        n_rows = 256 if S <= 262144 else 64
        ms_cpu, wall, cores, sample = oracle_sample(wl, d, reps, n_rows=n_rows)
        cpu = {"value": ms_cpu, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
               "sample_wall_s": wall}

    if rank == 0:
        nb = (S + 127) // 128
        dense_tiles = H * nb * (nb + 1) // 2
        line = {
            "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (planted video-grid Q/K, seeded)",
            "config": {"workload": wl.name, "seq_len": S, "heads": H, "kv_heads": Hkv, "head_dim": D,
                       "parallelism": f"kv-head-group x{N}" if N > 1 else "single",
                       "rank_heads": [[r[0], r[1]] for r in ranges] if N > 1 else None,
                       "l2": "inputs larger than L2 (no flush)", "head_patterns": [c.describe() for c in wl.heads]},
            "stage_ms": stage,
            "dense_ms": dense_ms,
            "speedup_vs_dense": (dense_ms / ms) if dense_ms else None,
            "dense_library_ms": dense_sota,
            "tile_density": tiles_all / dense_tiles,
            "roofline": roof, "hbm": hbm, "estimate": est,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": count_launches(lheads, int(st["fused"])) * args.steps,
            "gpu_launches_per_step": count_launches(lheads, int(st["fused"])),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
