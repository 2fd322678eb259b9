#!/usr/bin/env python
"""Benchmark: one sparse pre-fill attention layer (MMInference hot path) on B200.

A step = one pass of the whole hot path over one layer of synthetic
video-shaped input (+ a9 output all-gather for N > 1):
mmi_estimate_index -> mmi_permute -> mmi_sparse_prefill -> mmi_unpermute.
Default workload: BASELINE.json configs[1] (LongVILA-7B-shaped layer, 128K).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload I] [--impl mmi|reference]

N > 1 (torchrun): the layer's heads are sharded by KV-head group across ranks
(strong scaling of one layer), each rank runs its share, then one NCCL output
exchange (per-rank broadcasts over NVLink) assembles O on every rank.
Timing: CUDA events on the launching stream, barrier + synchronize on both
sides of the K timed steps, max over ranks.  Inputs (Q: 0.94 GB at 128K) are
larger than L2 (126 MB), so no explicit flush between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth.config import KIND_GRID, KIND_VSLASH, BND_2D, BND_Q  # noqa: E402
from synth.workloads import build_workload  # noqa: E402
from synth.gen import gen_qkv  # noqa: E402

METRIC = "sparse pre-fill attention ms/layer at 128K-1M tokens; speedup vs dense; TC util"
UNIT = "ms/layer"


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "_fallback": True}


def _patterns(cfg):
    from synth.config import KIND_NONE
    out = [cfg.intra[0]] if cfg.boundary in (0, 1) else (
        cfg.intra if cfg.boundary == BND_Q else [p for row in cfg.pair for p in row])
    return [p for p in out if p.kind != KIND_NONE]


def count_launches(heads) -> int:
    """Kernels of libmmi.so launched per step (library CUB scan/sort kernels excluded)."""
    pats = [p for c in heads for p in _patterns(c)]
    n = 4                                   # modality count / scan / place / pad
    if any(p.kind in (KIND_GRID, KIND_VSLASH) for p in pats):
        n += 4                              # slab rows, pass 1, combine, pass 2
    if any(p.kind == KIND_GRID for p in pats):
        n += 4                              # gather-rank, total, fold, pick
    if any(p.kind == KIND_VSLASH for p in pats):
        n += 1                              # vs select
    n += 2 + 1 + 3                          # views (Q̄, K̄), inst params, items count / fill / gather
    n += 2                                  # permute gathers
    n += 1                                  # sparse attention
    n += int(any(p.kind == KIND_GRID and p.use_slash for c in heads for p in _patterns(c)))  # LSE merge
    return n


from paper_2504_16083_b200.dist import shard_heads as shard, all_ranges, exchange_output  # noqa: E402


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
def oracle_sample(wl, d, seed=0, n_rows=256, heads=None):
    """Times the fp64 oracle (as it stands) on a bounded sample of the workload:
    full estimation (O2/O3) plus masked attention (O4/O5) on n_rows random rows,
    for a few representative heads; extrapolates to ms/layer."""
    from oracle.estimate import estimate_head
    from oracle.pipeline import run_head
    pb = wl.problem
    G = pb.n_heads // pb.n_kv_heads
    if heads is None:
        kinds = {}
        for h, c in enumerate(wl.heads):
            kinds.setdefault(c.describe().split("(")[0] + str(c.intra[0].stride > 0), h)
        heads = sorted(kinds.values())[:3]
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
    try:
        from threadpoolctl import threadpool_info
        cores = max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    sample = (f"heads {heads}: full last-64 estimation + {n_rows} sampled rows of masked fp64 attention each; "
              f"extrapolated to {pb.n_heads} heads x {pb.seq_len} rows")
    return ms_layer, wall, cores, sample


def _sdpa_sanity(q, k, v, G, stream):
    """SURVEY 8(d.3) sanity: the same dense causal layer through torch SDPA's cuDNN and flash
    backends (library kernels, timed beside the same-build comparator so it is not a strawman)."""
    from torch.nn.attention import sdpa_kernel, SDPBackend
    import torch.nn.functional as F
    out = {}
    qq = q.unsqueeze(0)
    kk = k.repeat_interleave(G, dim=0).unsqueeze(0)
    vv = v.repeat_interleave(G, dim=0).unsqueeze(0)
    for name, be in (("cudnn", SDPBackend.CUDNN_ATTENTION), ("flash", SDPBackend.FLASH_ATTENTION)):
        try:
            with sdpa_kernel([be]):
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", type=int, default=1)
    ap.add_argument("--impl", default="mmi", choices=["mmi", "reference"])
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--dense", type=int, default=-1, help="time the same-build dense comparator (default: S<=256K)")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    N = max(world, 1)
    wl = build_workload(args.workload)
    pb = wl.problem

    if args.impl == "reference":
        if rank != 0:
            return 0
        d = gen_qkv(wl, seed=args.seed)
        vals, walls = [], []
        for step in range(args.warmup + args.steps):
            ms, wall, cores, sample = oracle_sample(wl, d, seed=step, n_rows=1024)
            if step >= args.warmup:
                vals.append(ms)
                walls.append(wall)
        v = statistics.median(vals)
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

    d = gen_qkv(wl, seed=args.seed)
    h0, h1, kv0, kv1 = shard(pb.n_heads, pb.n_kv_heads, N, rank)
    from synth.config import Problem
    lpb = Problem(h1 - h0, kv1 - kv0, pb.seq_len, pb.head_dim, pb.n_modalities, pb.last_q, pb.block, pb.scale)
    lheads = wl.heads[h0:h1]
    q_full = d["q"].to(dev)
    k = d["k"][kv0:kv1].contiguous().to(dev)
    v = d["v"][kv0:kv1].contiguous().to(dev)
    q = q_full[h0:h1]
    lab = torch.from_numpy(np.ascontiguousarray(d["labels"])).to(dev)
    O = torch.empty((pb.n_heads, pb.seq_len, pb.head_dim), dtype=torch.bfloat16, device=dev)
    o = O[h0:h1]
    sp = mmi.SparsePrefill(lpb, lheads, device=dev)
    ranges = all_ranges(pb.n_heads, pb.n_kv_heads, N)

    def gather_out():
        if N > 1:
            exchange_output(O, ranges, dist)

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
        gather_out()
        if e: e[5].record(stream)
        return e

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    tiles = sp.total_tiles()           # computed key tiles of this rank's index (outside the timed region)
    moved = mmi.mmi_traffic_stats(lpb, lheads, sp.ws)  # rows the permute step moves (outside the timed region)
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
    if dist:
        t = torch.tensor([elapsed], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    ms = elapsed / args.steps
    stage = {k_: statistics.mean(v_) for k_, v_ in stage_ms.items()}

    # roofline of the dominant kernel (sparse attention): computed-tile FLOPs / its event time
    peaks = _peaks()
    flops_tile = 4 * 128 * 128 * pb.head_dim
    sparse_ms = stage["sparse"]
    achieved = tiles * flops_tile / (sparse_ms * 1e-3) / 1e12
    peak = float(peaks["bf16_tflops"])
    traffic = None
    try:  # dram bytes per launch of this kernel, from the committed `ncu --set full` capture of this workload
        tr = json.load(open(os.path.join(ROOT, "profiles", "attn_traffic.json")))
        if tr.get("workload") == wl.name and N == 1:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        pass
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_unit": "bytes/launch (ncu dram read+write)", "kernel": "mmi::attn_kernel<%d>" % pb.head_dim, "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)"
            if "_fallback" not in peaks else "fallback 1.59 PF", "tiles": int(tiles),
            "flops_per_tile": flops_tile}

    # memory-bound stages: algorithmic bytes per step / stage event time, vs the measured HBM peak
    st = mmi.mmi_plan_stats(lpb, lheads)
    D, S_ = pb.head_dim, pb.seq_len
    nkv = kv1 - kv0
    hbm_peak = float(peaks["hbm_gbs"])
    alg = {
        # gathered Q-bar / K-bar / V-bar rows: read + write, bf16
        "permute": ((moved["qg_read"] + moved["qg_written"] + 2 * (moved["kg_read"] + moved["kg_written"])) * D * 2,
                    "(rows read + rows written) of Qbar, Kbar, Vbar x D x 2 B (mmi_traffic_stats)"),
        # LSE merge: two fp32 partial rows + LSEs in, one bf16 row out, per token of a merged head
        "unpermute": (st["merge_heads"] * S_ * (2 * D * 4 + 2 * 4 + D * 2),
                      "merged heads x S x (2 fp32 partial rows + 2 LSE + 1 bf16 row)"),
        # slab estimation: K streamed once per pass (2 passes) + column masses written per slab
        "estimate": (2 * nkv * S_ * D * 2 + st["slabs"] * S_ * 4,
                     "2 passes x K [Hkv,S,D] bf16 + slabs x S x 4 B column masses"),
    }
    hbm = {"peak_GBs": hbm_peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs", "stages": {}}
    for name, (nbytes, how) in alg.items():
        gbs = nbytes / (stage[name] * 1e-3) / 1e9 if stage[name] > 0 else None
        hbm["stages"][name] = {"bytes": int(nbytes), "GBps": gbs, "frac": (gbs / hbm_peak) if gbs else None, "bytes_def": how}

    # same-build dense comparator (a separate measurement, not in the timed steps)
    dense_ms, dense_sota = None, None
    G = pb.n_heads // pb.n_kv_heads
    want_dense = args.dense if args.dense >= 0 else int(pb.seq_len <= 262144)
    if want_dense:
        od = torch.empty_like(o)
        mmi.dense_prefill(lpb, q, k, v, od)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)
        for _ in range(2):
            mmi.dense_prefill(lpb, q, k, v, od)
        b.record(stream)
        torch.cuda.synchronize()
        dense_ms = a.elapsed_time(b) / 2
        del od
        dense_sota = _sdpa_sanity(q, k, v, G, stream) if rank == 0 else None

    # end to end through the public API with host buffers (pinned), per step
    e2e = None
    try:
        hp = mmi.HostSparsePrefill(lpb, lheads, device=dev)
        q_h = d["q"][h0:h1].contiguous().pin_memory()
        k_h = d["k"][kv0:kv1].contiguous().pin_memory()
        v_h = d["v"][kv0:kv1].contiguous().pin_memory()
        lab_h = torch.from_numpy(np.ascontiguousarray(d["labels"])).pin_memory()
        o_h = torch.empty(q_h.shape, dtype=torch.bfloat16).pin_memory()
        for _ in range(max(1, args.warmup // 2)):
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
        e2e = {"value": et / args.steps, "unit": UNIT, "h2d_bytes_per_step": int(hb), "d2h_bytes_per_step": int(db)}
        del hp
    except Exception as ex:  # pragma: no cover
        e2e = {"value": None, "unit": UNIT, "error": str(ex)[:200]}

    cpu = None
    if rank == 0 and N == 1 and not args.no_cpu:
        ms_cpu, wall, cores, sample = oracle_sample(wl, d, n_rows=1536)
        cpu = {"value": ms_cpu, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
               "sample_wall_s": wall}

    if rank == 0:
        nb = (pb.seq_len + 127) // 128
        dense_tiles = (h1 - h0) * nb * (nb + 1) // 2
        line = {
            "metric": METRIC, "value": ms, "unit": UNIT, "n_gpus": N, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": False, "scaling": "strong" if N > 1 else "strong",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic (planted video-grid Q/K, seeded)",
            "config": {"workload": wl.name, "seq_len": pb.seq_len, "heads": pb.n_heads, "kv_heads": pb.n_kv_heads,
                       "head_dim": pb.head_dim, "parallelism": f"kv-head-group x{N}" if N > 1 else "single",
                       "l2": "inputs larger than L2 (no flush)", "head_patterns": [c.describe() for c in wl.heads]},
            "stage_ms": stage,
            "dense_ms": dense_ms,
            "speedup_vs_dense": (dense_ms / ms) if dense_ms else None,
            "dense_library_ms": dense_sota,
            "tile_density": tiles / dense_tiles,
            "roofline": roof, "hbm": hbm,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": count_launches(lheads),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
