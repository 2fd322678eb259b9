"""Markdown table of bench.py JSON lines: python profiles/tools/bench_table.py f1.json f2.json ..."""
import json, sys
print("| workload | ms/layer | estimate | permute | sparse | unpermute | dense ms (same build) | cuDNN SDPA ms | speed-up vs same-build dense | sparse TFLOP/s | frac of measured peak | tile density | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for f in sys.argv[1:]:
    for l in open(f):
        if not l.startswith("{"):
            continue
        d = json.loads(l)
        st = d["stage_ms"]
        lib = d.get("dense_library_ms") or {}
        dn = d.get("dense_ms")
        r = d["roofline"]
        print(f"| {d['config']['workload']} | {d['value']:.2f} | {st['estimate']:.2f} | {st['permute']:.2f} | {st['sparse']:.2f} | "
              f"{st['unpermute']:.2f} | {dn:.1f} | {lib.get('cudnn') or float('nan'):.1f} | {d['speedup_vs_dense'] or float('nan'):.1f} | "
              f"{r['achieved']:.0f} | {r['frac']:.3f} | {d['tile_density']:.4f} | {d['clocks']['sm_mhz']} |"
              if dn else
              f"| {d['config']['workload']} | {d['value']:.2f} | {st['estimate']:.2f} | {st['permute']:.2f} | {st['sparse']:.2f} | "
              f"{st['unpermute']:.2f} | — | — | — | {r['achieved']:.0f} | {r['frac']:.3f} | {d['tile_density']:.4f} | {d['clocks']['sm_mhz']} |")
