"""Builds profiles/r2_summary.md from the gpurun_out/e_* files of profiles/tools/r2_eval.sh."""
import csv
import collections
import json
import os
import subprocess
import sys

O = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
out = []


def line(path):
    try:
        rows = [l for l in open(path).read().splitlines() if l.strip().startswith("{")]
        return json.loads(rows[-1]) if rows else None
    except Exception:
        return None


out.append("# Round-2 measurements (one B200, sm_100a)\n")
out.append("All numbers from `profiles/tools/r2_eval.sh` on one fresh box; bench lines verbatim in "
           "`profiles/r2_bench_*.json`. Peaks: `MEASURED_PEAKS.json` (bf16 burst 1666.7 TFLOP/s, HBM 6535 GB/s).\n")
out.append("## Bench lines\n")
out.append("| workload | ms/layer | estimate | permute | sparse | unpermute | frac (live tiles) | admitted TF/s | "
           "tile eff. | estimate bound / frac | dense ms | speed-up | e2e ms | SM MHz |")
out.append("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for name in ["default", "w1", "w2", "w3", "w5"]:
    d = line(os.path.join(O, f"e_bench_{name}.json"))
    if not d:
        out.append(f"| {name} | (missing) |")
        continue
    st, r, e = d.get("stage_ms", {}), d.get("roofline", {}), d.get("estimate", {})
    e2e = d.get("e2e") or {}
    out.append(f"| {d['config']['workload']} | {d['value']:.2f} | {st.get('estimate', 0):.2f} | {st.get('permute', 0):.2f} | "
               f"{st.get('sparse', 0):.2f} | {st.get('unpermute', 0):.2f} | {r.get('frac', 0):.3f} | "
               f"{r.get('admitted_tflops', 0):.0f} | {r.get('tile_efficiency', 0) or 0:.2f} | "
               f"{e.get('bound_ms', 0):.2f} / {e.get('frac', 0) or 0:.2f} | {d.get('dense_ms') or 0:.0f} | "
               f"{d.get('speedup_vs_dense') or 0:.1f} | {e2e.get('value') or 0:.1f} | {d['clocks'].get('sm_mhz')} |")
n = line(os.path.join(O, "e_bench_w6.json"))
if n:
    out.append(f"\nNATTEN (f4, {n['config']['workload']}, grid {n['config']['grid']}, window {n['config']['window']}): "
               f"{n['value']:.2f} ms/layer, same-kernel dense (window = grid) {n['dense_ms']:.1f} ms "
               f"(x{n['speedup_vs_dense']:.1f}), admitted-element {n['roofline']['achieved']:.0f} TFLOP/s "
               f"({n['roofline']['frac']:.3f} of burst).")
ref = line(os.path.join(O, "e_bench_ref.json"))
if ref:
    out.append(f"\nReference arm (fp64 oracle, {ref['cpu_baseline']['cores']} host threads, bounded sample): "
               f"{ref['value']:.3g} ms/layer extrapolated ({ref['cpu_baseline']['sample']}).")
try:
    for l in open(os.path.join(O, "e_analysis.json")).read().splitlines():
        if l.startswith("{"):
            a = json.loads(l)
            out.append("\n" + a["measurement"] + ": " + json.dumps({k: v for k, v in a.items()
                                                                     if k not in ("picked", "generator_heads",
                                                                                  "recall_per_head",
                                                                                  "topk95_fraction_per_head")}))
except Exception:
    pass


def launches(path):
    try:
        rows = list(csv.reader(open(path)))
    except Exception:
        return None
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    names = [d["Kernel Name"] for d in data]
    starts = [i for i, n in enumerate(names) if "mod_count" in n]
    if not starts:
        return None
    tot = collections.OrderedDict()
    for d in data[starts[-1]:]:
        k = d["Kernel Name"].split("(")[0][:48]
        tot[k] = tot.get(k, 0.0) + float(d["Metric Value"]) / 1e6
    return tot


for tag in ("1m", "128k"):
    t = launches(os.path.join(O, f"e_launches_{tag}.csv"))
    if t:
        s = sum(t.values())
        out.append(f"\n## Launch list, one pipeline pass at {tag} (ncu gpu__time_duration, cold-cache, serialised)\n")
        out.append("| kernel | ms | share |")
        out.append("|---|---|---|")
        for k, v in t.items():
            out.append(f"| `{k}` | {v:.3f} | {v / s:.3f} |")

for tag in ("1m", "128k"):
    rep = os.path.join(O, f"e_sections_{tag}.ncu-rep")
    if os.path.exists(rep):
        txt = subprocess.run([sys.executable, "profiles/tools/ncu_summary.py", rep], capture_output=True, text=True).stdout
        out.append(f"\n## ncu sections at {tag}\n\n```\n{txt}```")
for tool in ("memcheck", "racecheck", "synccheck", "initcheck"):
    p = os.path.join(O, f"sanitize_{tool}.log")
    if os.path.exists(p):
        t = open(p).read().splitlines()
        summ = [l for l in t if "ERROR SUMMARY" in l or l.startswith("tool=") or "sanitize run ok" in l
                or "Barrier error" in l][:6]
        out.append(f"\ncompute-sanitizer {tool}: " + " / ".join(summ))
open(sys.argv[2] if len(sys.argv) > 2 else "profiles/r2_summary.md", "w").write("\n".join(out) + "\n")
print("\n".join(out[:40]))
