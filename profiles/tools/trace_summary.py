"""Summarises a trace_dump.py JSON: per softmax region the sub-tile compute / exp / hand-over
times, epilogue phases, the S-issue -> S-visible and P-arrive -> P V-issue latencies, and an optional
event window.  usage: python profiles/tools/trace_summary.py TRACE.json [first_event n_events]"""
import json, sys, numpy as np
d = json.load(open(sys.argv[1]))
ev = []
for r in range(3):
    for x in d["ev"][r]:
        ev.append((x >> 8, r, (x >> 4) & 15, x & 15))
ev.sort()
names = {1: "PV", 2: "S", 3: "ITEM", 4: "Srdy", 5: "expd", 6: "Parr", 7: "epi0", 8: "epi1", 9: "item"}
# per-region stats
for r in (1, 2):
    e = [(t, c, a) for (t, rr, c, a) in ev if rr == r]
    comp, waits, exps = [], [], []
    last6 = None
    for i, (t, c, a) in enumerate(e):
        if c == 4:
            t4 = t
            if last6 is not None: waits.append(t - last6)
        if c == 5: exps.append(t - t4)
        if c == 6:
            comp.append(t - t4); last6 = t
        if c in (7, 9): last6 = None
    print(f"region {r}: subtiles {len(comp)} compute med {np.median(comp):.0f} mean {np.mean(comp):.0f} | ld+exp med {np.median(exps):.0f} | gap(Parr->next Srdy) med {np.median(waits):.0f} mean {np.mean(waits):.0f}")
    ep = []; ew = []; el = []; es = {0: [], 1: [], 2: []}; path = 0; t10 = t11 = t7 = 0
    for i, (t, c, a) in enumerate(e):
        if c == 7: t7 = t
        if c == 10: t10 = t; ew.append(t - t7)
        if c == 11: t11 = t; el.append(t - t10); path = a
        if c == 8: ep.append(t - t7); es[path].append(t - t11)
    if ep: print(f"   epilogue med {np.median(ep):.0f} mean {np.mean(ep):.0f} n {len(ep)} | o wait med {np.median(ew):.0f} | ld+pack med {np.median(el):.0f} | stores by path (0 tma-final,1 scatter,2 tma-partial): " + ", ".join(f"{k}: n={len(v)} med={np.median(v) if v else 0:.0f}" for k, v in es.items()))
# issuer: PV issue latency after P arrive, S ready latency after S issue
iss = [(t, c, a) for (t, rr, c, a) in ev if rr == 0]
tot = iss[-1][0] - iss[0][0] if iss else 0
print("issuer events", len(iss), "span", tot)
# latency S issue(hf) -> Srdy(u0) on region 1+hf
lat = {0: [], 1: []}
pend = {0: [], 1: []}
for (t, rr, c, a) in ev:
    if rr == 0 and c == 2 and a % 2 == 0: pend[a // 2].append(t)
    if rr in (1, 2) and c == 4 and a == 0:
        h = rr - 1
        if pend[h]: lat[h].append(t - pend[h].pop(0))
for h in (0, 1):
    if lat[h]: print(f"half {h}: S issue -> S ready seen med {np.median(lat[h]):.0f} mean {np.mean(lat[h]):.0f}")
lat2 = {0: [], 1: []}
pend = {0: [], 1: []}
for (t, rr, c, a) in ev:
    if rr in (1, 2) and c == 6:
        pend[rr - 1].append(t)
    if rr == 0 and c == 1:
        h = a // 2
        if pend[h]: lat2[h].append(t - pend[h].pop(0))
for h in (0, 1):
    if lat2[h]: print(f"half {h}: P arrive -> PV issue med {np.median(lat2[h]):.0f} mean {np.mean(lat2[h]):.0f}")
# print a window
if len(sys.argv) > 2:
    a0 = int(sys.argv[2]); n = int(sys.argv[3])
    t0 = ev[a0][0]
    for (t, rr, c, a) in ev[a0:a0 + n]:
        print(f"{t - t0:8d} {'   ' * rr}{['ISS','A','B'][rr]}:{names.get(c, c)}{a}")
