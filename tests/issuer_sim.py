"""Protocol model of attn_kernel's warp roles (csrc/attn.cu): the dynamic two-half MMA issuer state
machine, the Q / K / V / key-coordinate loaders and the two softmax halves with their pv_done
bookkeeping, run under random interleavings over random per-half tile-liveness patterns.  The
kernel's issuer ("static") uses pv_done[h] as a completion counter waited only by a rescale, with
the parity of P V number n - 1 at sub-tile n -- the check below proves that wait unambiguous (at
most one phase outstanding); the dropped "dynamic" issuer needed a per-slot barrier that every
phase is waited on ("owe" bookkeeping).
Every mbarrier is a phase counter; a wait on a phase that an unobserved later phase already
overtook is reported as aliasing (the parity wait would be ambiguous), and a state where no role
can move is a deadlock.  MMAs complete at issue (the protocol, not the timing, is modelled)."""
import random, sys

class Bar:
    def __init__(s, name, count): s.name, s.count, s.arr, s.done = name, count, 0, 0
    def arrive(s):
        s.arr += 1
        if s.arr == s.count: s.arr = 0; s.done += 1
    def test(s, k):  # phase k (absolute index) completed?  flags aliasing (k+2 completed unobserved)
        return s.done > k
    def check(s, k):
        if s.done > k + 1: raise RuntimeError(f"aliasing on {s.name}: waiting phase {k}, done {s.done}")

def run(items, KST=2, VST=2, NKP=4, seed=0, issuer="static", coupled=False, s64=False):
    """issuer="static": the kernel's issuer (per key tile P_A(t,0)V P_B(t,0)V P_A(t,1)V S_A(t+1)
    P_B(t,1)V S_B(t+1)); "dynamic": the measured-and-dropped per-half dynamic issuer (N=64 scores
    one tile ahead); coupled=True with "dynamic": its first version, whose state 2 blocked on the
    next tile's K load (deadlocks); s64=True with "static": S as two N=64 slot groups, each issued
    right after the P V that freed its slot (MMI_S64)."""
    rnd = random.Random(seed)
    B = {}
    def bar(n, c=1):
        if n not in B: B[n] = Bar(n, c)
        return B[n]
    for i in range(KST): bar(f"kf{i}"); bar(f"ke{i}")
    for i in range(VST): bar(f"vf{i}"); bar(f"ve{i}")
    for i in range(NKP): bar(f"kpf{i}"); bar(f"kpe{i}", 2)
    for h in range(2):
        bar(f"oe{h}"); bar(f"of{h}")
        for u in range(2): bar(f"sf{h}{u}"); bar(f"pf{h}{u}"); bar(f"pv{h}{u}")
        bar(f"pv{h}")
    bar("qf"); bar("qe")
    live_s = [0] * KST

    def wait(name, k):  # generator helper: block until phase k of bar completed (k = -1: passes)
        b = B[name]
        while not b.test(k):
            yield
        b.check(k)

    def qloader():
        for i, it in enumerate(items):
            yield from wait("qe", i - 1)
            B["qf"].arrive()
    def kloader():
        g = 0; kp = 0
        for it in items:
            for t in range(it["n"]):
                yield from wait(f"ke{g % KST}", g // KST - 1)
                live_s[g % KST] = it["live"][t]
                B[f"kf{g % KST}"].arrive()
                if it["kp"][t]:
                    yield from wait(f"kpe{kp % NKP}", kp // NKP - 1)
                    B[f"kpf{kp % NKP}"].arrive(); kp += 1
                g += 1
    def vloader():
        g = 0
        for it in items:
            for t in range(it["n"]):
                yield from wait(f"ve{g % VST}", g // VST - 1)
                B[f"vf{g % VST}"].arrive(); g += 1
    def issuer_static():
        ks = vs = 0; kph = vph = 0
        pcount = {(h, u): 0 for h in range(2) for u in range(2)}
        ocount = [0, 0]
        qk = 0
        for it in items:
            n = it["n"]; nh = 2 if it["has_b"] else 1
            yield from wait("qf", qk); qk += 1
            started = 0
            def issue_pv(h, u):
                nonlocal started
                yield from wait(f"pf{h}{u}", pcount[(h, u)]); pcount[(h, u)] += 1
                if not (started >> h) & 1:
                    yield from wait(f"oe{h}", ocount[h] - 1)
                started |= 1 << h
                B[f"pv{h}"].arrive()
            def issue_s(h, u=None):
                if not s64:
                    B[f"sf{h}0"].arrive()  # one commit for both 64-key slots of the M128 N128 group
                else:
                    for x in ((0, 1) if u is None else (u,)): B[f"sf{h}{x}"].arrive()
            g = None
            yield from wait(f"kf{ks}", kph_count[0] // KST)
            kph_count[0] += 1
            live_cur = live_s[ks]
            for h in range(nh):
                if (live_cur >> h) & 1: issue_s(h)
            if n == 1: B["qe"].arrive()
            B[f"ke{ks}"].arrive(); ks = (ks + 1) % KST
            for t in range(n):
                ahead = t + 1 < n
                yield from wait(f"vf{vs}", vph_count[0] // VST); vph_count[0] += 1
                live_next = 0
                if ahead:
                    yield from wait(f"kf{ks}", kph_count[0] // KST); kph_count[0] += 1
                    live_next = live_s[ks]
                if ahead and s64:
                    for u in range(2):
                        for h in range(nh):
                            if (live_cur >> h) & 1: yield from issue_pv(h, u)
                            if (live_next >> h) & 1: issue_s(h, u)
                elif ahead:
                    for h in range(nh):
                        if (live_cur >> h) & 1: yield from issue_pv(h, 0)
                    for h in range(nh):
                        if (live_cur >> h) & 1: yield from issue_pv(h, 1)
                        if (live_next >> h) & 1: issue_s(h)
                else:
                    for h in range(nh):
                        if (live_cur >> h) & 1:
                            yield from issue_pv(h, 0); yield from issue_pv(h, 1)
                        if (started >> h) & 1:
                            B[f"of{h}"].arrive(); ocount[h] += 1
                if t + 1 == n - 1: B["qe"].arrive()
                B[f"ve{vs}"].arrive(); vs = (vs + 1) % VST
                if ahead:
                    B[f"ke{ks}"].arrive(); ks = (ks + 1) % KST
                live_cur = live_next
    kph_count = [0]; vph_count = [0]
    def issuer():
        kr_g = 0
        pcount = {(h, u): 0 for h in range(2) for u in range(2)}
        ocount = [0, 0]
        qk = 0
        for it in items:
            n = it["n"]; has_b = it["has_b"]
            yield from wait("qf", qk); qk += 1
            pres = 3 if has_b else 1
            gb = kr_g; kw = vw = kr = vr = gb
            lring = {}; kmask = {}; vmask = {}
            st = [0 if (pres >> h) & 1 else 6 for h in range(2)]
            np_ = [-1, -1]; ns = [0, 0]
            sdone = 0 if has_b else 2
            started = 0; qrel = False
            def k_known(t):
                nonlocal kw
                while kw <= gb + t:
                    if not B[f"kf{kw % KST}"].test(kw // KST): return False
                    B[f"kf{kw % KST}"].check(kw // KST)
                    lring[kw] = live_s[kw % KST]; kw += 1
                return True
            def v_known(t):
                nonlocal vw
                while vw <= gb + t:
                    if not B[f"vf{vw % VST}"].test(vw // VST): return False
                    vw += 1
                return True
            def scan(h):
                while ns[h] < n:
                    if not k_known(ns[h]): return 0
                    if (lring[gb + ns[h]] >> h) & 1: return 1
                    kmask[gb + ns[h]] = kmask.get(gb + ns[h], 0) | (1 << h)
                    vmask[gb + ns[h]] = vmask.get(gb + ns[h], 0) | (1 << h)
                    ns[h] += 1
                return 2
            def issue_s(h, t, u): B[f"sf{h}{u}"].arrive()
            def issue_pv(h, t, u):
                nonlocal started
                started |= 1 << h; B[f"pv{h}{u}"].arrive()
            s0 = [False, False]; nonext = [False, False]
            def step(h):
                nonlocal sdone
                prog = False
                while True:
                    s = st[h]
                    if s == 0:
                        r = scan(h)
                        if r == 0: return prog
                        prog = True
                        if r == 2:
                            sdone |= 1 << h; st[h] = 6; continue
                        issue_s(h, ns[h], 0); issue_s(h, ns[h], 1)
                        kmask[gb + ns[h]] = kmask.get(gb + ns[h], 0) | (1 << h)
                        np_[h] = ns[h]; ns[h] += 1; st[h] = 1
                    elif s == 2:
                        r = scan(h)
                        if coupled and r == 0: return prog
                        prog = True
                        s0[h] = False; nonext[h] = False
                        if r == 1: issue_s(h, ns[h], 0); s0[h] = True
                        elif r == 2: sdone |= 1 << h; nonext[h] = True
                        st[h] = 3
                    elif s in (1, 3):
                        u = 1 if s == 3 else 0
                        if not v_known(np_[h]): return prog
                        if not (started >> h) & 1 and not B[f"oe{h}"].test(ocount[h] - 1): return prog
                        if not B[f"pf{h}{u}"].test(pcount[(h, u)]): return prog
                        pcount[(h, u)] += 1
                        issue_pv(h, np_[h], u); prog = True
                        if u == 0: st[h] = 2
                        else:
                            vmask[gb + np_[h]] = vmask.get(gb + np_[h], 0) | (1 << h)
                            st[h] = 4
                    elif s == 4:
                        if nonext[h]:
                            B[f"of{h}"].arrive(); ocount[h] += 1; st[h] = 6; prog = True; continue
                        if not s0[h]:
                            r = scan(h)
                            if r == 0: return prog
                            prog = True
                            if r == 2:
                                sdone |= 1 << h; nonext[h] = True; continue
                            issue_s(h, ns[h], 0)
                        issue_s(h, ns[h], 1); kmask[gb + ns[h]] = kmask.get(gb + ns[h], 0) | (1 << h)
                        np_[h] = ns[h]; ns[h] += 1; st[h] = 1; prog = True
                    else: return prog
            def release():
                nonlocal kr, vr, vw, qrel
                while kr < kw and kmask.get(kr, 0) == pres:
                    B[f"ke{kr % KST}"].arrive(); kr += 1
                while vr < gb + n and vmask.get(vr, 0) == pres:
                    if vr == vw:
                        if not B[f"vf{vw % VST}"].test(vw // VST): break
                        vw += 1
                    B[f"ve{vr % VST}"].arrive(); vr += 1
                if not qrel and sdone == 3:
                    B["qe"].arrive(); qrel = True
            while True:
                step(0)
                if has_b: step(1)
                release()
                if st[0] == 6 and st[1] == 6 and kr == gb + n and vr == gb + n and qrel: break
                yield
            kr_g = gb + n
    def softmax(h):
        kp = 0
        sph = [0, 0]; pvph = [0, 0]; owe = [False, False]; oph = 0; nsub = 0
        for it in items:
            n = it["n"]
            present = h == 0 or it["has_b"]
            nl = 0
            for t in range(n):
                if it["kp"][t]:
                    yield from wait(f"kpf{kp % NKP}", kp // NKP)
                    B[f"kpe{kp % NKP}"].arrive(); kp += 1
                if not present or not (it["live"][t] >> h) & 1: continue
                nl += 1
                for u in range(2):
                    if issuer != "static" or u == 0 or s64:
                        yield from wait(f"sf{h}{u}", sph[u]); sph[u] += 1
                    if issuer == "static":
                        if rnd.random() < 0.3 and nsub > 0:  # rescale: P V number nsub - 1 landed
                            yield from wait(f"pv{h}", nsub - 1)
                        B[f"pf{h}{u}"].arrive(); nsub += 1
                        continue
                    if owe[u]:
                        yield from wait(f"pv{h}{u}", pvph[u]); pvph[u] += 1; owe[u] = False
                    if rnd.random() < 0.3 and owe[u ^ 1]:
                        yield from wait(f"pv{h}{u ^ 1}", pvph[u ^ 1]); pvph[u ^ 1] += 1; owe[u ^ 1] = False
                    B[f"pf{h}{u}"].arrive(); owe[u] = True
            if present and nl > 0:
                yield from wait(f"of{h}", oph); oph += 1
                for u in range(2):
                    if owe[u]:
                        yield from wait(f"pv{h}{u}", pvph[u]); pvph[u] += 1
                owe = [False, False]
                B[f"oe{h}"].arrive()
    procs = {"q": qloader(), "k": kloader(), "v": vloader(), "iss": issuer_static() if issuer == "static" else issuer(), "sA": softmax(0), "sB": softmax(1)}
    alive = dict(procs)
    stuck = 0
    while alive:
        name = rnd.choice(list(alive))
        try:
            next(alive[name]); 
        except StopIteration:
            del alive[name]; stuck = 0; continue
        stuck += 1
        if stuck > 20000:
            return "DEADLOCK", {k: (b.done, b.arr) for k, b in B.items()}, list(alive)
    return "ok", None, None

def rand_items(rnd, n_items):
    items = []
    for _ in range(n_items):
        n = rnd.randint(1, 12)
        has_b = rnd.random() < 0.8
        live = []
        for t in range(n):
            a = rnd.random() < 0.8; b = has_b and rnd.random() < 0.8
            if not has_b and rnd.random() < 0.2: a = False
            x = (1 if a else 0) | (2 if b else 0)
            if has_b and x == 0 and rnd.random() < 0.5: x = 1
            live.append(x)
        kp = [rnd.random() < 0.5 for _ in range(n)]
        items.append(dict(n=n, has_b=has_b, live=live, kp=kp))
    return items

if __name__ == "__main__":
    rnd = random.Random(1)
    for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 300):
        items = rand_items(rnd, rnd.randint(1, 6))
        r, st, alive = run(items, seed=trial)
        if r != "ok":
            print("trial", trial, r, alive)
            for it in items: print(it)
            print({k: v for k, v in st.items()})
            break
    else:
        print("all ok")
