"""Deterministic planted-structure Q/K/V generator (SURVEY.md §8d.1 "Generator").

Structure is planted in Q/K geometry, never in attention matrices:
  * per KV group g: unit patch directions phi_g[x] (x in [0,256)) give "same
    patch in another frame" similarity (slash lines at multiples of 256),
  * a vertical-line family u_g1 on keys with patch index x_g1 (stride 256 in
    frame coordinates), and a second family u_g2 on keys j = p_g2 (mod s_g2),
    s_g2 in {128, 512}, for searched-stride heads,
  * a sink direction on keys j < 4, and a rotary-like locality block,
  * VS heads: a sparse random set of keys carrying u_vs.
Each Q head adds the direction of its planted family.  V ~ N(0, 1).
Seeds: per-head / per-group streams from np.random.SeedSequence(seed).spawn.
The planted truth (stride, phase) is returned beside the tensors.
"""
from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from typing import Dict

import numpy as np
import torch

from .config import KIND_ASHAPE, KIND_GRID, KIND_VSLASH, BND_NONE, BND_K, BND_Q, BND_2D
from .workloads import Workload, layout_labels, TPF, VISION, TEXT

# gains (logit units after the 1/sqrt(D) scale); tuned so that the oracle
# recovers the planted (stride, phase) on every grid head.
G_LINE = 3.2     # vertical line family 1 (frame stride, phase-only search)
G_LINE2 = 5.0    # family 2 (searched stride): must beat divisor/noise classes under reading C5
G_PATCH = 1.6    # same-patch (slash) similarity
G_SINK = 3.5
G_LOCAL = 2.0
G_VS = 3.0
NOISE = 1.0
Q_NOISE = 0.5    # query noise scale: logit noise std ~0.5 (keeps planted lines above noise peaks)


def _unit(rng, n, D):
    x = rng.standard_normal((n, D))
    return x / np.linalg.norm(x, axis=1, keepdims=True)


def _patch_index(labels: np.ndarray) -> np.ndarray:
    """Index within the current vision run, mod 256 (-1 for text)."""
    S = labels.shape[0]
    x = np.full(S, -1, dtype=np.int64)
    run = 0
    for i in range(S):
        if labels[i] == VISION:
            x[i] = run % TPF
            run += 1
        else:
            run = 0
    return x


def _vision_rank(labels: np.ndarray) -> np.ndarray:
    r = np.cumsum(labels == VISION) - 1
    return r


def _head_role(cfg) -> Dict[str, object]:
    """Which planted family each query modality of this head carries."""
    role = {}
    if cfg.boundary in (BND_NONE, BND_K):
        role[VISION] = role[TEXT] = cfg.intra[0]
    elif cfg.boundary == BND_Q:
        role[VISION], role[TEXT] = cfg.intra[0], cfg.intra[1]
    else:
        role[VISION], role[TEXT] = cfg.pair[0][0], cfg.pair[1][1]
    return role


def gen_qkv(wl: Workload, seed: int = 0, chunk: int = 1 << 16,
            dtype=torch.bfloat16, only_heads=None) -> Dict[str, object]:
    """only_heads: generate Q for these heads and K/V for their KV groups only (the other
    entries stay zero); the generated values are bit-identical to a full call, since every
    head and group draws from its own SeedSequence stream."""
    pb = wl.problem
    H, Hkv, S, D = pb.n_heads, pb.n_kv_heads, pb.seq_len, pb.head_dim
    G = H // Hkv
    labels = layout_labels(wl.segments)
    assert labels.shape[0] == S
    px = _patch_index(labels)
    vr = _vision_rank(labels)
    first_vis = int(np.argmax(labels == VISION)) if (labels == VISION).any() else 0
    scale_dir = D ** 0.25          # so that (a*u).(b*u)/sqrt(D) = a*b
    ss = np.random.SeedSequence(seed)
    kv_seeds = ss.spawn(Hkv)
    q_seeds = ss.spawn(H)

    alloc = torch.empty if only_heads is None else torch.zeros
    q = alloc((H, S, D), dtype=dtype)
    k = alloc((Hkv, S, D), dtype=dtype)
    v = alloc((Hkv, S, D), dtype=dtype)

    pos = np.arange(S)
    is_vis = labels == VISION
    freqs = 2 * np.pi / np.array([61.0, 157.0])   # short periods, coprime, far from 2^k strides

    def make_group(g):
        rng = np.random.default_rng(kv_seeds[g])
        phi = _unit(rng, TPF, D)
        # 0:g1 1:g2 2:sink 3:vs 4..7 locality basis; orthonormal so that one
        # family never leaks into another (a leak mixes strides 256 and s_g2)
        u = np.linalg.qr(rng.standard_normal((D, 8)))[0].T
        # patch directions orthogonal to the planted directions too: otherwise
        # phi[x].u acts as a per-patch-index (stride-256) bias on every frame
        phi = phi - (phi @ u.T) @ u
        phi /= np.linalg.norm(phi, axis=1, keepdims=True)
        x_g1 = int(rng.integers(0, TPF))
        s_g2 = int(rng.choice([128, 512]))
        p_g2 = int(rng.integers(0, s_g2))
        vs_keys = rng.random(S) < (1.0 / 400.0)
        vs_keys[:4] = False
        for c0 in range(0, S, chunk):
            c1 = min(S, c0 + chunk)
            n = c1 - c0
            kk = rng.standard_normal((n, D)) * NOISE
            kk -= (kk @ u.T) @ u          # key noise orthogonal to the planted directions
            pc = pos[c0:c1]
            vis = is_vis[c0:c1]
            xx = px[c0:c1]
            kk[vis] += G_PATCH ** 0.5 * scale_dir * phi[xx[vis]]
            kk += (G_LINE ** 0.5 * scale_dir) * np.outer(((xx == x_g1) & vis).astype(np.float64), u[0])
            kk += (G_LINE2 ** 0.5 * scale_dir) * np.outer((pc % s_g2 == p_g2).astype(np.float64), u[1])
            kk += (G_SINK ** 0.5 * scale_dir) * np.outer((pc < 4).astype(np.float64), u[2])
            kk += (G_VS ** 0.5 * scale_dir) * np.outer(vs_keys[c0:c1].astype(np.float64), u[3])
            for f, w in enumerate(freqs):
                a = (G_LOCAL / len(freqs)) ** 0.5 * scale_dir
                kk += a * (np.outer(np.cos(w * pc), u[4 + 2 * f]) + np.outer(np.sin(w * pc), u[5 + 2 * f]))
            k[g, c0:c1] = torch.from_numpy(kk.astype(np.float32)).to(dtype)
            v[g, c0:c1] = torch.from_numpy(rng.standard_normal((n, D)).astype(np.float32)).to(dtype)
        return dict(phi=phi, u=u, x_g1=x_g1, s_g2=s_g2, p_g2=p_g2, vs_keys=vs_keys)

    # every KV group / query head draws from its own SeedSequence stream, so the groups and heads
    # are generated in parallel threads (numpy RNG and BLAS release the GIL) with a result that is
    # bit-identical to a sequential loop
    with ThreadPoolExecutor(max_workers=max(1, min(os.cpu_count() or 1, 32))) as ex:
        need_g = sorted({h // G for h in (only_heads if only_heads is not None else range(H))})
        made = dict(zip(need_g, ex.map(make_group, need_g)))
    groups = [made.get(g) for g in range(Hkv)]

    def make_head(h):
        g = h // G
        gr = groups[g]
        u, phi = gr["u"], gr["phi"]
        rng = np.random.default_rng(q_seeds[h])
        role = _head_role(wl.heads[h])
        info = {}
        dirs = {}
        for lab in (VISION, TEXT):
            p = role[lab]
            d = np.zeros(D)
            if p.kind == KIND_GRID:
                if p.stride > 0:
                    d += u[0]
                    if wl.heads[h].boundary == BND_2D:
                        info[lab] = (TPF, gr["x_g1"])
                    else:
                        info[lab] = (TPF, (first_vis + gr["x_g1"]) % TPF)
                else:
                    d += u[1] * (G_LINE2 / G_LINE) ** 0.5
                    info[lab] = (gr["s_g2"], gr["p_g2"])
            elif p.kind == KIND_VSLASH:
                d += u[3]
            dirs[lab] = d
        for c0 in range(0, S, chunk):
            c1 = min(S, c0 + chunk)
            n = c1 - c0
            qq = rng.standard_normal((n, D)) * Q_NOISE
            pc = pos[c0:c1]
            vis = is_vis[c0:c1]
            xx = px[c0:c1]
            lab = labels[c0:c1]
            qq[vis] += G_PATCH ** 0.5 * scale_dir * phi[xx[vis]]
            for L in (VISION, TEXT):
                sel = (lab == L)
                if dirs[L].any():
                    qq[sel] += (G_LINE ** 0.5 * scale_dir) * dirs[L]
            qq += (G_SINK ** 0.5 * scale_dir) * u[2]
            for f, w in enumerate(freqs):
                a = (G_LOCAL / len(freqs)) ** 0.5 * scale_dir
                qq += a * (np.outer(np.cos(w * pc), u[4 + 2 * f]) + np.outer(np.sin(w * pc), u[5 + 2 * f]))
            q[h, c0:c1] = torch.from_numpy(qq.astype(np.float32)).to(dtype)
        return info

    with ThreadPoolExecutor(max_workers=max(1, min(os.cpu_count() or 1, 32))) as ex:
        hs = list(only_heads) if only_heads is not None else list(range(H))
        made_h = dict(zip(hs, ex.map(make_head, hs)))
    planted = [made_h.get(h, {}) for h in range(H)]

    return dict(q=q, k=k, v=v, labels=labels, planted=planted, vision_rank=vr)
