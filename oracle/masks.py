"""O4 — element-exact masks from the paper's pattern definitions.

Predicates A_P(x, y) over query coordinate x and key coordinate y (always
intersected with causality y <= x by the caller):
  FULL                      true
  NONE                      false
  ASHAPE(sink, local)       y < sink  or  x - y < local
        ("initial tokens along with a local attention window";
         tab:impl_details P:685 Sink=128, Local=4096; reading C17)
  VS(V, Sl)                 y in V  or  (x - y) in Sl
        (P:706-708 vertical lines i_v and slash lines i_s; element-exact, C16)
  GRID(s, p, h, v, sl, sink, local)
        y < sink or x - y < local or (h and x = p mod s) or (v and y = p mod s)
        or (sl and x - y = 0 mod s)
        ("horizontal and vertical lines are evenly spaced and often
         symmetrical"; tab:search_space flags P:755-766; C8 sink/local)
  TRISHAPE(sink, local, bottom) over n rows
                            y < sink  or  x - y < local  or  x >= n - bottom
        ("full attention for all tokens to the last window's queries";
         tab:impl_details P:688 Sink 128, Local 4096, Bottom 128)
  SF_FIXED(l, stride)       floor(y / l) = floor(x / l)  or  y = 0 mod stride
        ("attention within each segment ... the segment's initial tokens";
         P:686 Local = vline_stride = token_per_frame; reading C23)
  SF_STRIDED(l, stride)     x - y < l  or  (x - y) = 0 mod stride
        ("local windows with dilated attention"; reading C23)
Boundary application (readings C12, C13):
  No/K-boundary  M(i,j) = A_P(i, j) with the global index
  Q-boundary     M(i,j) = A_{intra[lab(i)]}(i, j)          (original coordinates)
  2D-boundary    a = lab(i), b = lab(j):
                 a == b -> A_{pair[a][a]}(rho(i), rho(j))   (rank coordinates)
                 a != b -> A_{pair[a][b]}(i, j)             (original coordinates)
"""
from __future__ import annotations

from typing import Dict

import numpy as np

from synth.config import (KIND_NONE, KIND_FULL, KIND_ASHAPE, KIND_VSLASH, KIND_GRID,
                          KIND_TRISHAPE, KIND_SF_FIXED, KIND_SF_STRIDED,
                          BND_NONE, BND_K, BND_Q, BND_2D)


def member(values: np.ndarray, sorted_set: np.ndarray) -> np.ndarray:
    """Boolean: values in sorted_set (sorted_set ascending, unique)."""
    if sorted_set.size == 0:
        return np.zeros(np.shape(values), dtype=bool)
    idx = np.searchsorted(sorted_set, values)
    idx = np.clip(idx, 0, sorted_set.size - 1)
    return sorted_set[idx] == values


def pattern_pred(inst: Dict, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """A_P(x, y) for one pattern instance (index already estimated).  x, y broadcast."""
    x = np.asarray(x, dtype=np.int64)
    y = np.asarray(y, dtype=np.int64)
    kind = inst["kind"]
    shape = np.broadcast(x, y).shape
    if kind == KIND_FULL:
        return np.ones(shape, dtype=bool)
    if kind == KIND_NONE:
        return np.zeros(shape, dtype=bool)
    if kind == KIND_ASHAPE:
        return (y < inst["sink"]) | ((x - y) < inst["local"])
    if kind == KIND_VSLASH:
        return member(y, inst["V"]) | member(x - y, inst["Sl"])
    if kind == KIND_GRID:
        s, p = inst["s"], inst["p"]
        m = (y < inst["sink"]) | ((x - y) < inst["local"])
        if inst["h"]:
            m = m | (np.mod(x, s) == p)
        if inst["v"]:
            m = m | (np.mod(y, s) == p)
        if inst["sl"]:
            m = m | (np.mod(x - y, s) == 0)
        return np.broadcast_to(m, shape)
    if kind == KIND_TRISHAPE:
        m = (y < inst["sink"]) | ((x - y) < inst["local"]) | (x >= inst["n"] - inst["bottom"])
        return np.broadcast_to(m, shape)
    if kind == KIND_SF_FIXED:
        m = (np.floor_divide(y, inst["local"]) == np.floor_divide(x, inst["local"])) | (np.mod(y, inst["stride"]) == 0)
        return np.broadcast_to(m, shape)
    if kind == KIND_SF_STRIDED:
        m = ((x - y) < inst["local"]) | (np.mod(x - y, inst["stride"]) == 0)
        return np.broadcast_to(m, shape)
    raise ValueError(f"unknown pattern kind {kind}")


def head_mask_rows(boundary: int, index: Dict, labels: np.ndarray, rho: np.ndarray,
                   rows: np.ndarray, S: int) -> np.ndarray:
    """Element-exact mask M(i, j) for the given query rows (original positions),
    all keys j in [0, S).  Causality j <= i always applies."""
    rows = np.asarray(rows, dtype=np.int64)
    j = np.arange(S, dtype=np.int64)[None, :]
    i = rows[:, None]
    causal = j <= i
    if boundary in (BND_NONE, BND_K):
        return causal & pattern_pred(index["intra"][0], i, j)
    if boundary == BND_Q:
        out = np.zeros((rows.shape[0], S), dtype=bool)
        lr = labels[rows]
        for m in np.unique(lr):
            sel = lr == m
            out[sel] = pattern_pred(index["intra"][int(m)], i[sel], j)
        return out & causal
    if boundary == BND_2D:
        out = np.zeros((rows.shape[0], S), dtype=bool)
        lr = labels[rows]
        lk = labels[None, :]
        rk = rho[None, :]
        for a in np.unique(lr):
            sel = lr == a
            ia = i[sel]
            ra = rho[rows[sel]][:, None]
            m = np.zeros((ia.shape[0], S), dtype=bool)
            for b in np.unique(labels):
                colb = (lk == b)
                inst = index["pair"][int(a)][int(b)]
                if a == b:
                    pb = pattern_pred(inst, ra, rk)
                else:
                    pb = pattern_pred(inst, ia, j)
                m |= colb & pb
            out[sel] = m
        return out & causal
    raise ValueError(f"unknown boundary {boundary}")


def brute_force_mask(boundary: int, index: Dict, labels, rho, S: int) -> np.ndarray:
    """Pure-Python double loop over (i, j) of the same definitions — used only to
    cross-check the vectorised builder on tiny S."""
    def pred(inst, x, y):
        k = inst["kind"]
        if k == KIND_FULL:
            return True
        if k == KIND_NONE:
            return False
        if k == KIND_ASHAPE:
            return y < inst["sink"] or x - y < inst["local"]
        if k == KIND_VSLASH:
            return (y in set(int(t) for t in inst["V"])) or ((x - y) in set(int(t) for t in inst["Sl"]))
        if k == KIND_GRID:
            s, p = inst["s"], inst["p"]
            return (y < inst["sink"] or x - y < inst["local"] or (inst["h"] and x % s == p)
                    or (inst["v"] and y % s == p) or (inst["sl"] and (x - y) % s == 0))
        if k == KIND_TRISHAPE:
            return y < inst["sink"] or x - y < inst["local"] or x >= inst["n"] - inst["bottom"]
        if k == KIND_SF_FIXED:
            return y // inst["local"] == x // inst["local"] or y % inst["stride"] == 0
        if k == KIND_SF_STRIDED:
            return x - y < inst["local"] or (x - y) % inst["stride"] == 0
        raise ValueError(k)

    M = np.zeros((S, S), dtype=bool)
    for i in range(S):
        for jj in range(i + 1):
            if boundary in (BND_NONE, BND_K):
                M[i, jj] = pred(index["intra"][0], i, jj)
            elif boundary == BND_Q:
                M[i, jj] = pred(index["intra"][int(labels[i])], i, jj)
            else:
                a, b = int(labels[i]), int(labels[jj])
                if a == b:
                    M[i, jj] = pred(index["pair"][a][a], int(rho[i]), int(rho[jj]))
                else:
                    M[i, jj] = pred(index["pair"][a][b], i, jj)
    return M
