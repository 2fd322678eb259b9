"""The five BASELINE.json workloads, as layouts + head configs.

Layouts are video-shaped: frames of 256 tokens ("256 tokens per frame")
with interleaved text segments (MM-NIAH: 25 % text).  Label 0 = vision,
label 1 = text.  Head-config cycling follows SURVEY.md §8d.1 (the search-space
tuples of `tab:search_space`; A-shape (128, 4096) of P:685/770).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

from .config import (HeadConfig, Pattern, Problem, ashape, grid, vslash, none, full,
                     BND_NONE)

VISION, TEXT = 0, 1
TPF = 256  # tokens per frame

# Grid flag combinations of tab:search_space P:755-760 (h, v, sl)
GRID_FLAGS = [(True, False, False), (False, True, False), (False, False, True),
              (True, True, False), (False, True, True), (True, True, True)]
# Vertical-slash entries of tab:search_space P:772-781 (printed values, reading C18)
VS_ENTRIES = [(1000, 1024), (1000, 2048), (2000, 2048), (1000, 3096), (2000, 3096),
              (1000, 4096), (2000, 4096), (3500, 200), (1000, 2500)]


@dataclass
class Workload:
    name: str
    segments: List[Tuple[int, int]]   # (label, length) in order
    problem: Problem
    heads: List[HeadConfig]
    frame_stride: int = TPF

    @property
    def seq_len(self) -> int:
        return self.problem.seq_len


def layout_labels(segments: List[Tuple[int, int]]) -> np.ndarray:
    return np.concatenate([np.full(n, lab, dtype=np.uint8) for lab, n in segments])


def _segments(spec: List[Tuple[str, int]]) -> List[Tuple[int, int]]:
    out = []
    for kind, n in spec:
        if kind == "T":
            out.append((TEXT, n))
        else:  # frames
            out.append((VISION, n * TPF))
    return out


def _longvila_heads(H: int, Hkv: int) -> List[HeadConfig]:
    heads = []
    gi = 0
    for h in range(H):
        if h % 4 == 3:
            heads.append(HeadConfig.no_boundary(ashape(128, 4096)))
        else:
            hf, vf, sf = GRID_FLAGS[gi % len(GRID_FLAGS)]
            gi += 1
            stride = TPF if h % 2 == 0 else 0
            heads.append(HeadConfig.no_boundary(grid(stride, hf, vf, sf)))
    return heads


def _llava_heads(H: int) -> List[HeadConfig]:
    heads = []
    gi = vi = 0
    for h in range(H):
        if h % 2 == 0:
            hf, vf, sf = GRID_FLAGS[gi % len(GRID_FLAGS)]
            gi += 1
            heads.append(HeadConfig.no_boundary(grid(TPF, hf, vf, sf)))
        else:
            nv, ns = VS_ENTRIES[vi % len(VS_ENTRIES)]
            vi += 1
            heads.append(HeadConfig.no_boundary(vslash(nv, ns)))
    return heads


def _qwen_heads(H: int) -> List[HeadConfig]:
    heads = []
    for h in range(H):
        if h % 2 == 0:
            heads.append(HeadConfig.q_boundary([grid(TPF, True, True, False), vslash(1000, 2048)]))
        else:
            pairs = [[grid(TPF, False, True, True), none()],            # V->V grid, V->T none
                     [ashape(128, 4096), vslash(1000, 2048)]]          # T->V A-shape, T->T VS
            heads.append(HeadConfig.two_d(pairs))
    return heads


def build_workload(idx: int) -> Workload:
    """BASELINE.json configs[idx]."""
    if idx == 0:
        seg = _segments([("T", 128), ("F", 4), ("T", 256), ("F", 4), ("T", 128)])
        S = sum(n for _, n in seg)
        pb = Problem(1, 1, S, 64, n_modalities=2)
        return Workload("tiny", seg, pb, [HeadConfig.no_boundary(grid(TPF, True, True, False))])
    if idx == 1:
        seg = _segments([("T", 64), ("F", 511), ("T", 192)])
        pb = Problem(28, 4, sum(n for _, n in seg), 128, n_modalities=2)
        return Workload("longvila_128k", seg, pb, _longvila_heads(28, 4))
    if idx == 2:
        seg = _segments([("T", 64), ("F", 1023), ("T", 192)])
        pb = Problem(28, 4, sum(n for _, n in seg), 128, n_modalities=2)
        return Workload("llava_video_256k", seg, pb, _llava_heads(28))
    if idx == 3:
        seg = _segments([("F", 3), ("T", 256)] * 512)
        pb = Problem(28, 4, sum(n for _, n in seg), 128, n_modalities=2)
        return Workload("qwen25vl_512k", seg, pb, _qwen_heads(28))
    if idx == 4:
        seg = _segments([("T", 64), ("F", 4095), ("T", 192)])
        pb = Problem(28, 4, sum(n for _, n in seg), 128, n_modalities=2)
        return Workload("longvila_1m", seg, pb, _longvila_heads(28, 4))
    raise ValueError(idx)


def small_workload(S_frames: int = 8, text: int = 64, H: int = 2, Hkv: int = 1, D: int = 64,
                   heads: List[HeadConfig] = None, interleave: int = 0,
                   text_len: int = None) -> Workload:
    """Scaled-down layouts for parity tests (same shapes of structure, small S)."""
    if interleave:
        tl = text_len if text_len is not None else TPF
        seg = []
        for _ in range(interleave):
            seg += _segments([("F", S_frames)])
            seg.append((TEXT, tl))
    else:
        seg = _segments([("T", text), ("F", S_frames), ("T", text)])
    S = sum(n for _, n in seg)
    pb = Problem(H, Hkv, S, D, n_modalities=2)
    if heads is None:
        heads = [HeadConfig.no_boundary(grid(TPF, True, True, False))] * H
    return Workload("small", seg, pb, list(heads))


WORKLOADS = {i: (lambda i=i: build_workload(i)) for i in range(5)}


# ---------------------------------------------------------------- extra (non-BASELINE) workloads
def baselines_workload() -> Workload:
    """f3 static baselines (tab:impl_details P:685-688) on the LongVILA-shaped 128K
    layout: heads cycle A-shape(128, 4096), Tri-shape(128, 4096, 128), SparseTransformer fixed /
    strided with Local = vline_stride = tokens per frame."""
    from .config import trishape, sf_fixed, sf_strided
    seg = _segments([("T", 64), ("F", 511), ("T", 192)])
    pb = Problem(28, 4, sum(n for _, n in seg), 128, n_modalities=2)
    cyc = [ashape(128, 4096), trishape(128, 4096, 128), sf_fixed(TPF, TPF), sf_strided(TPF, TPF)]
    return Workload("baselines_128k", seg, pb, [HeadConfig.no_boundary(cyc[h % 4]) for h in range(28)])


def natten_workload():
    """f4 (App. F): a DiT-video-shaped layer -- 24 heads, D = 128, latent grid
    16 x 48 x 80 (61,440 tokens), 3D neighborhood window 5 x 15 x 15, tiles 2 x 8 x 8."""
    from .config import NattenConfig
    nc = NattenConfig(16, 48, 80, 5, 15, 15, 2, 8, 8)
    return "natten_dit_61k", Problem(24, 24, nc.seq_len, 128), nc
