"""Per-head pattern configuration (input data, not arithmetic).

The paper's offline search (Alg.4) emits, per head, a boundary type
(No/K/Q/2D-Boundary) and one intra-modality pattern per modality or
one pattern per (query-modality, key-modality) pair.  The parameter tuples are
those of `tab:search_space`:
  Grid    (stride, use_hline, use_vline, use_slash, max_stride)
  A-shape (sink, local)
  VS      (vertical size, slash size)
Readings C7/C8/C17: Grid also carries a
sink and a local window (default 128/128); stride>0 means a fixed frame_stride,
stride==0 means "search [stride_min, stride_max]".
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional

KIND_NONE, KIND_FULL, KIND_ASHAPE, KIND_VSLASH, KIND_GRID = 0, 1, 2, 3, 4
# static baseline patterns of the paper's evaluation (tab:impl_details P:685-688)
KIND_TRISHAPE, KIND_SF_FIXED, KIND_SF_STRIDED = 5, 6, 7
BND_NONE, BND_K, BND_Q, BND_2D = 0, 1, 2, 3
MAX_MOD = 4

KIND_NAMES = {KIND_NONE: "none", KIND_FULL: "full", KIND_ASHAPE: "ashape",
              KIND_VSLASH: "vslash", KIND_GRID: "grid", KIND_TRISHAPE: "trishape",
              KIND_SF_FIXED: "sf_fixed", KIND_SF_STRIDED: "sf_strided"}
BND_NAMES = {BND_NONE: "none", BND_K: "k", BND_Q: "q", BND_2D: "2d"}


@dataclass(frozen=True)
class Pattern:
    kind: int = KIND_NONE
    sink: int = 0
    local: int = 0
    n_vertical: int = 0
    n_slash: int = 0
    stride: int = 0          # Grid: >0 fixed (frame_stride); 0 => search
    stride_min: int = 2
    stride_max: int = 1024
    use_hline: bool = False
    use_vline: bool = False
    use_slash: bool = False
    bottom: int = 0          # Tri-shape: the last `bottom` query rows attend to every key

    def describe(self) -> str:
        k = KIND_NAMES[self.kind]
        if self.kind == KIND_ASHAPE:
            return f"ashape({self.sink},{self.local})"
        if self.kind == KIND_TRISHAPE:
            return f"trishape({self.sink},{self.local},{self.bottom})"
        if self.kind in (KIND_SF_FIXED, KIND_SF_STRIDED):
            return f"{k}({self.local},{self.stride})"
        if self.kind == KIND_VSLASH:
            return f"vs({self.n_vertical},{self.n_slash})"
        if self.kind == KIND_GRID:
            st = self.stride if self.stride > 0 else f"[{self.stride_min},{self.stride_max}]"
            fl = "".join(c for c, f in zip("hvs", (self.use_hline, self.use_vline, self.use_slash)) if f)
            return f"grid({st},{fl},sink={self.sink},local={self.local})"
        return k


def ashape(sink: int = 128, local: int = 4096) -> Pattern:
    return Pattern(kind=KIND_ASHAPE, sink=sink, local=local)


def vslash(n_vertical: int, n_slash: int) -> Pattern:
    return Pattern(kind=KIND_VSLASH, n_vertical=n_vertical, n_slash=n_slash)


def grid(stride: int = 0, h: bool = True, v: bool = True, sl: bool = False,
         sink: int = 128, local: int = 128, stride_min: int = 2, stride_max: int = 1024) -> Pattern:
    return Pattern(kind=KIND_GRID, stride=stride, stride_min=stride_min, stride_max=stride_max,
                   use_hline=h, use_vline=v, use_slash=sl, sink=sink, local=local)


def trishape(sink: int = 128, local: int = 4096, bottom: int = 128) -> Pattern:
    """Tri-shape (tab:impl_details P:688): A-shape plus dense rows for the last `bottom`
    queries ("full attention for all tokens to the last window's queries")."""
    return Pattern(kind=KIND_TRISHAPE, sink=sink, local=local, bottom=bottom)


def sf_fixed(local: int = 256, stride: int = 256) -> Pattern:
    """SparseTransformer fixed (tab:impl_details P:686, Local = vline_stride = tokens per
    frame): attention inside the query's segment of `local` tokens plus every segment's initial
    token (keys y = 0 mod stride) -- reading C23."""
    return Pattern(kind=KIND_SF_FIXED, local=local, stride=stride)


def sf_strided(local: int = 256, stride: int = 256) -> Pattern:
    """SparseTransformer strided (tab:impl_details P:687): a local window of `local`
    tokens plus dilated lines x - y = 0 mod stride -- reading C23."""
    return Pattern(kind=KIND_SF_STRIDED, local=local, stride=stride)


def full() -> Pattern:
    return Pattern(kind=KIND_FULL)


def none() -> Pattern:
    return Pattern(kind=KIND_NONE)


@dataclass
class HeadConfig:
    """One head: boundary type + intra patterns (per query modality) or pair patterns."""
    boundary: int = BND_NONE
    intra: List[Pattern] = field(default_factory=lambda: [none()] * MAX_MOD)
    pair: List[List[Pattern]] = field(default_factory=lambda: [[none()] * MAX_MOD for _ in range(MAX_MOD)])

    @staticmethod
    def no_boundary(p: Pattern) -> "HeadConfig":
        intra = [none()] * MAX_MOD
        intra[0] = p
        return HeadConfig(boundary=BND_NONE, intra=intra)

    @staticmethod
    def q_boundary(per_mod: List[Pattern]) -> "HeadConfig":
        intra = list(per_mod) + [none()] * (MAX_MOD - len(per_mod))
        return HeadConfig(boundary=BND_Q, intra=intra)

    @staticmethod
    def two_d(pairs: List[List[Pattern]]) -> "HeadConfig":
        pr = [[none()] * MAX_MOD for _ in range(MAX_MOD)]
        for a, row in enumerate(pairs):
            for b, p in enumerate(row):
                pr[a][b] = p
        return HeadConfig(boundary=BND_2D, pair=pr)

    def describe(self) -> str:
        if self.boundary in (BND_NONE, BND_K):
            return f"{BND_NAMES[self.boundary]}:{self.intra[0].describe()}"
        if self.boundary == BND_Q:
            return "q:" + "|".join(p.describe() for p in self.intra if p.kind != KIND_NONE)
        return "2d:" + ";".join(
            f"{a}{b}={self.pair[a][b].describe()}" for a in range(MAX_MOD) for b in range(MAX_MOD)
            if self.pair[a][b].kind != KIND_NONE)


@dataclass(frozen=True)
class Problem:
    n_heads: int
    n_kv_heads: int
    seq_len: int
    head_dim: int
    n_modalities: int = 1
    last_q: int = 64          # P:412 "we set last_q = 64"
    block: int = 128          # reading C19
    scale: float = 0.0        # 0 => 1/sqrt(D)

    @property
    def tau(self) -> float:
        return self.scale if self.scale > 0 else 1.0 / (self.head_dim ** 0.5)


# ---------------------------------------------------------------- JSON head-config contract
# The offline search (Alg.4) persists one entry per head; the runtime path reads it back
# ("HeadConfig table persisted as JSON").  Pure data, no arithmetic.
import json as _json
from dataclasses import asdict as _asdict, fields as _fields

BND_BY_NAME = {v: k for k, v in BND_NAMES.items()}


def pattern_to_dict(p: Pattern) -> dict:
    d = _asdict(p)
    d["kind"] = KIND_NAMES[p.kind]
    return d


def pattern_from_dict(d: dict) -> Pattern:
    kinds = {v: k for k, v in KIND_NAMES.items()}
    d = dict(d)
    d["kind"] = kinds[d["kind"]] if isinstance(d["kind"], str) else int(d["kind"])
    names = {f.name for f in _fields(Pattern)}
    return Pattern(**{k: v for k, v in d.items() if k in names})


def head_config_to_dict(c: HeadConfig, head_id: int = 0, **extra) -> dict:
    d = {"head_id": head_id, "boundary": BND_NAMES[c.boundary]}
    if c.boundary in (BND_NONE, BND_K):
        d["intra"] = {"0": pattern_to_dict(c.intra[0])}
    elif c.boundary == BND_Q:
        d["intra"] = {str(m): pattern_to_dict(p) for m, p in enumerate(c.intra) if p.kind != KIND_NONE}
    else:
        d["pair"] = {f"{a},{b}": pattern_to_dict(c.pair[a][b]) for a in range(MAX_MOD) for b in range(MAX_MOD)
                     if c.pair[a][b].kind != KIND_NONE}
    d.update(extra)
    return d


def head_config_from_dict(d: dict) -> HeadConfig:
    b = BND_BY_NAME[d["boundary"]]
    if b in (BND_NONE, BND_K):
        c = HeadConfig.no_boundary(pattern_from_dict(d["intra"]["0"]))
        c.boundary = b
        return c
    if b == BND_Q:
        intra = [none()] * MAX_MOD
        for m, p in d["intra"].items():
            intra[int(m)] = pattern_from_dict(p)
        return HeadConfig(boundary=BND_Q, intra=intra)
    pr = [[none()] * MAX_MOD for _ in range(MAX_MOD)]
    for key, p in d.get("pair", {}).items():
        a, bb = (int(x) for x in key.split(","))
        pr[a][bb] = pattern_from_dict(p)
    return HeadConfig(boundary=BND_2D, pair=pr)


def save_head_configs(path: str, cfgs: List[HeadConfig], meta: Optional[dict] = None,
                      per_head: Optional[List[dict]] = None) -> None:
    heads = [head_config_to_dict(c, h, **((per_head or [{}] * len(cfgs))[h])) for h, c in enumerate(cfgs)]
    with open(path, "w") as f:
        _json.dump({"meta": meta or {}, "heads": heads}, f, indent=1, sort_keys=True)


def load_head_configs(path: str) -> List[HeadConfig]:
    with open(path) as f:
        d = _json.load(f)
    heads = sorted(d["heads"], key=lambda x: x["head_id"])
    return [head_config_from_dict(h) for h in heads]


# ---------------------------------------------------------------- permuted NATTEN / DiT
@dataclass(frozen=True)
class NattenConfig:
    """3D neighborhood (sliding-window) attention over a T x Hh x Ww token grid in raster order
    (App. F: "the 2D/3D sliding window attention in NATTEN can be converted into dense
    tensor core computation via permutation").  Window kt x kh x kw, clamped inside the grid
    (NATTEN semantics, reading C25); tiles bt x bh x bw of 128 tokens define the permutation."""
    T: int
    Hh: int
    Ww: int
    kt: int
    kh: int
    kw: int
    bt: int = 2
    bh: int = 8
    bw: int = 8

    @property
    def seq_len(self) -> int:
        return self.T * self.Hh * self.Ww
