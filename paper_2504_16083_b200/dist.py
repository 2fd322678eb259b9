"""Multi-GPU plumbing (torch.distributed): KV-head-group sharding of one layer
and the single output exchange.

Heads are independent (Alg.1-3 act per head), so ranks share no data on the
hot path; the only collective is the final all-gather of each rank's output
heads.  Partition:
  * N <= Hkv: each rank owns whole KV groups (contiguous).
  * N >  Hkv: the ranks mapped to one KV group split its G query heads into
    contiguous ranges balanced by COMPUTED-TILE COST (the per-head tile counts
    of the group's sparse index, which every rank of the group builds
    identically), instead of by head count: one h-line head costs several
    A-shape heads.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import torch

Range = Tuple[int, int, int, int]   # h0, h1, kv0, kv1


def group_of_rank(Hkv: int, N: int, r: int) -> Tuple[int, int, List[int]]:
    """(kv0, kv1, ranks sharing that KV range) for rank r of N."""
    if N <= Hkv:
        g0, g1 = r * Hkv // N, (r + 1) * Hkv // N
        return g0, g1, [r]
    g = r * Hkv // N
    return g, g + 1, [x for x in range(N) if x * Hkv // N == g]


def split_by_cost(costs: Sequence[float], k: int) -> List[Tuple[int, int]]:
    """Split items 0..n-1 into k contiguous (possibly empty) ranges minimising the largest
    range cost (exact DP; ties -> earliest split points, so every rank computes the same split)."""
    n = len(costs)
    pre = [0.0]
    for c in costs:
        pre.append(pre[-1] + float(c))
    INF = float("inf")
    # best[j][i]: minimal max-cost splitting the first i items into j ranges
    best = [[INF] * (n + 1) for _ in range(k + 1)]
    arg = [[0] * (n + 1) for _ in range(k + 1)]
    best[0][0] = 0.0
    for j in range(1, k + 1):
        for i in range(n + 1):
            for t in range(i + 1):
                v = max(best[j - 1][t], pre[i] - pre[t])
                if v < best[j][i] - 1e-12:
                    best[j][i], arg[j][i] = v, t
    cuts, i = [], n
    for j in range(k, 0, -1):
        t = arg[j][i]
        cuts.append((t, i))
        i = t
    return cuts[::-1]


def shard_heads(H: int, Hkv: int, N: int, r: int, head_cost: Optional[Sequence[float]] = None) -> Range:
    """Heads [h0, h1) and KV heads [kv0, kv1) owned by rank r of N.  head_cost (length H, e.g.
    computed tiles per head) balances the split of a shared KV group; default: equal counts."""
    G = H // Hkv
    kv0, kv1, ranks = group_of_rank(Hkv, N, r)
    if len(ranks) == 1:
        return kv0 * G, kv1 * G, kv0, kv1
    costs = list(head_cost[kv0 * G:kv1 * G]) if head_cost is not None else [1.0] * G
    a, b = split_by_cost(costs, len(ranks))[ranks.index(r)]
    return kv0 * G + a, kv0 * G + b, kv0, kv1


def all_ranges(H: int, Hkv: int, N: int, head_cost: Optional[Sequence[float]] = None) -> List[Range]:
    return [shard_heads(H, Hkv, N, r, head_cost) for r in range(N)]


class OutputExchange:
    """The single collective of the hot path: every rank owns O[h0:h1] of its range; after
    `__call__` every rank holds the whole O [H, S, D].  Ranks may own different head counts
    (cost-balanced split), so each rank's heads are packed into an equal-size slot of
    max_heads rows (one all_gather_into_tensor over NVLink), then unpacked in place."""

    def __init__(self, O: torch.Tensor, ranges: List[Range], rank: int):
        self.O, self.ranges, self.rank = O, ranges, rank
        self.hmax = max(1, max(h1 - h0 for h0, h1, _, _ in ranges))
        S, D = O.shape[1], O.shape[2]
        h0, h1 = ranges[rank][0], ranges[rank][1]
        n = h1 - h0
        # a rank owning hmax heads sends its slice of O directly; others pack into a padded slot
        self.send = O[h0:h1] if n == self.hmax else torch.zeros((self.hmax, S, D), dtype=O.dtype, device=O.device)
        self.recv = torch.empty((len(ranges) * self.hmax, S, D), dtype=O.dtype, device=O.device)

    def __call__(self, dist) -> None:
        h0, h1 = self.ranges[self.rank][0], self.ranges[self.rank][1]
        if self.send.data_ptr() != self.O[h0:h1].data_ptr():
            self.send[:h1 - h0].copy_(self.O[h0:h1])
        dist.all_gather_into_tensor(self.recv, self.send)
        for r, (a, b, _, _) in enumerate(self.ranges):
            if r != self.rank and b > a:
                self.O[a:b].copy_(self.recv[r * self.hmax:r * self.hmax + (b - a)])


def exchange_output(O, ranges, dist, rank: Optional[int] = None) -> None:
    """One-shot form of OutputExchange (allocates its buffers on every call)."""
    OutputExchange(O, ranges, dist.get_rank() if rank is None else rank)(dist)
