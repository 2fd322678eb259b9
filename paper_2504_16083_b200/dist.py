"""Multi-GPU plumbing (torch.distributed): KV-head-group sharding of one layer
and the single output exchange.  Heads are independent (Alg.1-3
act per head), so ranks share no data on the hot path; the only collective is
the final exchange of each rank's output head slice."""
from __future__ import annotations

from typing import List, Tuple


def shard_heads(H: int, Hkv: int, N: int, r: int) -> Tuple[int, int, int, int]:
    """Heads [h0, h1) and KV heads [kv0, kv1) owned by rank r of N.

    N <= Hkv: contiguous KV groups per rank.  N > Hkv: each KV group's G query
    heads are split contiguously across the ranks mapped to that group."""
    G = H // Hkv
    if N <= Hkv:
        g0, g1 = r * Hkv // N, (r + 1) * Hkv // N
        return g0 * G, g1 * G, g0, g1
    g = r * Hkv // N
    ranks = [x for x in range(N) if x * Hkv // N == g]
    i = ranks.index(r)
    h0 = g * G + i * G // len(ranks)
    h1 = g * G + (i + 1) * G // len(ranks)
    return h0, h1, g, g + 1


def all_ranges(H: int, Hkv: int, N: int) -> List[Tuple[int, int, int, int]]:
    return [shard_heads(H, Hkv, N, r) for r in range(N)]


def exchange_output(O, ranges, dist) -> None:
    """Every rank owns O[h0:h1] of its range; after the call every rank holds the
    whole O [H, S, D].  One broadcast per rank slice, written in place into the
    final layout (no padding, no unpack)."""
    works = [dist.broadcast(O[r0:r1], src=r, async_op=True) for r, (r0, r1, _, _) in enumerate(ranges) if r1 > r0]
    for w in works:
        w.wait()
