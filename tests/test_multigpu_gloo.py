"""World-size-2 gloo test of the N>1 host logic: KV-head-group
sharding covers every head exactly once and the output exchange assembles the
full O on every rank (CPU, gloo; the GPU path uses the same code over NCCL)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_16083_b200.dist import shard_heads, all_ranges, exchange_output, split_by_cost, OutputExchange


@pytest.mark.parametrize("H,Hkv", [(28, 4), (8, 2), (4, 4)])
@pytest.mark.parametrize("N", [1, 2, 3, 4, 8])
def test_shard_partition(H, Hkv, N):
    G = H // Hkv
    seen = []
    for r in range(N):
        h0, h1, kv0, kv1 = shard_heads(H, Hkv, N, r)
        seen += list(range(h0, h1))
        for h in range(h0, h1):
            assert kv0 <= h // G < kv1          # GQA mapping stays inside the rank's KV slice
        if h1 > h0:
            assert (h1 - h0) % max(1, kv1 - kv0) == 0 or kv1 - kv0 == 1
    assert sorted(seen) == list(range(H))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, H, Hkv, S, D, q, cost=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ranges = all_ranges(H, Hkv, world, cost)
    h0, h1, _, _ = ranges[rank]
    O = torch.zeros(H, S, D)
    # each rank "computes" its heads: a head-identifying pattern
    for h in range(h0, h1):
        O[h] = h + 0.5 * torch.arange(S * D, dtype=torch.float32).view(S, D) / (S * D)
    exchange_output(O, ranges, dist)
    want = torch.stack([h + 0.5 * torch.arange(S * D, dtype=torch.float32).view(S, D) / (S * D) for h in range(H)])
    q.put((rank, bool(torch.equal(O, want))))
    dist.destroy_process_group()


@pytest.mark.parametrize("H,Hkv", [(28, 4), (6, 2)])
def test_exchange_output_world2(H, Hkv):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, H, Hkv, 16, 8, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: True, 1: True}


def test_split_by_cost_is_optimal_and_contiguous():
    """Cost-balanced split of a KV group's heads (SURVEY §8e, N > Hkv): contiguous ranges covering
    every head once, minimal largest cost (checked against brute force over split points)."""
    import itertools
    import random
    rnd = random.Random(0)
    for _ in range(200):
        n = rnd.randint(1, 9)
        k = rnd.randint(1, 4)
        costs = [rnd.choice([1, 2, 5, 40, 300]) for _ in range(n)]
        parts = split_by_cost(costs, k)
        assert len(parts) == k and parts[0][0] == 0 and parts[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        got = max(sum(costs[a:b]) for a, b in parts)
        best = min(max(sum(costs[a:b]) for a, b in zip((0,) + c, c + (n,)))
                   for c in itertools.combinations_with_replacement(range(n + 1), k - 1) if list(c) == sorted(c))
        assert got == best


def test_cost_split_at_8_ranks():
    """N = 8 > Hkv = 4: a group's 7 heads are split by cost, not 4/3 by count."""
    H, Hkv = 28, 4
    cost = [1.0] * H
    cost[0] = cost[7] = 100.0          # one very expensive head per group 0 / 1
    r = all_ranges(H, Hkv, 8, cost)
    assert r[0][:2] == (0, 1) and r[1][:2] == (1, 7)
    assert sorted(h for a, b, _, _ in r for h in range(a, b)) == list(range(H))


@pytest.mark.parametrize("world,H,Hkv", [(2, 28, 4), (2, 7, 1), (3, 6, 2)])
def test_output_exchange_uneven_ranges(world, H, Hkv):
    """all_gather_into_tensor exchange with cost-balanced (uneven) head ranges, gloo world 2-3."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    cost = [float(1 + (h * 7) % 5) * (50 if h % 3 == 0 else 1) for h in range(H)]
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, Hkv, 8, 4, q, cost)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=10) for _ in range(world))
    assert res == {r: True for r in range(world)}
