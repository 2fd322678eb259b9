"""World-size-2 gloo test of the N>1 host logic: KV-head-group
sharding covers every head exactly once and the output exchange assembles the
full O on every rank (CPU, gloo; the GPU path uses the same code over NCCL)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_16083_b200.dist import shard_heads, all_ranges, exchange_output


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


def _worker(rank, world, port, H, Hkv, S, D, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ranges = all_ranges(H, Hkv, world)
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
