"""GPU parity of the offline pattern search (Alg.4): the GPU search
(paper_2504_16083_b200.search, candidates evaluated by the library's hot path) and the fp64 oracle
of the selection rule (oracle/search.py, fed the GPU's kernel-measured cost table) pick the same
per-head configuration (planted inputs whose candidates are well separated: no near-ties); the
chosen configs round-trip through the JSON head-config contract."""
import numpy as np
import pytest
import torch

from synth.config import (HeadConfig, grid, ashape, vslash, full, none, save_head_configs, load_head_configs)
from synth.workloads import small_workload, _qwen_heads
from synth.gen import gen_qkv
from oracle import search as osearch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("interleave", [0, 3])
def test_search_matches_oracle(interleave, tmp_path):
    from paper_2504_16083_b200.search import PatternSearch
    heads = [HeadConfig.no_boundary(grid(256, True, True, False)), HeadConfig.no_boundary(ashape(128, 512))]
    if interleave:
        heads = _qwen_heads(2)
        wl = small_workload(S_frames=3, interleave=interleave, text_len=200, H=2, Hkv=1, D=64, heads=heads)
    else:
        wl = small_workload(S_frames=10, text=64, H=2, Hkv=1, D=64, heads=heads)
    d = gen_qkv(wl, seed=3)
    pb = wl.problem
    space = dict(intra=[ashape(64, 256), ashape(64, 1024), vslash(100, 128), grid(256, True, True, False),
                        grid(0, False, True, True, stride_min=2, stride_max=300), full()],
                 cross=[none(), full(), ashape(64, 256), vslash(100, 0)])
    lab = torch.from_numpy(np.ascontiguousarray(d["labels"])).cuda()
    ps = PatternSearch(pb, d["q"].cuda(), d["k"].cuda(), d["v"].cuda(), lab, space=space,
                       budget_pattern=ashape(64, 1024))
    cfgs, rep = ps.run()
    budget = rep["budget_tiles"]
    for h in range(pb.n_heads):
        cost = lambda c, h=h: ps.cost_table[c.describe()][h]  # noqa: E731
        ocfg, orep = osearch.search_head(pb, d["q"][h].double().numpy(), d["k"][0].double().numpy(),
                                         d["v"][0].double().numpy(), d["labels"], space, cost, budget[h])
        assert ocfg.describe() == cfgs[h].describe(), (h, ocfg.describe(), cfgs[h].describe(), orep, rep)
    path = tmp_path / "heads.json"
    save_head_configs(str(path), cfgs)
    back = load_head_configs(str(path))
    assert [c.describe() for c in back] == [c.describe() for c in cfgs]
