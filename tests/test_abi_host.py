"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/mmi.h declares, sizes workspaces, and rejects invalid problems / configs
on the host with the documented status codes (no GPU needed)."""
import ctypes
import os
import re

import pytest

from synth.config import HeadConfig, Problem, grid, ashape, vslash, none, full
from synth.workloads import build_workload

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2504_16083_b200 import lib
    return lib()


def test_library_exports_header_symbols():
    hdr = open(os.path.join(ROOT, "include", "mmi.h")).read()
    names = re.findall(r"MMI_API\s+[\w\s\*]*?\b(mmi_\w+)\s*\(", hdr)
    assert len(names) >= 10
    L = _lib()
    for n in names:
        assert hasattr(L, n), n
    assert L.mmi_version().startswith(b"mmi-b200")


@pytest.mark.parametrize("idx", range(5))
def test_workspace_sizes_for_baseline_configs(idx):
    from paper_2504_16083_b200 import mmi_workspace_bytes
    wl = build_workload(idx)
    n = mmi_workspace_bytes(wl.problem, wl.heads)
    assert n > 0
    assert n < 64 << 30   # fits a 180 GB B200 with room for Q/K/V/O


def _ws(pb, heads):
    from paper_2504_16083_b200 import mmi_workspace_bytes
    return mmi_workspace_bytes(pb, heads)


def test_invalid_configs_rejected_on_host():
    from paper_2504_16083_b200.mmi import lib, to_c_problem, to_c_configs
    pb = Problem(2, 1, 4096, 128, n_modalities=2)
    bad = [
        [HeadConfig.no_boundary(none())] * 2,                                   # no keys for any row
        [HeadConfig.no_boundary(ashape(128, 0))] * 2,                           # local < 1
        [HeadConfig.no_boundary(vslash(0, 10))] * 2,                            # n_vertical < 1
        [HeadConfig.no_boundary(grid(2000))] * 2,                               # stride > 1024
        [HeadConfig.two_d([[grid(256), grid(256)], [ashape(), full()]])] * 2,   # grid on a cross pair
        [HeadConfig.two_d([[none(), none()], [none(), full()]])] * 2,           # pair[a][a] NONE
        [HeadConfig.two_d([[full(), vslash(10, 5)], [none(), full()]])] * 2,    # cross VS with slashes
        [HeadConfig.q_boundary([grid(256), none()])] * 2,                       # Q-boundary modality NONE
    ]
    for heads in bad:
        assert _ws(pb, heads) == 0
        assert len(lib().mmi_last_error()) > 0
    # shape errors
    assert _ws(Problem(3, 2, 4096, 128), [HeadConfig.no_boundary(full())] * 3) == 0
    assert b"multiple" in lib().mmi_last_error()
    assert _ws(Problem(2, 1, 4096, 96), [HeadConfig.no_boundary(full())] * 2) == 0
    assert _ws(Problem(2, 1, 0, 128), [HeadConfig.no_boundary(full())] * 2) == 0
    # valid
    assert _ws(pb, [HeadConfig.no_boundary(full())] * 2) > 0


def test_compute_calls_validate_before_launch():
    """Null workspace / pointers return a status (no launch, safe without a GPU)."""
    from paper_2504_16083_b200.mmi import lib, to_c_problem, to_c_configs
    pb = Problem(1, 1, 1024, 64)
    heads = [HeadConfig.no_boundary(full())]
    L = lib()
    st = L.mmi_estimate_index(ctypes.byref(to_c_problem(pb)), to_c_configs(heads), None, None, None, None, 0, None)
    assert st == 5  # MMI_E_WORKSPACE
    st = L.mmi_dense_prefill(ctypes.byref(to_c_problem(pb)), None, None, None, None, None, None)
    assert st == 1  # MMI_E_INVALID


def test_binding_refuses_cpu_fallback():
    """The product path never computes on the CPU: without CUDA the binding raises."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2504_16083_b200 import SparsePrefill
    wl = build_workload(0)
    sp_err = None
    try:
        sp = SparsePrefill(wl.problem, wl.heads, device="cpu")
        q = torch.zeros(1, wl.problem.seq_len, 64, dtype=torch.bfloat16)
        sp(q, q[:1], q[:1], torch.zeros(wl.problem.seq_len, dtype=torch.uint8))
    except (RuntimeError, ValueError) as e:
        sp_err = e
    assert sp_err is not None


@pytest.mark.parametrize("idx", [1, 3])
def test_plan_stats_consistent_with_config(idx):
    """mmi_plan_stats (host-only): one estimation slab per estimated pattern instance
    (Grid / VS; per query modality for Q-/2D-boundary heads), merge heads = heads with
    a multi-pass Grid (slash) instance, gathered rows padded to whole 128-row tiles."""
    from paper_2504_16083_b200 import mmi_plan_stats
    from synth.config import KIND_GRID, KIND_VSLASH
    wl = build_workload(idx)
    st = mmi_plan_stats(wl.problem, wl.heads)
    assert st["qg_rows"] % 128 == 0 and st["kg_rows"] % 128 == 0
    assert st["qg_rows"] > 0 and st["kg_rows"] > 0
    n_est = sum(1 for h in wl.heads if any(p.kind in (KIND_GRID, KIND_VSLASH) for p in
                                           ([h.intra[0]] if h.boundary in (0, 1) else
                                            h.intra[:wl.problem.n_modalities] if h.boundary == 2 else
                                            [q for row in h.pair for q in row])))
    assert 1 <= st["slabs"]
    assert st["slabs"] >= n_est
    assert 0 <= st["merge_heads"] <= wl.problem.n_heads
    if idx == 1:   # LongVILA-shaped: grid heads with slash lines need the LSE merge
        n_slash = sum(1 for h in wl.heads if h.intra[0].kind == KIND_GRID and h.intra[0].use_slash)
        assert st["merge_heads"] == n_slash


def test_plan_stats_rejects_invalid():
    from paper_2504_16083_b200.mmi import lib, to_c_problem, to_c_configs
    pb = Problem(3, 2, 4096, 128)    # H % Hkv != 0
    out = (ctypes.c_int64 * 5)()
    st = lib().mmi_plan_stats(ctypes.byref(to_c_problem(pb)), to_c_configs([HeadConfig.no_boundary(full())] * 3),
                              out, 5)
    assert st != 0
    assert lib().mmi_plan_stats(None, None, out, 5) != 0


def test_binding_checks_dtype_and_shape():
    """The binding checks dtype / shape before handing raw pointers to the C ABI."""
    import torch
    from paper_2504_16083_b200.mmi import _check_io
    pb = Problem(4, 2, 300, 64)
    ok = dict(q=torch.zeros(4, 300, 64, dtype=torch.bfloat16), k=torch.zeros(2, 300, 64, dtype=torch.bfloat16),
              v=torch.zeros(2, 300, 64, dtype=torch.bfloat16), modality=torch.zeros(300, dtype=torch.uint8),
              o=torch.zeros(4, 300, 64, dtype=torch.bfloat16), lse=torch.zeros(4, 300))
    _check_io(pb, **ok)
    bad = [("q", torch.zeros(4, 300, 64, dtype=torch.float16)), ("q", torch.zeros(300, 4, 64, dtype=torch.bfloat16)),
           ("k", torch.zeros(4, 300, 64, dtype=torch.bfloat16)), ("modality", torch.zeros(300, dtype=torch.int64)),
           ("lse", torch.zeros(4, 300, dtype=torch.float64)), ("o", torch.zeros(4, 300, 128, dtype=torch.bfloat16))]
    for name, t in bad:
        with pytest.raises((TypeError, ValueError)):
            _check_io(pb, **dict(ok, **{name: t}))


def test_plan_rejects_32bit_overflow():
    """A config whose gathered spaces exceed 32-bit row indexing is rejected on the host."""
    # many searched-stride grid heads with slash lines at the largest S that passes check_problem
    pb = Problem(16, 16, (1 << 26) - 1024, 128)   # (S + 512) * H <= 2^30 passes check_problem
    heads = [HeadConfig.no_boundary(grid(0, True, True, True, stride_min=1, stride_max=1024))] * 16
    assert _ws(pb, heads) == 0
    from paper_2504_16083_b200.mmi import lib
    assert b"32-bit" in lib().mmi_last_error()


def test_plan_cache_is_stable():
    """The cached plan (built once per distinct config) gives the same sizes as a fresh one."""
    wl = build_workload(1)
    a = _ws(wl.problem, wl.heads)
    for _ in range(3):
        assert _ws(wl.problem, wl.heads) == a
    for i in range(20):   # more distinct configs than the cache keeps: eviction path
        assert _ws(Problem(1, 1, 1000 + i, 64), [HeadConfig.no_boundary(full())]) > 0
    assert _ws(wl.problem, wl.heads) == a
