"""B200-native (sm_100a) MMInference sparse pre-fill: C-ABI library libmmi.so
(include/mmi.h) + this thin ctypes binding.  See DESIGN.md."""
from .mmi import (  # noqa: F401
    SparsePrefill, HostSparsePrefill, NattenPrefill, dense_prefill, lib, MMIError,
    mmi_workspace_bytes, mmi_estimate_index, mmi_permute, mmi_sparse_prefill, mmi_unpermute,
    mmi_dense_prefill, mmi_export_index, mmi_sparse_fingerprint, mmi_plan_stats, mmi_traffic_stats,
    mmi_workspace_flags, mmi_topk_coverage,
)
