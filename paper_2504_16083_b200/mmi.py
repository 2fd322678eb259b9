"""Thin ctypes binding of include/mmi.h (argument marshalling only).

Every step of the hot path runs in libmmi.so (CUDA kernels for sm_100a); this
module only converts torch tensors / config dataclasses to pointers and C
structs.  There is no CPU fallback: if the shared library or a CUDA device is
missing, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import torch

from synth.config import HeadConfig, Pattern, Problem, MAX_MOD

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MMI_LIB") or os.path.join(_HERE, "libmmi.so")  # MMI_LIB: an alternative in-tree build

MMI_OK = 0
STATUS = {0: "MMI_OK", 1: "MMI_E_INVALID", 2: "MMI_E_SHAPE", 3: "MMI_E_CONFIG", 4: "MMI_E_UNSUPPORTED",
          5: "MMI_E_WORKSPACE", 6: "MMI_E_CUDA"}


class MMIError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class c_pattern(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("sink", ctypes.c_int32), ("local", ctypes.c_int32),
                ("n_vertical", ctypes.c_int32), ("n_slash", ctypes.c_int32), ("stride", ctypes.c_int32),
                ("stride_min", ctypes.c_int32), ("stride_max", ctypes.c_int32),
                ("use_hline", ctypes.c_uint8), ("use_vline", ctypes.c_uint8), ("use_slash", ctypes.c_uint8),
                ("_pad", ctypes.c_uint8), ("bottom", ctypes.c_int32)]


class c_head_config(ctypes.Structure):
    _fields_ = [("boundary", ctypes.c_int32), ("intra", c_pattern * MAX_MOD),
                ("pair", (c_pattern * MAX_MOD) * MAX_MOD)]


class c_natten_config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("T", "Hh", "Ww", "kt", "kh", "kw", "bt", "bh", "bw")]


class c_problem(ctypes.Structure):
    _fields_ = [("n_heads", ctypes.c_int32), ("n_kv_heads", ctypes.c_int32), ("seq_len", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("n_modalities", ctypes.c_int32), ("last_q", ctypes.c_int32),
                ("block", ctypes.c_int32), ("scale", ctypes.c_float)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32
        P, C = ctypes.POINTER(c_problem), ctypes.POINTER(c_head_config)
        L.mmi_workspace_bytes.restype = sz
        L.mmi_workspace_bytes.argtypes = [P, C]
        L.mmi_estimate_index.argtypes = [P, C, vp, vp, vp, vp, sz, vp]
        L.mmi_permute.argtypes = [P, C, vp, sz, vp, vp, vp, vp]
        L.mmi_sparse_prefill.argtypes = [P, C, vp, sz, vp, vp, vp, vp, vp, vp]
        L.mmi_unpermute.argtypes = [P, C, vp, sz, vp, vp, vp]
        L.mmi_dense_prefill.argtypes = [P, vp, vp, vp, vp, vp, vp]
        L.mmi_export_index.argtypes = [P, C, vp, sz, i32, vp, ctypes.POINTER(sz), vp]
        L.mmi_sparse_fingerprint.argtypes = [P, C, vp, sz, vp, vp, vp, vp, vp]
        L.mmi_plan_stats.argtypes = [P, C, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
        L.mmi_traffic_stats.argtypes = [P, C, vp, sz, ctypes.POINTER(ctypes.c_int64), vp]
        L.mmi_workspace_flags.argtypes = [P, C, vp, sz, ctypes.POINTER(ctypes.c_uint32), vp]
        NC = ctypes.POINTER(c_natten_config)
        L.mmi_natten_workspace_bytes.restype = sz
        L.mmi_natten_workspace_bytes.argtypes = [P, NC]
        L.mmi_natten_prefill.argtypes = [P, NC, vp, sz, vp, vp, vp, vp, vp, vp]
        L.mmi_natten_fingerprint.argtypes = [P, NC, vp, sz, vp, vp, vp, vp, vp]
        L.mmi_natten_prefill.restype = ctypes.c_int
        L.mmi_natten_fingerprint.restype = ctypes.c_int
        L.mmi_natten_last_error.restype = ctypes.c_char_p
        L.mmi_topk_coverage_scratch_bytes.restype = sz
        L.mmi_topk_coverage_scratch_bytes.argtypes = [P, i32]
        L.mmi_topk_coverage.argtypes = [P, vp, vp, vp, i32, ctypes.c_float, vp, vp, sz, vp]
        L.mmi_last_error.restype = ctypes.c_char_p
        L.mmi_version.restype = ctypes.c_char_p
        for fn in ("mmi_estimate_index", "mmi_permute", "mmi_sparse_prefill", "mmi_unpermute",
                   "mmi_dense_prefill", "mmi_export_index", "mmi_sparse_fingerprint", "mmi_plan_stats",
                   "mmi_traffic_stats", "mmi_workspace_flags", "mmi_topk_coverage"):
            getattr(L, fn).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(st: int):
    if st != MMI_OK:
        raise MMIError(st, lib().mmi_last_error().decode())


def to_c_pattern(p: Pattern) -> c_pattern:
    return c_pattern(p.kind, p.sink, p.local, p.n_vertical, p.n_slash, p.stride, p.stride_min, p.stride_max,
                     int(p.use_hline), int(p.use_vline), int(p.use_slash), 0, p.bottom)


def to_c_configs(cfgs: Sequence[HeadConfig]):
    arr = (c_head_config * len(cfgs))()
    for i, c in enumerate(cfgs):
        arr[i].boundary = c.boundary
        for m in range(MAX_MOD):
            arr[i].intra[m] = to_c_pattern(c.intra[m])
            for b in range(MAX_MOD):
                arr[i].pair[m][b] = to_c_pattern(c.pair[m][b])
    return arr


def to_c_problem(pb: Problem) -> c_problem:
    return c_problem(pb.n_heads, pb.n_kv_heads, pb.seq_len, pb.head_dim, pb.n_modalities, pb.last_q, pb.block,
                     float(pb.scale))


def _ptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device tensor expected")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need_cuda(*ts):
    if not torch.cuda.is_available():
        raise RuntimeError("mmi: CUDA device required (no CPU fallback)")
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise ValueError("mmi: contiguous CUDA tensors required")


def _check_tensor(name, t, dtype, shape):
    """The C ABI reads raw pointers: dtype and shape are checked here (include/mmi.h layouts)."""
    if t is None:
        return
    if t.dtype != dtype:
        raise TypeError(f"mmi: {name} must be {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"mmi: {name} must have shape {tuple(shape)}, got {tuple(t.shape)}")


def _check_io(pb: Problem, q=None, k=None, v=None, modality=None, o=None, lse=None):
    H, Hkv, S, D = pb.n_heads, pb.n_kv_heads, pb.seq_len, pb.head_dim
    _check_tensor("q", q, torch.bfloat16, (H, S, D))
    _check_tensor("k", k, torch.bfloat16, (Hkv, S, D))
    _check_tensor("v", v, torch.bfloat16, (Hkv, S, D))
    _check_tensor("modality", modality, torch.uint8, (S,))
    _check_tensor("o", o, torch.bfloat16, (H, S, D))
    _check_tensor("lse", lse, torch.float32, (H, S))


# ------------------------------------------------------------------ C ABI mirrors
def mmi_workspace_bytes(pb: Problem, cfgs: Sequence[HeadConfig]) -> int:
    return int(lib().mmi_workspace_bytes(ctypes.byref(to_c_problem(pb)), to_c_configs(cfgs)))


def mmi_plan_stats(pb: Problem, cfgs: Sequence[HeadConfig]) -> dict:
    """Host-only plan sizes (for algorithmic-traffic reporting)."""
    out = (ctypes.c_int64 * 6)()
    _check(lib().mmi_plan_stats(ctypes.byref(to_c_problem(pb)), to_c_configs(cfgs), out, 6))
    return dict(qg_rows=out[0], kg_rows=out[1], merge_heads=out[2], slabs=out[3], part_rows=out[4], fused=out[5])


def mmi_traffic_stats(pb: Problem, cfgs: Sequence[HeadConfig], ws, stream=None) -> dict:
    """Rows moved by the permute step (reporting only; synchronises)."""
    out = (ctypes.c_int64 * 4)()
    _check(lib().mmi_traffic_stats(ctypes.byref(to_c_problem(pb)), to_c_configs(cfgs), _ptr(ws), ws.numel() * ws.element_size(), out,
                                   _stream(stream)))
    return dict(qg_read=out[0], qg_written=out[1], kg_read=out[2], kg_written=out[3])


def mmi_estimate_index(pb, cfgs, q, k, modality, ws, stream=None):
    _need_cuda(q, k, modality, ws)
    _check_io(pb, q=q, k=k, modality=modality)
    _check(lib().mmi_estimate_index(ctypes.byref(to_c_problem(pb)), to_c_configs(cfgs), _ptr(q), _ptr(k),
                                    _ptr(modality), _ptr(ws), ws.numel() * ws.element_size(), _stream(stream)))


def mmi_permute(pb, cfgs, ws, q, k, v, stream=None):
    _need_cuda(q, k, v, ws)
    _check_io(pb, q=q, k=k, v=v)
    _check(lib().mmi_permute(ctypes.byref(to_c_problem(pb)), to_c_configs(cfgs), _ptr(ws),
                             ws.numel() * ws.element_size(), _ptr(q), _ptr(k), _ptr(v), _stream(stream)))


def mmi_sparse_prefill(pb, cfgs, ws, q, k, v, o, lse=None, stream=None):
    _need_cuda(q, k, v, o, ws, lse)
    _check_io(pb, q=q, k=k, v=v, o=o, lse=lse)
    _check(lib().mmi_sparse_prefill(ctypes.byref(to_c_problem(pb)), to_c_configs(cfgs), _ptr(ws),
                                    ws.numel() * ws.element_size(), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                                    _stream(stream)))


def mmi_unpermute(pb, cfgs, ws, o, lse=None, stream=None):
    _need_cuda(o, ws, lse)
    _check_io(pb, o=o, lse=lse)
    _check(lib().mmi_unpermute(ctypes.byref(to_c_problem(pb)), to_c_configs(cfgs), _ptr(ws),
                               ws.numel() * ws.element_size(), _ptr(o), _ptr(lse), _stream(stream)))


def mmi_dense_prefill(pb, q, k, v, o, lse=None, stream=None):
    _need_cuda(q, k, v, o, lse)
    _check_io(pb, q=q, k=k, v=v, o=o, lse=lse)
    _check(lib().mmi_dense_prefill(ctypes.byref(to_c_problem(pb)), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                                   _stream(stream)))


def mmi_sparse_fingerprint(pb, cfgs, ws, q, k, v, fp, stream=None):
    _need_cuda(q, k, v, ws, fp)
    _check(lib().mmi_sparse_fingerprint(ctypes.byref(to_c_problem(pb)), to_c_configs(cfgs), _ptr(ws),
                                        ws.numel() * ws.element_size(), _ptr(q), _ptr(k), _ptr(v), _ptr(fp),
                                        _stream(stream)))


def mmi_workspace_flags(pb, cfgs, ws, stream=None) -> int:
    """DIAGNOSTIC (synchronises): device-side error flags of the last estimate on ws
    (1 = a modality label >= n_modalities, 2 = segment-bound overflow)."""
    f = ctypes.c_uint32(0)
    _check(lib().mmi_workspace_flags(ctypes.byref(to_c_problem(pb)), to_c_configs(cfgs), _ptr(ws),
                                     ws.numel() * ws.element_size(), ctypes.byref(f), _stream(stream)))
    return int(f.value)


def mmi_topk_coverage(pb, q, k, rows, target=0.95, stream=None) -> torch.Tensor:
    """ANALYSIS: [H, n_rows] fraction of causal keys whose top mass reaches `target` (C ABI)."""
    _need_cuda(q, k, rows)
    _check_io(pb, q=q, k=k)
    if rows.dtype != torch.int32:
        raise TypeError("mmi: rows must be int32")
    n = rows.numel()
    out = torch.empty((pb.n_heads, n), dtype=torch.float32, device=q.device)
    c_pb = to_c_problem(pb)
    nb = int(lib().mmi_topk_coverage_scratch_bytes(ctypes.byref(c_pb), n))
    scratch = torch.empty(nb, dtype=torch.uint8, device=q.device)
    _check(lib().mmi_topk_coverage(ctypes.byref(c_pb), _ptr(q), _ptr(k), _ptr(rows), n, float(target), _ptr(out),
                                   _ptr(scratch), nb, _stream(stream)))
    return out


def mmi_export_index(pb, cfgs, ws, head: int, stream=None) -> torch.Tensor:
    """TEST ONLY: int32 words of head `head`'s index (layout: see api.cu export)."""
    n = ctypes.c_size_t(0)
    c_pb, c_cfg = to_c_problem(pb), to_c_configs(cfgs)
    sz = ws.numel() * ws.element_size()
    _check(lib().mmi_export_index(ctypes.byref(c_pb), c_cfg, _ptr(ws), sz, head, None, ctypes.byref(n),
                                  _stream(stream)))
    buf = torch.zeros(int(n.value), dtype=torch.int32)
    _check(lib().mmi_export_index(ctypes.byref(c_pb), c_cfg, _ptr(ws), sz, head,
                                  ctypes.c_void_p(buf.data_ptr()), ctypes.byref(n), _stream(stream)))
    return buf


# ------------------------------------------------------------------ convenience
class SparsePrefill:
    """One layer's sparse pre-fill: owns the workspace (or uses a caller's buffer of at least
    `workspace_bytes()`) and the marshalled C structs; each call runs the four C-ABI calls on the
    current stream."""

    def __init__(self, pb: Problem, cfgs: List[HeadConfig], device="cuda", ws: Optional[torch.Tensor] = None):
        self.pb, self.cfgs = pb, list(cfgs)
        self.c_pb = to_c_problem(pb)
        self.c_cfg = to_c_configs(self.cfgs)
        nbytes = self.workspace_bytes()
        if ws is None:
            ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
        elif ws.numel() * ws.element_size() < nbytes:
            raise MMIError(5, "workspace buffer smaller than mmi_workspace_bytes")
        self.ws = ws
        self.ws_bytes = ws.numel() * ws.element_size()

    def workspace_bytes(self) -> int:
        nbytes = int(lib().mmi_workspace_bytes(ctypes.byref(self.c_pb), self.c_cfg))
        if nbytes == 0:
            raise MMIError(1, lib().mmi_last_error().decode())
        return nbytes

    def estimate(self, q, k, modality, stream=None):
        _need_cuda(q, k, modality)
        _check_io(self.pb, q=q, k=k, modality=modality)
        _check(lib().mmi_estimate_index(ctypes.byref(self.c_pb), self.c_cfg, _ptr(q), _ptr(k), _ptr(modality),
                                        _ptr(self.ws), self.ws_bytes, _stream(stream)))

    def permute(self, q, k, v, stream=None):
        _need_cuda(q, k, v)
        _check_io(self.pb, q=q, k=k, v=v)
        _check(lib().mmi_permute(ctypes.byref(self.c_pb), self.c_cfg, _ptr(self.ws), self.ws_bytes, _ptr(q), _ptr(k),
                                 _ptr(v), _stream(stream)))

    def sparse(self, q, k, v, o, lse=None, stream=None):
        _need_cuda(q, k, v, o, lse)
        _check_io(self.pb, q=q, k=k, v=v, o=o, lse=lse)
        _check(lib().mmi_sparse_prefill(ctypes.byref(self.c_pb), self.c_cfg, _ptr(self.ws), self.ws_bytes, _ptr(q),
                                        _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _stream(stream)))

    def unpermute(self, o, lse=None, stream=None):
        _need_cuda(o, lse)
        _check_io(self.pb, o=o, lse=lse)
        _check(lib().mmi_unpermute(ctypes.byref(self.c_pb), self.c_cfg, _ptr(self.ws), self.ws_bytes, _ptr(o),
                                   _ptr(lse), _stream(stream)))

    def __call__(self, q, k, v, modality, o=None, lse=None, stream=None):
        pb = self.pb
        _need_cuda(q, k, v, modality, o, lse)
        if o is None:
            o = torch.empty((pb.n_heads, pb.seq_len, pb.head_dim), dtype=torch.bfloat16, device=q.device)
        self.estimate(q, k, modality, stream)
        self.permute(q, k, v, stream)
        self.sparse(q, k, v, o, lse, stream)
        self.unpermute(o, lse, stream)
        return o

    def flags(self, stream=None) -> int:
        """DIAGNOSTIC (synchronises): device-side error flags of the last estimate."""
        return mmi_workspace_flags(self.pb, self.cfgs, self.ws, stream)

    def head_tiles(self) -> List[int]:
        """Computed 128x128 key tiles per head of the last index (bench helper: synchronises)."""
        import struct
        out = []
        for h in range(self.pb.n_heads):
            w = mmi_export_index(self.pb, self.cfgs, self.ws, h).tolist()
            out.append(struct.unpack("<q", struct.pack("<ii", w[-3], w[-2]))[0])
        return out

    def total_tiles(self) -> int:
        """Computed key tiles of the last index (TEST/bench helper: synchronises)."""
        return sum(self.head_tiles())


def dense_prefill(pb: Problem, q, k, v, o=None, lse=None, stream=None):
    if o is None:
        o = torch.empty((pb.n_heads, pb.seq_len, pb.head_dim), dtype=torch.bfloat16, device=q.device)
    mmi_dense_prefill(pb, q, k, v, o, lse, stream)
    return o


class HostSparsePrefill:
    """End-to-end sparse pre-fill from pinned HOST buffers: each call copies the
    step's inputs host -> device, runs the four C-ABI calls and copies O back.

    Heads are independent (Alg.1-3 act per head), so the layer is processed in chunks of
    heads (a KV group's K and V are copied once, before its first chunk).  Three streams:
    host -> device copies in chunk order, the chunks' library calls in chunk order (one shared
    workspace), device -> host copies of each chunk's O -- chunk c computes while chunk c + 1 is
    copied in and chunk c - 1 copied out (the copy engines are full duplex).  Every chunk is the
    same library call on a sub-problem, so O is bit-identical to the one-shot call.  The
    caller's stream waits for the last copy before returning.

    Chunking: with n_chunks=None the first call runs one chunk per KV group and times its
    compute against its input copy; a copy-bound layer then switches to chunks of about 16K
    tokens x heads (the last chunk's compute and output copy, the only parts not hidden under
    the input copy, get short), a compute-bound one keeps whole groups (fewer, longer kernels).
    Measured on one B200 (ms/layer): 1M 4 / 8 / 14 / 28 chunks 236 / 215 / 204 / 199;
    128K 30.1 / 28.7 / 30.4 / 36.6; 256K 229 / 238 / 268 / 255; 512K 257 / 263 / 313 / 382."""

    TOKENS_PER_CHUNK = 16384  # fine chunking: about this many tokens x heads per chunk

    def __init__(self, pb: Problem, cfgs: List[HeadConfig], device="cuda", n_chunks: Optional[int] = None):
        H, Hkv, S, D = pb.n_heads, pb.n_kv_heads, pb.seq_len, pb.head_dim
        self.pb, self.cfgs, self.device = pb, list(cfgs), device
        self.ws = None
        self.fixed = n_chunks is not None
        self.chunks = self._build(max(1, min(H, n_chunks)) if n_chunks else Hkv)
        self.fine = min(H, max(Hkv, S // self.TOKENS_PER_CHUNK))
        self.q = torch.empty((H, S, D), dtype=torch.bfloat16, device=device)
        self.k = torch.empty((Hkv, S, D), dtype=torch.bfloat16, device=device)
        self.v = torch.empty((Hkv, S, D), dtype=torch.bfloat16, device=device)
        self.lab = torch.empty((S,), dtype=torch.uint8, device=device)
        self.o = torch.empty((H, S, D), dtype=torch.bfloat16, device=device)
        self.s_in, self.s_cmp, self.s_out = (torch.cuda.Stream(device=device) for _ in range(3))

    def _build(self, n: int):
        pb, cfgs = self.pb, self.cfgs
        H, Hkv, S, D = pb.n_heads, pb.n_kv_heads, pb.seq_len, pb.head_dim
        G = H // Hkv
        if n <= Hkv:  # whole KV groups per chunk
            bounds = [(c * Hkv // n * G, (c + 1) * Hkv // n * G) for c in range(n)]
        else:  # every group split into ceil(n / Hkv) head ranges
            per = -(-n // Hkv)
            bounds = [(g * G + i * G // per, g * G + (i + 1) * G // per) for g in range(Hkv) for i in range(per)]
        chunks = []
        for h0, h1 in bounds:
            if h1 <= h0:
                continue
            g0, g1 = h0 // G, (h1 - 1) // G + 1
            sub = Problem(h1 - h0, g1 - g0, S, D, pb.n_modalities, pb.last_q, pb.block, pb.scale)
            sp = SparsePrefill.__new__(SparsePrefill)
            sp.pb, sp.cfgs = sub, cfgs[h0:h1]
            sp.c_pb, sp.c_cfg = to_c_problem(sub), to_c_configs(sp.cfgs)
            chunks.append(dict(h0=h0, h1=h1, g0=g0, g1=g1, sp=sp))
        # one workspace for every chunk: the chunks run in order on the compute stream
        need = max(ch["sp"].workspace_bytes() for ch in chunks)
        if self.ws is None or self.ws.numel() < need:
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        for ch in chunks:
            ch["sp"].ws, ch["sp"].ws_bytes = self.ws, self.ws.numel()
        for ch in getattr(self, "chunks", []):  # earlier chunking shares the (possibly new) buffer
            ch["sp"].ws, ch["sp"].ws_bytes = self.ws, self.ws.numel()
        return chunks

    def h2d_bytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (self.q, self.k, self.v, self.lab))

    def d2h_bytes(self) -> int:
        return self.o.numel() * self.o.element_size()

    def __call__(self, q_h, k_h, v_h, lab_h, o_h, stream=None):
        caller = stream if stream is not None else torch.cuda.current_stream()
        decide = not self.fixed and len(self.chunks) != self.fine
        timing = decide and not getattr(self, "_decided", False)
        start = torch.cuda.Event(enable_timing=timing)
        start.record(caller)
        for st in (self.s_in, self.s_cmp, self.s_out):
            st.wait_event(start)
        kv_done = -1  # K / V of groups < kv_done are on the device
        marks = []
        with torch.cuda.stream(self.s_in):
            self.lab.copy_(lab_h, non_blocking=True)
        for ch in self.chunks:
            h0, h1, g0, g1 = ch["h0"], ch["h1"], ch["g0"], ch["g1"]
            with torch.cuda.stream(self.s_in):
                if g1 > kv_done:
                    a = max(g0, kv_done)
                    self.k[a:g1].copy_(k_h[a:g1], non_blocking=True)
                    self.v[a:g1].copy_(v_h[a:g1], non_blocking=True)
                    kv_done = g1
                self.q[h0:h1].copy_(q_h[h0:h1], non_blocking=True)
                ready = torch.cuda.Event(enable_timing=timing)
                ready.record(self.s_in)
            self.s_cmp.wait_event(ready)
            with torch.cuda.stream(self.s_cmp):
                c0 = torch.cuda.Event(enable_timing=timing)
                c0.record(self.s_cmp)
                ch["sp"](self.q[h0:h1], self.k[g0:g1], self.v[g0:g1], self.lab, o=self.o[h0:h1], stream=self.s_cmp)
                computed = torch.cuda.Event(enable_timing=timing)
                computed.record(self.s_cmp)
            marks.append((ready, c0, computed))
            self.s_out.wait_event(computed)
            with torch.cuda.stream(self.s_out):
                o_h[h0:h1].copy_(self.o[h0:h1], non_blocking=True)
        done = torch.cuda.Event()
        done.record(self.s_out)
        caller.wait_event(done)
        if timing:  # first call: copy-bound -> fine chunks (synchronises once)
            done.synchronize()
            copy_ms = start.elapsed_time(marks[-1][0])
            compute_ms = sum(c0.elapsed_time(c1) for _, c0, c1 in marks)
            self._decided = True
            if compute_ms < 0.6 * copy_ms:
                self.chunks = self._build(self.fine)
        return o_h


class NattenPrefill:
    """Permuted NATTEN / DiT neighborhood attention: owns the workspace; each call
    runs mmi_natten_prefill on the current stream."""

    def __init__(self, pb: Problem, nc, device="cuda"):
        self.pb, self.nc = pb, nc
        self.c_pb = to_c_problem(pb)
        self.c_nc = c_natten_config(nc.T, nc.Hh, nc.Ww, nc.kt, nc.kh, nc.kw, nc.bt, nc.bh, nc.bw)
        nbytes = int(lib().mmi_natten_workspace_bytes(ctypes.byref(self.c_pb), ctypes.byref(self.c_nc)))
        if nbytes == 0:
            raise MMIError(3, lib().mmi_natten_last_error().decode())
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=device)

    def _st(self, st):
        if st != MMI_OK:
            raise MMIError(st, lib().mmi_natten_last_error().decode())

    def __call__(self, q, k, v, o=None, lse=None, stream=None):
        pb = self.pb
        _need_cuda(q, k, v, o, lse)
        _check_io(pb, q=q, k=k, v=v, o=o, lse=lse)
        if o is None:
            o = torch.empty((pb.n_heads, pb.seq_len, pb.head_dim), dtype=torch.bfloat16, device=q.device)
        self._st(lib().mmi_natten_prefill(ctypes.byref(self.c_pb), ctypes.byref(self.c_nc), _ptr(self.ws),
                                          self.ws.numel(), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                                          _stream(stream)))
        return o

    def fingerprint(self, q, k, v, fp, stream=None):
        _need_cuda(q, k, v, fp)
        self._st(lib().mmi_natten_fingerprint(ctypes.byref(self.c_pb), ctypes.byref(self.c_nc), _ptr(self.ws),
                                              self.ws.numel(), _ptr(q), _ptr(k), _ptr(v), _ptr(fp), _stream(stream)))
