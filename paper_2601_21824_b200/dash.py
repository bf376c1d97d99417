"""Thin ctypes binding of libdash.so (include/dash.h).

Argument marshalling only: every step of the attention path runs in the
library's sm_100a kernels.  torch is used for device memory and the current
stream.  There is no CPU fallback: if libdash.so is missing or fails to load,
importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# DASH_LIB_PATH: an experiment build of the same library (scripts/build_variant.py)
LIB_PATH = os.environ.get("DASH_LIB_PATH") or os.path.join(_HERE, "libdash.so")

NAIVE, DESCENDING, SHIFT, AUTO = 0, 1, 2, 3
FULL, CAUSAL = 0, 1
SCHEDULES = {"naive": NAIVE, "descending": DESCENDING, "shift": SHIFT, "auto": AUTO}

OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_WORKSPACE, ERR_CUDA, ERR_DEADLOCK = range(6)


class DashError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {status_string(status)} ({status})")
        self.status = status


class Shape(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int), ("seqlen", ctypes.c_int), ("heads", ctypes.c_int),
                ("head_dim", ctypes.c_int), ("softmax_scale", ctypes.c_float)]


class DagParams(ctypes.Structure):
    _fields_ = [("n_heads", ctypes.c_int), ("n_sm", ctypes.c_int),
                ("c", ctypes.c_int64), ("r", ctypes.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(python -m paper_2601_21824_b200.build)")
    lib = ctypes.CDLL(LIB_PATH)
    vp, i, sz, st = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_int
    SP = ctypes.POINTER(Shape)
    lib.dash_status_string.restype = ctypes.c_char_p
    lib.dash_status_string.argtypes = [st]
    lib.dash_version.restype = ctypes.c_char_p
    lib.dash_attn_fwd.restype = st
    lib.dash_attn_fwd.argtypes = [SP, vp, vp, vp, vp, vp, i, vp]
    lib.dash_attn_bwd_workspace_bytes.restype = sz
    lib.dash_attn_bwd_workspace_bytes.argtypes = [SP, i, i, i]
    lib.dash_attn_bwd.restype = st
    lib.dash_attn_bwd.argtypes = [SP, vp, vp, vp, vp, vp, vp, vp, vp, vp, i, i, i, vp, sz, vp]
    lib.dash_attn_bwd_trace.restype = st
    lib.dash_attn_bwd_trace.argtypes = [SP, vp, vp, vp, vp, vp, vp, vp, vp, vp, i, i, i, vp, sz,
                                        vp, i, vp]
    lib.dash_attn_bwd_resolve_schedule.restype = i
    lib.dash_attn_bwd_resolve_schedule.argtypes = [SP, i, i]
    lib.dash_attn_bwd_acc_split.restype = i
    lib.dash_attn_bwd_acc_split.argtypes = [SP, i, i]
    lib.dash_attn_bwd_set_acc_split.restype = st
    lib.dash_attn_bwd_set_acc_split.argtypes = [i]
    lib.dash_attn_bwd_dump_bytes.restype = sz
    lib.dash_attn_bwd_dump_bytes.argtypes = [SP, i, i]
    lib.dash_attn_bwd_dump.restype = st
    lib.dash_attn_bwd_dump.argtypes = [SP, vp, vp, vp, vp, vp, vp, vp, vp, vp, i, i, i, vp, sz,
                                       vp, sz, vp]
    lib.dash_attn_bwd_host_workspace_bytes.restype = sz
    lib.dash_attn_bwd_host_workspace_bytes.argtypes = [SP, i, i, i]
    lib.dash_last_cuda_error.restype = i
    lib.dash_last_cuda_error.argtypes = []
    lib.dash_attn_bwd_host.restype = st
    lib.dash_attn_bwd_host.argtypes = [SP, vp, vp, vp, vp, vp, vp, vp, vp, vp, i, i, i, vp, sz, vp]
    lib.dash_check_workspace.restype = st
    lib.dash_check_workspace.argtypes = [SP, i, i, i, vp, vp]
    lib.dash_schedule_critical_path.restype = st
    lib.dash_schedule_critical_path.argtypes = [i, i, i, i, ctypes.POINTER(DagParams),
                                                ctypes.POINTER(ctypes.c_int64)]
    ip = ctypes.POINTER(ctypes.c_int32)
    lib.dash_schedule_table.restype = st
    lib.dash_schedule_table.argtypes = [i, i, i, i, ip, ip, ip, ip, ip, ip]
    lib.dash_profile_begin.restype = st
    lib.dash_profile_begin.argtypes = []
    dp = ctypes.POINTER(ctypes.c_double)
    lib.dash_profile_end.restype = st
    lib.dash_profile_end.argtypes = [dp, dp, dp, ctypes.POINTER(ctypes.c_int)]
    lib.dash_attn_bwd_launches.restype = i
    lib.dash_attn_bwd_launches.argtypes = [i, i, i]
    lib.dash_attn_bwd_set_watchdog.restype = st
    lib.dash_attn_bwd_set_watchdog.argtypes = [ctypes.c_longlong]
    lib.dash_attn_bwd_inject_fault.restype = st
    lib.dash_attn_bwd_inject_fault.argtypes = [i]
    lib.dash_attn_bwd_tile.restype = i
    lib.dash_attn_bwd_tile.argtypes = [SP, i, i]
    lib.dash_attn_bwd_set_tile.restype = st
    lib.dash_attn_bwd_set_tile.argtypes = [i]
    lib.dash_attn_bwd_set_plane_budget.restype = st
    lib.dash_attn_bwd_set_plane_budget.argtypes = [ctypes.c_size_t]
    lib.dash_attn_bwd_head_chunk.restype = i
    lib.dash_attn_bwd_head_chunk.argtypes = [SP, i, i, i]
    lib.dash_attn_bwd_set_fused_dq.restype = st
    lib.dash_attn_bwd_set_fused_dq.argtypes = [i]
    lib.dash_attn_bwd_fused_dq.restype = i
    lib.dash_attn_bwd_fused_dq.argtypes = []
    lib.dash_attn_bwd_launch_count.restype = i
    lib.dash_attn_bwd_launch_count.argtypes = [SP, i, i, i]
    return lib


_lib = _load()


def lib():
    return _lib


def status_string(s: int) -> str:
    return _lib.dash_status_string(int(s)).decode()


def version() -> str:
    return _lib.dash_version().decode()


def _check(status: int, what: str):
    if status != OK:
        if status == ERR_CUDA:
            what = f"{what} (cudaError {_lib.dash_last_cuda_error()})"
        raise DashError(status, what)


def _shape(q: torch.Tensor, scale):
    B, N, H, d = q.shape
    return Shape(B, N, H, d, float(scale) if scale else 0.0)


def _stream(t: torch.Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _sched(s):
    return SCHEDULES[s] if isinstance(s, str) else int(s)


def attn_fwd(q, k, v, causal: bool, scale=None, out=None, lse=None):
    """dash_attn_fwd: returns (o [B,N,H,d] bf16, lse [B,H,N] fp32)."""
    B, N, H, d = q.shape
    o = torch.empty_like(q) if out is None else out
    lse = torch.empty((B, H, N), device=q.device, dtype=torch.float32) if lse is None else lse
    shp = _shape(q, scale)
    _check(_lib.dash_attn_fwd(ctypes.byref(shp), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                              int(causal), _stream(q)), "dash_attn_fwd")
    return o, lse


def workspace_bytes(shape_bnhd, causal: bool, schedule=NAIVE, deterministic=True, scale=None) -> int:
    B, N, H, d = shape_bnhd
    shp = Shape(B, N, H, d, float(scale) if scale else 0.0)
    return int(_lib.dash_attn_bwd_workspace_bytes(ctypes.byref(shp), int(causal), _sched(schedule),
                                                  int(deterministic)))


def alloc_workspace(shape_bnhd, causal: bool, schedule=NAIVE, deterministic=True, device="cuda"):
    n = workspace_bytes(shape_bnhd, causal, schedule, deterministic)
    return torch.empty(n, dtype=torch.uint8, device=device)


def attn_bwd(q, k, v, o, dout, lse, causal: bool, schedule=NAIVE, deterministic: bool = True,
             scale=None, workspace=None, out=None):
    """dash_attn_bwd: returns (dq, dk, dv), bf16 [B,N,H,d]."""
    sched = _sched(schedule)
    if workspace is None:
        workspace = alloc_workspace(q.shape, causal, sched, deterministic, q.device)
    if out is None:
        dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    else:
        dq, dk, dv = out
    shp = _shape(q, scale)
    _check(_lib.dash_attn_bwd(ctypes.byref(shp), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(dout),
                              _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv), int(causal), sched,
                              int(deterministic), _ptr(workspace), workspace.numel(), _stream(q)),
           "dash_attn_bwd")
    return dq, dk, dv


def attn_bwd_trace(q, k, v, o, dout, lse, causal: bool, schedule, deterministic, trace_cap=512,
                   scale=None, workspace=None, out=None):
    """dash_attn_bwd_trace: returns ((dq, dk, dv), trace [grid, trace_cap, 32] int64 on device)."""
    sched = _sched(schedule)
    if workspace is None:
        workspace = alloc_workspace(q.shape, causal, sched, deterministic, q.device)
    dq, dk, dv = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)) if out is None else out
    props = torch.cuda.get_device_properties(q.device)
    trace = torch.zeros((props.multi_processor_count, trace_cap, 32), dtype=torch.int64,
                        device=q.device)
    shp = _shape(q, scale)
    _check(_lib.dash_attn_bwd_trace(ctypes.byref(shp), _ptr(q), _ptr(k), _ptr(v), _ptr(o),
                                    _ptr(dout), _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv),
                                    int(causal), sched, int(deterministic), _ptr(workspace),
                                    workspace.numel(), _ptr(trace), trace_cap, _stream(q)),
           "dash_attn_bwd_trace")
    return (dq, dk, dv), trace


def resolve_schedule(shape_bnhd, causal: bool, schedule) -> str:
    """dash_attn_bwd_resolve_schedule: the paper schedule `schedule` runs as."""
    B, N, H, d = shape_bnhd
    shp = Shape(B, N, H, d, 0.0)
    r = int(_lib.dash_attn_bwd_resolve_schedule(ctypes.byref(shp), int(causal), _sched(schedule)))
    if r < 0:
        raise DashError(ERR_INVALID_ARG, "dash_attn_bwd_resolve_schedule")
    return {NAIVE: "naive", DESCENDING: "descending", SHIFT: "shift"}[r]


def acc_split(shape_bnhd=None, causal: bool = True, schedule="auto") -> int:
    """dash_attn_bwd_acc_split: the W a deterministic backward with this shape
    uses (AMB-27); shape None returns the setting (0 = automatic)."""
    if shape_bnhd is None:
        return int(_lib.dash_attn_bwd_acc_split(None, 0, 0))
    B, N, H, d = shape_bnhd
    shp = Shape(B, N, H, d, 0.0)
    return int(_lib.dash_attn_bwd_acc_split(ctypes.byref(shp), int(causal), _sched(schedule)))


def set_acc_split(w: int):
    """dash_attn_bwd_set_acc_split (host-global)."""
    _check(_lib.dash_attn_bwd_set_acc_split(int(w)), "dash_attn_bwd_set_acc_split")


def set_fused_dq(mode: int):
    """dash_attn_bwd_set_fused_dq (host-global): 0 = K4 convert kernel, 1 = in the main
    kernel from N = 2048 (default), 2 = always in the main kernel."""
    _check(_lib.dash_attn_bwd_set_fused_dq(int(mode)), "dash_attn_bwd_set_fused_dq")


def fused_dq() -> int:
    return int(_lib.dash_attn_bwd_fused_dq())


def bwd_launch_count(shape_bnhd, causal=True, schedule="auto", deterministic=True) -> int:
    """dash_attn_bwd_launch_count: device launches of one dash_attn_bwd with these arguments."""
    B, N, H, d = shape_bnhd
    shp = Shape(B, N, H, d, 0.0)
    return int(_lib.dash_attn_bwd_launch_count(ctypes.byref(shp), int(causal), _sched(schedule),
                                               int(deterministic)))


def set_plane_budget(nbytes: int):
    """dash_attn_bwd_set_plane_budget (host-global; 0 = default 4 GiB)."""
    _check(_lib.dash_attn_bwd_set_plane_budget(int(nbytes)), "dash_attn_bwd_set_plane_budget")


def head_chunk(shape_bnhd, causal: bool = True, schedule="auto", deterministic=True) -> int:
    """dash_attn_bwd_head_chunk: flattened heads per launch under the dQ-plane budget."""
    B, N, H, d = shape_bnhd
    shp = Shape(B, N, H, d, 0.0)
    return int(_lib.dash_attn_bwd_head_chunk(ctypes.byref(shp), int(causal), _sched(schedule),
                                             int(deterministic)))


def attn_bwd_dump(q, k, v, o, dout, lse, causal: bool, schedule, deterministic=True, scale=None,
                  workspace=None, out=None):
    """dash_attn_bwd_dump: returns ((dq, dk, dv), partials [B*H, n, N, d] fp32 on device, workspace)."""
    sched = _sched(schedule)
    if workspace is None:
        workspace = alloc_workspace(q.shape, causal, sched, deterministic, q.device)
    dq, dk, dv = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)) if out is None else out
    B, N, H, d = q.shape
    shp = _shape(q, scale)
    nbytes = int(_lib.dash_attn_bwd_dump_bytes(ctypes.byref(shp), int(causal), sched))
    parts = torch.zeros((B * H, N // tile(q.shape, causal, sched), N, d), dtype=torch.float32,
                        device=q.device)
    assert parts.numel() * 4 == nbytes
    _check(_lib.dash_attn_bwd_dump(ctypes.byref(shp), _ptr(q), _ptr(k), _ptr(v), _ptr(o),
                                   _ptr(dout), _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv),
                                   int(causal), sched, int(deterministic), _ptr(workspace),
                                   workspace.numel(), _ptr(parts), nbytes, _stream(q)),
           "dash_attn_bwd_dump")
    return (dq, dk, dv), parts, workspace


def host_workspace_bytes(shape_bnhd, causal: bool, schedule=NAIVE, deterministic=True) -> int:
    B, N, H, d = shape_bnhd
    shp = Shape(B, N, H, d, 0.0)
    return int(_lib.dash_attn_bwd_host_workspace_bytes(ctypes.byref(shp), int(causal),
                                                       _sched(schedule), int(deterministic)))


def attn_bwd_host(q, k, v, o, dout, lse, dq, dk, dv, causal: bool, schedule, deterministic,
                  workspace, scale=None, stream=None):
    """dash_attn_bwd_host: host (pinned) tensors in and out; synchronises."""
    shp = _shape(q, scale)
    s = ctypes.c_void_p(stream if stream is not None else torch.cuda.current_stream().cuda_stream)
    _check(_lib.dash_attn_bwd_host(ctypes.byref(shp), _ptr(q), _ptr(k), _ptr(v), _ptr(o),
                                   _ptr(dout), _ptr(lse), _ptr(dq), _ptr(dk), _ptr(dv),
                                   int(causal), _sched(schedule), int(deterministic),
                                   _ptr(workspace), workspace.numel(), s), "dash_attn_bwd_host")


def check_workspace(q_shape, causal, schedule, deterministic, workspace):
    B, N, H, d = q_shape
    shp = Shape(B, N, H, d, 0.0)
    return int(_lib.dash_check_workspace(ctypes.byref(shp), int(causal), _sched(schedule),
                                         int(deterministic), _ptr(workspace),
                                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))


def schedule_critical_path(schedule, n_q: int, n_kv: int, mask: int, n_heads=None, n_sm=None,
                           c: int = 1, r: int = 1) -> int:
    """dash_schedule_critical_path (host DAG model, §3 of the paper)."""
    out = ctypes.c_int64(0)
    if n_heads is None and n_sm is None and c == 1 and r == 1:
        p = None
    else:
        p = ctypes.byref(DagParams(2 if n_heads is None else n_heads,
                                   n_kv if n_sm is None else n_sm, c, r))
    _check(_lib.dash_schedule_critical_path(_sched(schedule), n_q, n_kv, mask, p,
                                            ctypes.byref(out)), "dash_schedule_critical_path")
    return int(out.value)


def schedule_table(schedule, n_kv: int, mask: int):
    """dash_schedule_table: list of jobs, each a list of (kv, q, rank)."""
    nt, nj = ctypes.c_int32(0), ctypes.c_int32(0)
    st = _lib.dash_schedule_table(_sched(schedule), n_kv, mask, 0, None, None, None, None,
                                  ctypes.byref(nt), ctypes.byref(nj))
    if st not in (OK, ERR_WORKSPACE):
        _check(st, "dash_schedule_table")
    n = nt.value
    arrs = [(ctypes.c_int32 * max(n, 1))() for _ in range(4)]
    _check(_lib.dash_schedule_table(_sched(schedule), n_kv, mask, n, *arrs, ctypes.byref(nt),
                                    ctypes.byref(nj)), "dash_schedule_table")
    jobs = [[] for _ in range(nj.value)]
    for t in range(n):
        jobs[arrs[0][t]].append((arrs[1][t], arrs[2][t], arrs[3][t]))
    return jobs


def profile_begin():
    _check(_lib.dash_profile_begin(), "dash_profile_begin")


def profile_end():
    """Returns (ms_preprocess, ms_main, ms_convert, n_calls) summed over profiled calls."""
    a, b, c, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    _check(_lib.dash_profile_end(ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), ctypes.byref(n)),
           "dash_profile_end")
    return a.value, b.value, c.value, n.value


def bwd_launches(causal, schedule, deterministic) -> int:
    return int(_lib.dash_attn_bwd_launches(int(causal), _sched(schedule), int(deterministic)))


def set_watchdog(cycles: int):
    """dash_attn_bwd_set_watchdog: bound of one ticket wait in clock64 cycles (0 = default)."""
    _check(_lib.dash_attn_bwd_set_watchdog(int(cycles)), "dash_attn_bwd_set_watchdog")


def inject_fault(poison: int):
    """dash_attn_bwd_inject_fault (verification only): the next backward on this
    thread presets its first ticket to `poison`, a value no ordered add reaches."""
    _check(_lib.dash_attn_bwd_inject_fault(int(poison)), "dash_attn_bwd_inject_fault")


def tile(shape_bnhd, causal: bool = True, schedule="auto") -> int:
    """dash_attn_bwd_tile: schedule tile size the backward runs with (128: the
    single-CTA kernel, 256: the CTA-pair kernel)."""
    B, N, H, d = shape_bnhd
    shp = Shape(B, N, H, d, 0.0)
    return int(_lib.dash_attn_bwd_tile(ctypes.byref(shp), int(causal), _sched(schedule)))


def set_tile(t: int):
    """dash_attn_bwd_set_tile: 0 = automatic, 128 forces the single-CTA kernel."""
    _check(_lib.dash_attn_bwd_set_tile(int(t)), "dash_attn_bwd_set_tile")
