"""oracle -- TEST INFRASTRUCTURE ONLY.

CPU reference for the DASH deterministic attention backward (PAPER.md
Algorithm 1) and its DAG schedule model (§3).

* ``attn_oracle.c`` -- fp64 attention forward/backward, the plain definition.
* ``dag_oracle.py`` -- brute-force schedule/critical-path simulator.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product (``paper_2601_21824_b200``, ``libdash.so``) never imports or links it,
and this package imports nothing from the product.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "attn_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile attn_oracle.c with plain gcc (no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        i, d = ctypes.c_int, ctypes.c_double
        lib.oracle_attn_fwd.argtypes = [i, i, i, i, d, i, dp, dp, dp, dp, dp]
        lib.oracle_attn_bwd.argtypes = [i, i, i, i, d, i, dp, dp, dp, dp, dp, dp, dp, dp, dp, dp]
        lib.oracle_attn_bwd_dq_rows.argtypes = [i, i, i, i, d, i, dp, dp, dp, dp, i, ip, i, ip, dp]
        lib.oracle_attn_bwd_kv_rows.argtypes = [i, i, i, i, d, i, dp, dp, dp, dp, i, ip, i, ip, dp, dp]
        lib.oracle_set_threads.argtypes = [i]
        lib.oracle_max_threads.restype = i
        _lib = lib
    return _lib


def _f64(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i32(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.int32))
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int))


def set_threads(n: int) -> None:
    _load().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _scale(d, scale):
    return (1.0 / np.sqrt(d)) if (scale is None or scale <= 0) else float(scale)


def attn_fwd(q, k, v, causal: bool, scale=None):
    """O [B,N,H,d] and natural-log L [B,H,N] in fp64."""
    lib = _load()
    q, qp = _f64(q)
    k, kp = _f64(k)
    v, vp = _f64(v)
    B, N, H, D = q.shape
    o = np.empty_like(q)
    lse = np.empty((B, H, N), dtype=np.float64)
    _, op = _f64(o)
    _, lp = _f64(lse)
    lib.oracle_attn_fwd(B, N, H, D, _scale(D, scale), int(causal), qp, kp, vp, op, lp)
    return o, lse


def attn_bwd(q, k, v, dout, causal: bool, scale=None):
    """dQ, dK, dV (and the oracle's own O, L, D) in fp64 (Alg. 1)."""
    lib = _load()
    q, qp = _f64(q)
    k, kp = _f64(k)
    v, vp = _f64(v)
    dout, dop = _f64(dout)
    B, N, H, D = q.shape
    dq, dk, dv, o = (np.empty_like(q) for _ in range(4))
    lse = np.empty((B, H, N), dtype=np.float64)
    Dv = np.empty((B, H, N), dtype=np.float64)
    ptr = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    lib.oracle_attn_bwd(B, N, H, D, _scale(D, scale), int(causal), qp, kp, vp, dop,
                        ptr(dq), ptr(dk), ptr(dv), ptr(o), ptr(lse), ptr(Dv))
    return {"dq": dq, "dk": dk, "dv": dv, "o": o, "lse": lse, "D": Dv}


def attn_bwd_dq_rows(q, k, v, dout, causal: bool, heads, rows, scale=None):
    """dQ of the listed query rows of the listed heads (b*H+h): [nheads, nrows, d]."""
    lib = _load()
    q, qp = _f64(q)
    k, kp = _f64(k)
    v, vp = _f64(v)
    dout, dop = _f64(dout)
    B, N, H, D = q.shape
    heads, hp = _i32(heads)
    rows, rp = _i32(rows)
    out = np.empty((len(heads), len(rows), D), dtype=np.float64)
    lib.oracle_attn_bwd_dq_rows(B, N, H, D, _scale(D, scale), int(causal), qp, kp, vp, dop,
                                len(heads), hp, len(rows), rp,
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def attn_bwd_kv_rows(q, k, v, dout, causal: bool, heads, cols, scale=None):
    """dK, dV of the listed key rows of the listed heads: two [nheads, ncols, d]."""
    lib = _load()
    q, qp = _f64(q)
    k, kp = _f64(k)
    v, vp = _f64(v)
    dout, dop = _f64(dout)
    B, N, H, D = q.shape
    heads, hp = _i32(heads)
    cols, cp = _i32(cols)
    dk = np.empty((len(heads), len(cols), D), dtype=np.float64)
    dv = np.empty_like(dk)
    ptr = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    lib.oracle_attn_bwd_kv_rows(B, N, H, D, _scale(D, scale), int(causal), qp, kp, vp, dop,
                                len(heads), hp, len(cols), cp, ptr(dk), ptr(dv))
    return dk, dv
