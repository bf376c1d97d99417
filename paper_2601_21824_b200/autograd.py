"""PyTorch autograd wrapper of the C ABI: `attention(q, k, v, causal, schedule,
deterministic)` with forward = dash_attn_fwd and backward = dash_attn_bwd.

Marshalling only (every step runs in libdash.so kernels): tensors are
bf16 [B, N, H, d] CUDA tensors (the layout a fused QKV projection produces
with .view(B, N, H, d)); the backward's workspace is cached for the last
few (shape, device, size) keys (an LRU of _WS_CACHE_MAX entries) so a
training loop does not reallocate it every step and variable sequence
lengths do not grow GPU memory without bound.  The
deterministic backward is bitwise reproducible (Algorithm 1, PAPER.md
P:351-397); `deterministic=False` selects the atomic comparison variant.
"""
from __future__ import annotations

import torch

from collections import OrderedDict

from . import dash

_WS_CACHE_MAX = 4
_ws_cache: "OrderedDict[tuple, torch.Tensor]" = OrderedDict()


def _workspace(shape, causal, deterministic, device):
    nbytes = dash.workspace_bytes(shape, causal, dash.NAIVE, deterministic)
    key = (tuple(shape), bool(causal), str(device), nbytes)
    ws = _ws_cache.pop(key, None)
    if ws is None:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=device)
    _ws_cache[key] = ws  # most recently used last
    while len(_ws_cache) > _WS_CACHE_MAX:
        _ws_cache.popitem(last=False)
    return ws


class DashAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, causal: bool, schedule, deterministic: bool):
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
        o, lse = dash.attn_fwd(q, k, v, causal)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.causal, ctx.schedule, ctx.deterministic = causal, schedule, deterministic
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        ws = _workspace(q.shape, ctx.causal, ctx.deterministic, q.device)
        dq, dk, dv = dash.attn_bwd(q, k, v, o, do.contiguous(), lse, ctx.causal, ctx.schedule,
                                   ctx.deterministic, workspace=ws)
        return dq, dk, dv, None, None, None


def attention(q, k, v, causal: bool = True, schedule="auto", deterministic: bool = True):
    """softmax(q k^T / sqrt(d)) v over [B, N, H, d] bf16 tensors, differentiable;
    the backward runs the DASH schedule `schedule` ("auto" = the library's
    per-shape choice; "naive" / "descending" / "shift")."""
    return DashAttention.apply(q, k, v, causal, schedule, deterministic)
