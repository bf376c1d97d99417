"""PyTorch autograd wrapper of the C ABI: `attention(q, k, v, causal, schedule,
deterministic)` with forward = dash_attn_fwd and backward = dash_attn_bwd.

Marshalling only (every step runs in libdash.so kernels): tensors are
bf16 [B, N, H, d] CUDA tensors (the layout a fused QKV projection produces
with .view(B, N, H, d)); the backward's workspace is cached per (shape,
device) so a training loop does not reallocate it every step.  The
deterministic backward is bitwise reproducible (Algorithm 1, PAPER.md
P:351-397); `deterministic=False` selects the atomic comparison variant.
"""
from __future__ import annotations

import torch

from . import dash

_ws_cache: dict = {}


def _workspace(shape, causal, device):
    key = (tuple(shape), bool(causal), str(device))
    ws = _ws_cache.get(key)
    if ws is None:
        ws = dash.alloc_workspace(shape, causal, dash.NAIVE, True, device)
        _ws_cache[key] = ws
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
        ws = _workspace(q.shape, ctx.causal, q.device)
        dq, dk, dv = dash.attn_bwd(q, k, v, o, do.contiguous(), lse, ctx.causal, ctx.schedule,
                                   ctx.deterministic, workspace=ws)
        return dq, dk, dv, None, None, None


def attention(q, k, v, causal: bool = True, schedule="auto", deterministic: bool = True):
    """softmax(q k^T / sqrt(d)) v over [B, N, H, d] bf16 tensors, differentiable;
    the backward runs the DASH schedule `schedule` ("auto" = the library's
    per-shape choice; "naive" / "descending" / "shift")."""
    return DashAttention.apply(q, k, v, causal, schedule, deterministic)
