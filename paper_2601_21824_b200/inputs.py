"""Seeded synthetic inputs shared by the tests, the bench and the oracle legs.

This module holds NO arithmetic of the method: it only draws random numbers.
Recipe (the paper says only
"BF16 precision random inputs"):

* a torch CPU generator seeded with ``seed`` draws q, k, v, dO in that order,
  each i.i.d. N(0, 1) in fp32 with shape [B, N, H, d], then rounds to bf16;
* ``qk_gain`` multiplies q and k before rounding (the "peaky softmax" stress
  set uses 3.0);
* drawing on the CPU makes every GPU count and every process see identical bits.
"""
from __future__ import annotations

import torch


def attn_inputs(B: int, N: int, H: int, d: int, seed: int = 0, qk_gain: float = 1.0):
    """Returns dict of bf16 CPU tensors q, k, v, do, each [B, N, H, d] contiguous."""
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    out = {}
    for name in ("q", "k", "v", "do"):
        x = torch.randn((B, N, H, d), generator=g, dtype=torch.float32)
        if name in ("q", "k") and qk_gain != 1.0:
            x = x * qk_gain
        out[name] = x.to(torch.bfloat16).contiguous()
    return out


# The paper's benchmark sweep: 16,384 total tokens, hidden 2,048,
# head dim 64 / 128, seqlen 512 .. 16,384.
SWEEP_SEQLENS = (512, 1024, 2048, 4096, 8192, 16384)
SWEEP_TOKENS = 16384
SWEEP_HIDDEN = 2048


def sweep_shape(seqlen: int, head_dim: int):
    """(B, N, H, d) of one sweep point."""
    return SWEEP_TOKENS // seqlen, seqlen, SWEEP_HIDDEN // head_dim, head_dim
