"""Multi-GPU plumbing for the DASH backward: (b, h) head sharding (SURVEY.md
§8(e)).

The backward of different (b, h) heads is independent, so G ranks each run
dash_attn_bwd on a contiguous slice of heads with no collective on the data
path; a head's Q visiting order and dQ reduction ranks depend only on
(n, mask, schedule, tile config), so the sharded outputs are bitwise equal to
the single-GPU ones.  torch.distributed (NCCL on GPUs, gloo on CPU) is used
only to gather results or digests for verification.
"""
from __future__ import annotations

import hashlib

import torch


def head_range(H: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split of H heads over `world` ranks: [h0, h1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(H, world)
    h0 = rank * base + min(rank, extra)
    return h0, h0 + base + (1 if rank < extra else 0)


def shard_bnhd(t: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """Rank's slice of a [B, N, H, d] tensor along heads (contiguous copy)."""
    h0, h1 = head_range(t.shape[2], world, rank)
    return t[:, :, h0:h1].contiguous()


def shard_bhn(t: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """Rank's slice of a [B, H, N] tensor (lse) along heads."""
    h0, h1 = head_range(t.shape[1], world, rank)
    return t[:, h0:h1].contiguous()


def gather_bnhd(local: torch.Tensor, H: int, world: int, group=None) -> torch.Tensor:
    """All-gather head shards of a [B, N, h_r, d] tensor back to [B, N, H, d]."""
    import torch.distributed as dist
    B, N, _, d = local.shape
    sizes = [head_range(H, world, r) for r in range(world)]
    hmax = max(h1 - h0 for h0, h1 in sizes)
    padded = torch.zeros((B, N, hmax, d), dtype=local.dtype, device=local.device)
    padded[:, :, : local.shape[2]] = local
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded, group=group)
    return torch.cat([bufs[r][:, :, : h1 - h0] for r, (h0, h1) in enumerate(sizes)], dim=2)


def digest(t: torch.Tensor) -> str:
    """SHA-256 of a tensor's bytes (long-context verification without gathering)."""
    return hashlib.sha256(t.detach().contiguous().cpu().view(torch.uint8).numpy().tobytes()).hexdigest()


def per_head_digests(t: torch.Tensor) -> list[str]:
    """SHA-256 per head of a [B, N, H, d] tensor, ordered by (b, h)."""
    B, _, H, _ = t.shape
    return [digest(t[b, :, h]) for b in range(B) for h in range(H)]


# --- flattened (b, h) units: the strong-scaling split of SURVEY.md §8(e) -----

def unit_range(U: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced split of U = B*H flattened units u = b*H + h."""
    return head_range(U, world, rank)


def unit_slices(B: int, H: int, world: int, rank: int) -> list[tuple[int, int, int]]:
    """The rank's units as (b, h0, h1) runs -- one run per batch it touches."""
    u0, u1 = unit_range(B * H, world, rank)
    runs = []
    u = u0
    while u < u1:
        b, h0 = divmod(u, H)
        h1 = min(H, h0 + (u1 - u))
        runs.append((b, h0, h1))
        u += h1 - h0
    return runs


def shard_units(t: torch.Tensor, world: int, rank: int, layout: str = "bnhd") -> torch.Tensor:
    """Rank's units of a [B, N, H, d] ("bnhd") or [B, H, N] ("bhn") tensor as
    one contiguous [B_r, N, H_r, d] / [B_r, H_r, N] tensor.  The units must
    form whole batches or one head range of a single batch (always true when
    world divides B*H and both are powers of two, as in every BASELINE
    config); otherwise ValueError."""
    if layout == "bnhd":
        B, _, H, _ = t.shape
    elif layout == "bhn":
        B, H, _ = t.shape
    else:
        raise ValueError(layout)
    runs = unit_slices(B, H, world, rank)
    if not runs:
        raise ValueError("empty shard")
    if all(h0 == 0 and h1 == H for _, h0, h1 in runs):
        b0, b1 = runs[0][0], runs[-1][0] + 1
        return t[b0:b1].contiguous()
    if len(runs) == 1:
        b, h0, h1 = runs[0]
        return (t[b:b + 1, :, h0:h1] if layout == "bnhd" else t[b:b + 1, h0:h1]).contiguous()
    raise ValueError("units do not form a rectangular [B_r, H_r] block")


def per_unit_digests(t: torch.Tensor) -> list[str]:
    """SHA-256 per (b, h) unit of a [B, N, H, d] tensor, in flattened order."""
    return per_head_digests(t)
