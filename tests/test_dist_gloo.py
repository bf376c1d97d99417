"""Multi-process (world_size 2, gloo, CPU) tests of the (b, h) sharding host
logic used by bench.py and scripts/verify_multi_gpu.py.

The per-rank compute is the fp64 oracle (a stand-in for the GPU call: the
point here is the split / gather / digest plumbing), so the sharded result
must equal the unsharded one bit for bit -- the property the GPU path keeps
because each head's schedule is independent of the shard.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_21824_b200 import dist as ddist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_head_range_covers_heads_exactly_once():
    for H in range(1, 40):
        for world in range(1, 9):
            seen = []
            for r in range(world):
                h0, h1 = ddist.head_range(H, world, r)
                assert 0 <= h0 <= h1 <= H
                seen.extend(range(h0, h1))
            assert seen == list(range(H))
            sizes = [ddist.head_range(H, world, r)[1] - ddist.head_range(H, world, r)[0]
                     for r in range(world)]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        ddist.head_range(4, 2, 2)


def _worker(rank, world, port, H, result_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2601_21824_b200.inputs import attn_inputs
    B, N, d = 2, 24, 8
    cpu = attn_inputs(B, N, H, d, seed=5)
    part = {k: ddist.shard_bnhd(v, world, rank) for k, v in cpu.items()}
    f = {k: v.double().numpy() for k, v in part.items()}
    g = oracle.attn_bwd(f["q"], f["k"], f["v"], f["do"], True)
    local = torch.from_numpy(np.ascontiguousarray(g["dq"]))
    full = ddist.gather_bnhd(local, H, world)
    digs = [None] * world
    dist.all_gather_object(digs, ddist.per_head_digests(local))
    if rank == 0:
        ff = {k: v.double().numpy() for k, v in cpu.items()}
        ref = torch.from_numpy(oracle.attn_bwd(ff["q"], ff["k"], ff["v"], ff["do"], True)["dq"])
        order = []
        for b in range(B):
            for r in range(world):
                h0, h1 = ddist.head_range(H, world, r)
                order.extend(digs[r][b * (h1 - h0):(b + 1) * (h1 - h0)])
        ok = torch.equal(full, ref) and order == ddist.per_head_digests(ref)
        with open(os.path.join(result_dir, "ok"), "w") as fh:
            fh.write("1" if ok else "0")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H", [4, 3])
def test_sharded_backward_gathers_bitwise_equal(tmp_path, H):
    mp.spawn(_worker, args=(2, _free_port(), H, str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok").read_text() == "1"


def test_shard_lse_and_bnhd_consistent():
    t = torch.arange(2 * 5 * 6 * 3, dtype=torch.float32).view(2, 5, 6, 3)
    lse = torch.arange(2 * 6 * 5, dtype=torch.float32).view(2, 6, 5)
    parts = [ddist.shard_bnhd(t, 4, r) for r in range(4)]
    assert torch.equal(torch.cat(parts, dim=2), t)
    lparts = [ddist.shard_bhn(lse, 4, r) for r in range(4)]
    assert torch.equal(torch.cat(lparts, dim=1), lse)
    assert all(p.is_contiguous() for p in parts + lparts)
