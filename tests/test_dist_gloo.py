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


# --- bench.py's distributed code path (strong scaling over (b, h) units) -----

def _bench_worker(rank, world, port, result_dir):
    import sys
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), WORLD_SIZE=str(world),
                      RANK=str(rank), LOCAL_RANK=str(rank))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    import oracle
    from paper_2601_21824_b200.inputs import attn_inputs

    class A:
        gpus = world
    w, r, _ = bench.dist_setup(A)          # gloo on a CPU-only host
    assert (w, r) == (world, rank)
    bench.relaunch_if_needed(A)            # WORLD_SIZE == --gpus: no re-exec, no error
    shapes = [(4, 16, 2, 8), (1, 24, 4, 8)]  # whole-batch units / head-range units
    shards = [bench.shard_inputs(attn_inputs(*s, seed=s[1]), world, rank, "strong") for s in shapes]

    def oracle_bwd(x):
        f = {k: v.double().numpy() for k, v in x.items()}
        g = oracle.attn_bwd(f["q"], f["k"], f["v"], f["do"], True)
        return tuple(torch.from_numpy(np.ascontiguousarray(g[n])) for n in ("dq", "dk", "dv"))

    ok = bench.verify_sharding(world, rank, shapes, lambda i: oracle_bwd(shards[i]),
                               lambda s: oracle_bwd(attn_inputs(*s, seed=s[1])))
    # a corrupted shard must be caught
    bad = bench.verify_sharding(world, rank, shapes[:1],
                                lambda i: tuple(t + (rank == 1) for t in oracle_bwd(shards[i])),
                                lambda s: oracle_bwd(attn_inputs(*s, seed=s[1])))
    mx = bench.max_over_ranks(float(rank + 1), world)
    units = sum(v["q"].shape[0] * v["q"].shape[2] for v in shards)
    tot = torch.tensor([units])
    dist.all_reduce(tot)
    if rank == 0:
        good = ok is True and bad is False and mx == float(world) and \
            int(tot) == sum(s[0] * s[2] for s in shapes)
        with open(os.path.join(result_dir, "ok"), "w") as fh:
            fh.write("1" if good else "0")
    dist.barrier()
    dist.destroy_process_group()


def test_bench_strong_scaling_path_gloo(tmp_path):
    """bench.py's N > 1 plumbing on two gloo ranks: dist_setup, the WORLD_SIZE
    check, the (b, h)-unit split of the shared problem (shard_inputs),
    max_over_ranks and the sharding digest check (verify_sharding, with the
    oracle standing in for the GPU call); a corrupted shard is detected."""
    mp.spawn(_bench_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    assert (tmp_path / "ok").read_text() == "1"


def test_unit_shards_cover_the_problem():
    for B, H, world in ((32, 16, 8), (1, 16, 8), (2, 16, 4), (4, 32, 8), (8, 32, 2), (3, 4, 3)):
        t = torch.arange(B * 3 * H * 2, dtype=torch.float32).view(B, 3, H, 2)
        parts = [ddist.shard_units(t, world, r) for r in range(world)]
        flat = torch.cat([p.permute(0, 2, 1, 3).reshape(-1, 3, 2) for p in parts])
        assert torch.equal(flat, t.permute(0, 2, 1, 3).reshape(-1, 3, 2))
        lse = torch.arange(B * H * 3, dtype=torch.float32).view(B, H, 3)
        lparts = [ddist.shard_units(lse, world, r, "bhn") for r in range(world)]
        assert torch.equal(torch.cat([p.reshape(-1, 3) for p in lparts]), lse.reshape(-1, 3))
    with pytest.raises(ValueError):
        ddist.shard_units(torch.zeros(3, 2, 3, 1), 2, 0)   # 9 units over 2 ranks: 5 = 3 + 2
