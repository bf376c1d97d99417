"""Verify that (b, h)-sharded multi-GPU backward equals the 1-GPU result bit for bit.

  python -m torch.distributed.run --nnodes=1 --nproc-per-node G --master-addr 127.0.0.1 \
      --master-port 29511 scripts/verify_multi_gpu.py [--seqlen 2048] [--schedule shift]

Every rank draws the full seeded input on the CPU, runs dash_attn_fwd /
dash_attn_bwd on its head shard (no collective on the data path), and the
shards are all-gathered (NCCL over NVLink) to rank 0, which recomputes the
whole problem on its GPU and compares bitwise.  Long context: per-head
SHA-256 digests are compared instead of gathering.
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_21824_b200 import dash  # noqa: E402
from paper_2601_21824_b200 import dist as ddist  # noqa: E402
from paper_2601_21824_b200.inputs import attn_inputs, sweep_shape  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqlen", type=int, default=2048)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--schedule", default="shift")
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--digests", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    causal = not args.full
    B, N, H, d = sweep_shape(args.seqlen, args.head_dim)
    cpu = attn_inputs(B, N, H, d, seed=11)
    part = {k: ddist.shard_bnhd(v, world, rank).cuda() for k, v in cpu.items()}
    o, lse = dash.attn_fwd(part["q"], part["k"], part["v"], causal)
    dq, dk, dv = dash.attn_bwd(part["q"], part["k"], part["v"], o, part["do"], lse, causal,
                               args.schedule, True)
    torch.cuda.synchronize()
    ok = True
    if args.digests:
        mine = [ddist.per_head_digests(t) for t in (dq, dk, dv)]
        allv = [None] * world
        if world > 1:
            dist.all_gather_object(allv, mine)
        else:
            allv = [mine]
        if rank == 0:
            full = {k: v.cuda() for k, v in cpu.items()}
            fo, fl = dash.attn_fwd(full["q"], full["k"], full["v"], causal)
            ref = dash.attn_bwd(full["q"], full["k"], full["v"], fo, full["do"], fl, causal,
                                args.schedule, True)
            for i, t in enumerate(ref):
                got = []
                for b in range(B):
                    for r in range(world):
                        h0, h1 = ddist.head_range(H, world, r)
                        got.extend(allv[r][i][b * (h1 - h0):(b + 1) * (h1 - h0)])
                want = ddist.per_head_digests(t)
                ok &= got == want
    else:
        gathered = [ddist.gather_bnhd(t, H, world) if world > 1 else t for t in (dq, dk, dv)]
        if rank == 0:
            full = {k: v.cuda() for k, v in cpu.items()}
            fo, fl = dash.attn_fwd(full["q"], full["k"], full["v"], causal)
            ref = dash.attn_bwd(full["q"], full["k"], full["v"], fo, full["do"], fl, causal,
                                args.schedule, True)
            ok = all(torch.equal(a, b) for a, b in zip(gathered, ref))
    if rank == 0:
        print(json.dumps({"world": world, "seqlen": N, "schedule": args.schedule,
                          "causal": causal, "bitwise_equal_to_1gpu": bool(ok)}))
    if world > 1:
        dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
