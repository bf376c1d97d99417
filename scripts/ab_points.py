"""A/B helper: main-kernel time per call (CUDA events, dash_profile) at every
sweep point of the hd128 (or --d 64) sweep, for the given schedules and masks.
Experiment switches come from the environment of the process.

  python scripts/ab_points.py TAG [--d 128] [--scheds auto,shift] [--full]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_21824_b200 import dash  # noqa: E402
from paper_2601_21824_b200.inputs import attn_inputs, sweep_shape  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("tag")
ap.add_argument("--d", type=int, default=128)
ap.add_argument("--scheds", default="auto")
ap.add_argument("--masks", default="causal")
ap.add_argument("--seqlens", default="512,1024,2048,4096,8192,16384")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tiles", default="0", help="dash_attn_bwd_set_tile values to compare (0 = library choice)")
ap.add_argument("--rounds", type=int, default=1, help="interleaved rounds (median reported)")
ap.add_argument("--splits", default="0", help="dash_attn_bwd_set_acc_split values to compare (0 = automatic)")
ap.add_argument("--total", action="store_true", help="report K1 + K2 + K4 instead of the main kernel")
ap.add_argument("--fused", default="1", help="dash_attn_bwd_set_fused_dq modes to compare (0 = K4, 1 = library choice, 2 = in-kernel)")
args = ap.parse_args()
res = {"tag": args.tag}
for mask in args.masks.split(","):
    causal = mask == "causal"
    for N in (int(s) for s in args.seqlens.split(",")):
        B, N, H, d = sweep_shape(N, args.d)
        g = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=N).items()}
        o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
        times = {}
        for _ in range(args.rounds):
            for tile, wsplit, fz in ((int(t), int(w), int(f)) for t in args.tiles.split(",")
                                     for w in args.splits.split(",") for f in args.fused.split(",")):
                dash.set_fused_dq(fz)
                dash.set_tile(tile)
                dash.set_acc_split(wsplit)
                for sched in args.scheds.split(","):
                    ws = dash.alloc_workspace(g["q"].shape, causal, sched, True, "cuda")
                    for _ in range(3):
                        dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, causal, sched, True,
                                      workspace=ws)
                    torch.cuda.synchronize()
                    dash.profile_begin()
                    for _ in range(args.reps):
                        dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, causal, sched, True,
                                      workspace=ws)
                    pre, main, post, n = dash.profile_end()
                    key = (f"{mask}/{sched}/{N}" + (f"/t{tile}" if tile else "") +
                           (f"/W{wsplit}" if wsplit else "") + ("" if fz == 1 else f"/fz{fz}"))
                    tot = (pre + main + post) if args.total else main
                    times.setdefault(key, []).append(1000 * tot / n)  # us per call
                    del ws
        dash.set_tile(0)
        dash.set_acc_split(0)
        dash.set_fused_dq(1)
        for key, v in times.items():
            res[key] = round(sorted(v)[len(v) // 2], 1)
print(json.dumps(res))
