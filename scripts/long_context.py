"""BASELINE.json config 4: long context -- B = 8, H = 32, N = 32768, d = 128,
causal.  Times dash_attn_bwd under NAIVE / DESCENDING / SHIFT (deterministic)
and the atomic variant (measurement only; the sampled-row parity of this
configuration is a GPU test, tests/test_gpu_bwd.py).

  python scripts/long_context.py [--out profiles/r01_long_context.json] [--batch 8]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_21824_b200 import dash  # noqa: E402
from paper_2601_21824_b200.inputs import attn_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    B, N, H, d = args.batch, 32768, 32, 128
    cpu = attn_inputs(B, N, H, d, seed=7)
    g = {k: v.cuda() for k, v in cpu.items()}
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], True)
    ws = dash.alloc_workspace(g["q"].shape, True)
    out = tuple(torch.empty_like(g["q"]) for _ in range(3))
    flops = 10.0 * B * H * N * N * d / 2
    res = {"config": "long-context", "B": B, "N": N, "H": H, "d": d, "mask": "causal",
           "flops_fa_convention": flops, "acc_split": dash.acc_split((B, N, H, d), True),
           "auto_schedule": dash.resolve_schedule((B, N, H, d), True, "auto")}
    for name, sched, det in (("naive", "naive", True), ("descending", "descending", True),
                             ("shift", "shift", True), ("atomic", "naive", False),
                             ("auto", "auto", True)):
        dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, True, sched, det, workspace=ws,
                      out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, True, sched, det, workspace=ws,
                          out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.reps
        res[name] = {"ms": ms, "tflops": flops / (ms / 1e3) / 1e12}
    # parity of this configuration against the fp64 oracle lives in
    # tests/test_gpu_bwd.py::test_long_context_config4_sampled_rows (sampled rows)
    res["deadlock_check"] = dash.check_workspace(g["q"].shape, True, "shift", True, ws)
    gap = res["atomic"]["tflops"] - res["naive"]["tflops"]
    best = max(res["shift"]["tflops"], res["descending"]["tflops"])
    res["gap_closed"] = (best - res["naive"]["tflops"]) / gap if gap > 0 else None
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
