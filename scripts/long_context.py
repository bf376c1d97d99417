"""BASELINE.json config 4: long context -- B = 8, H = 32, N = 32768, d = 128,
causal.  Times dash_attn_bwd under NAIVE / DESCENDING / SHIFT (deterministic)
and the atomic variant, and checks sampled dQ rows of two heads against the
fp64 oracle (computed one row at a time).

  python scripts/long_context.py [--out profiles/r01_long_context.json] [--batch 8]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (sampled parity only)
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
           "flops_fa_convention": flops, "acc_split": dash.acc_split(N),
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
        if name == "auto":
            dq = out[0]
            f = {k: v[:1].double().numpy() for k, v in cpu.items()}  # batch 0 only
            heads, rows = [0, 31], [0, 4097, 20000, 32767]
            ref = oracle.attn_bwd_dq_rows(f["q"], f["k"], f["v"], f["do"], True, heads, rows)
            got = np.stack([dq[0, rows, h].float().cpu().numpy() for h in heads])
            res["auto"]["sampled_dq_err_normalised"] = float(
                np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
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
