"""BASELINE.json config 4: long context -- B = 8, H = 32, N = 32768, d = 128,
causal.  Times dash_attn_bwd under NAIVE / DESCENDING / SHIFT (deterministic,
all at the library's W) and the atomic variant, with CUDA events on the
launching stream and bench.py's nvidia-smi clock sampler around every timed
region; reports the same-W gap closure of BASELINE north_star and the
workspace the dQ-plane budget leaves (include/dash.h).  Measurement only: the
sampled-row parity of this configuration is a GPU test
(tests/test_gpu_bwd.py::test_long_context_config4_sampled_rows).

  python scripts/long_context.py [--out profiles/r02_long_context.json] [--batch 8]
      [--budget BYTES] [--acc-split W]
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402
from paper_2601_21824_b200 import dash  # noqa: E402
from paper_2601_21824_b200.inputs import attn_inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--budget", type=int, default=0, help="dQ-plane budget in bytes (0 = default)")
    ap.add_argument("--acc-split", type=int, default=0, help="force W (0 = automatic)")
    args = ap.parse_args()
    B, N, H, d = args.batch, 32768, 32, 128
    shape = (B, N, H, d)
    dash.set_plane_budget(args.budget)
    dash.set_acc_split(args.acc_split)
    cpu = attn_inputs(B, N, H, d, seed=7)
    g = {k: v.cuda() for k, v in cpu.items()}
    del cpu
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], True)
    out = tuple(torch.empty_like(g["q"]) for _ in range(3))
    flops = 10.0 * B * H * N * N * d / 2
    res = {"config": "long-context (BASELINE configs[3])", "B": B, "N": N, "H": H, "d": d,
           "mask": "causal", "flops_fa_convention": flops,
           "acc_split": dash.acc_split(shape, True), "tile": dash.tile(shape, True, "auto"),
           "auto_schedule": dash.resolve_schedule(shape, True, "auto"),
           "plane_budget_bytes": args.budget or (4 << 30),
           "timing": "CUDA events on the launching stream, mean of --reps calls after one warm-up"}
    for name, sched, det in (("naive", "naive", True), ("descending", "descending", True),
                             ("shift", "shift", True), ("atomic", "naive", False),
                             ("auto", "auto", True)):
        ws = dash.alloc_workspace(shape, True, sched, det, "cuda")
        row = {"workspace_bytes": ws.numel(), "head_chunk": dash.head_chunk(shape, True, sched, det),
               "acc_split": dash.acc_split(shape, True, sched) if det else 1}
        try:
            dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, True, sched, det, workspace=ws,
                          out=out)
            torch.cuda.synchronize()
            with ClockSampler(torch.cuda.current_device()) as clk:
                time.sleep(0.3)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                clk.mark("t0")
                e0.record()
                for _ in range(args.reps):
                    dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, True, sched, det,
                                  workspace=ws, out=out)
                e1.record()
                torch.cuda.synchronize()
                clk.mark("t1")
            ms = e0.elapsed_time(e1) / args.reps
            row.update({"ms": ms, "tflops": flops / (ms / 1e3) / 1e12, "clocks": clk.summary(),
                        "deadlock_check": dash.check_workspace(shape, True, sched, det, ws)})
        except dash.DashError as e:
            row["error"] = str(e)
        res[name] = row
        del ws
        torch.cuda.empty_cache()
        print(name, json.dumps(row), flush=True)
    t = {k: res[k].get("tflops") for k in ("naive", "descending", "shift", "atomic")}
    if t["naive"] and t["atomic"] and t["atomic"] > t["naive"]:
        best = max([v for k, v in t.items() if k in ("descending", "shift") and v] or [t["naive"]])
        res["gap_closed_same_w"] = (best - t["naive"]) / (t["atomic"] - t["naive"])
        res["gate_pass"] = res["gap_closed_same_w"] >= 0.5
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
