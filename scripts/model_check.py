"""BASELINE.json config 5: schedule-model check -- DAG critical path (host
model, dash_schedule_critical_path) vs GPU timing, for n_q = n_kv = n tiles.

For each n (N = 128 n, d = 128, hidden 2048, 16k tokens per sweep point when
n >= 4) and mask, times the deterministic backward under NAIVE, DESCENDING
and SHIFT and reports measured T_sched / T_naive next to the model's
prediction on the same number of SMs, with c (compute) and r (reduction)
phase weights taken from the clock64 trace of one NAIVE run
(c = median sub-tile period x sub-tiles per task, r = median reduce-issue ->
release time).  "Insights, not predictions": the comparison
is reported, not fitted further.

  python scripts/model_check.py [--out profiles/r01_model_check.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402
from paper_2601_21824_b200 import dash  # noqa: E402
from paper_2601_21824_b200.inputs import attn_inputs  # noqa: E402


def time_bwd(g, causal, schedule, reps=5):
    ws = dash.alloc_workspace(g["q"].shape, causal)
    out = tuple(torch.empty_like(g["q"]) for _ in range(3))
    for _ in range(2):
        dash.attn_bwd(g["q"], g["k"], g["v"], g["o"], g["do"], g["lse"], causal, schedule, True,
                      workspace=ws, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        dash.attn_bwd(g["q"], g["k"], g["v"], g["o"], g["do"], g["lse"], causal, schedule, True,
                      workspace=ws, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def fit_c_r(g, causal):
    _, tr = dash.attn_bwd_trace(g["q"], g["k"], g["v"], g["o"], g["do"], g["lse"], causal,
                                "naive", True, trace_cap=512)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.int64)
    periods, reds = [], []
    for cta in range(t.shape[0]):
        nx = int(np.count_nonzero(t[cta, :, 0]))
        if nx < 3:
            continue
        a = t[cta, :nx]
        periods.extend(np.diff(a[:, 0]).tolist())
        reds.extend((a[:, 9] - a[:, 8]).tolist())
    sub_per_task = 2 if g["q"].shape[3] == 128 else 1
    c = int(np.median(periods)) * sub_per_task
    r = max(1, int(np.median(reds)))
    return c, r


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--ns", default="4,8,16,32,64,128")
    ap.add_argument("--acc-split", type=int, default=1,
                    help="W (AMB-27); the DAG model is the paper's single chain, W = 1")
    args = ap.parse_args()
    dash.set_acc_split(args.acc_split)
    dash.set_tile(128)  # the DAG model below is one SM per 128-row KV tile
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    rows = []
    for n in (int(v) for v in args.ns.split(",")):
        N, d = 128 * n, 128
        B, H = max(1, 16384 // N), 2048 // d
        cpu = attn_inputs(B, N, H, d, seed=n)
        g = {k: v.cuda() for k, v in cpu.items()}
        for causal in (True, False):
            g["o"], g["lse"] = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
            c, r = fit_c_r(g, causal)
            mask = dash.CAUSAL if causal else dash.FULL
            m = B * H
            row = {"n": n, "N": N, "B": B, "H": H, "mask": "causal" if causal else "full",
                   "acc_split": dash.acc_split((B, N, H, d), causal),
                   "c_cycles": c, "r_cycles": r, "n_sm": sms, "heads_m": m}
            with ClockSampler(torch.cuda.current_device()) as clk:  # clocks over the row's timings
                clk.mark("t0")
                t_naive = time_bwd(g, causal, "naive")
                cp_naive = dash.schedule_critical_path(dash.NAIVE, n, n, mask, m, sms, c, r)
                for name, sched in (("naive", dash.NAIVE), ("descending", dash.DESCENDING),
                                    ("shift", dash.SHIFT)):
                    try:
                        cp = dash.schedule_critical_path(sched, n, n, mask, m, sms, c, r)
                    except dash.DashError as e:
                        row[name] = {"error": str(e)}
                        continue
                    t = t_naive if name == "naive" else time_bwd(g, causal, name)
                    row[name] = {"gpu_ms": t, "model_cycles": cp,
                                 "gpu_ratio_vs_naive": t / t_naive,
                                 "model_ratio_vs_naive": cp / cp_naive}
                clk.mark("t1")
            row["clocks"] = clk.summary()
            rows.append(row)
            print(json.dumps(row), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
