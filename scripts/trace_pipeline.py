"""Pipeline timeline of the backward main kernel from dash_attn_bwd_trace.

Runs one sweep point, reads the per-(CTA, sub-tile) clock64 stamps and prints
median stage durations in SM cycles (measurement tool; not a bench line).

  python scripts/trace_pipeline.py --seqlen 2048 --schedule shift [--full] [--head-dim 128]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_21824_b200 import dash  # noqa: E402
from paper_2601_21824_b200.inputs import attn_inputs, sweep_shape  # noqa: E402

SLOTS = ["sdp_issue", "p_seen", "dq_issue", "smx_start", "smx_done", "drain_start", "staged",
         "acquired", "reduce_issued", "released", "load_issued", "read_done", "write_done"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqlen", type=int, default=2048)
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--schedule", default="shift")
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--atomic", action="store_true")
    ap.add_argument("--out", default=None)
    ap.add_argument("--npz", default=None, help="also save the raw stamps [grid, sub-tiles, 16]")
    args = ap.parse_args()
    causal = not args.full
    B, N, H, d = sweep_shape(args.seqlen, args.head_dim)
    g = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=0).items()}
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
    for _ in range(3):
        dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, causal, args.schedule, not args.atomic)
    cap = 1024
    _, tr = dash.attn_bwd_trace(g["q"], g["k"], g["v"], o, g["do"], lse, causal, args.schedule,
                                not args.atomic, trace_cap=cap)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.int64)  # [grid, cap, 16]
    if args.npz:
        nmax = int(max(np.count_nonzero(t[c, :, 0]) for c in range(t.shape[0])))
        np.savez_compressed(args.npz, stamps=t[:, :nmax, :32])
    res = {"seqlen": N, "head_dim": d, "schedule": args.schedule, "causal": causal,
           "deterministic": not args.atomic}
    per = {}
    for cta in range(t.shape[0]):
        nx = int(np.count_nonzero(t[cta, :, 0]))
        if nx < 2:
            continue
        a = t[cta, :nx, :16]
        per.setdefault("reduce_read", []).extend((a[:, 11] - a[:, 8]).tolist())
        per.setdefault("reduce_write", []).extend((a[:, 12] - a[:, 11]).tolist())
        per.setdefault("write_to_release", []).extend((a[:, 9] - a[:, 12]).tolist())
        per.setdefault("load_to_sdp_issue", []).extend((a[:, 0] - a[:, 10]).tolist())
        per.setdefault("period", []).extend(np.diff(a[:, 0]).tolist())
        per.setdefault("mma_wait_p", []).extend((a[:, 1] - a[:, 0]).tolist())
        per.setdefault("softmax", []).extend((a[:, 4] - a[:, 3]).tolist())
        if np.count_nonzero(a[:, 15]) > 0:  # pair kernel: softmax sub-steps
            per.setdefault("smx_to_ds_ready", []).extend((a[:, 13] - a[:, 3]).tolist())
            per.setdefault("smx_ds_stores", []).extend((a[:, 14] - a[:, 13]).tolist())
            per.setdefault("smx_fences", []).extend((a[:, 15] - a[:, 14]).tolist())
            per.setdefault("smx_arrive", []).extend((a[:, 4] - a[:, 15]).tolist())
        per.setdefault("s_ready_to_smx", []).extend((a[:, 3] - a[:, 0]).tolist())
        per.setdefault("p_to_dq_issue", []).extend((a[:, 2] - a[:, 1]).tolist())
        per.setdefault("drain", []).extend((a[:, 6] - a[:, 5]).tolist())
        per.setdefault("dq_issue_to_drain", []).extend((a[:, 5] - a[:, 2]).tolist())
        per.setdefault("staged_to_acquired", []).extend((a[:, 7] - a[:, 6]).tolist())
        per.setdefault("acquire_before_staged", []).extend((a[:, 6] - a[:, 7]).tolist())
        per.setdefault("reduce_to_release", []).extend((a[:, 9] - a[:, 8]).tolist())
        per.setdefault("staged_to_release", []).extend((a[:, 9] - a[:, 6]).tolist())
    for k, v in per.items():
        v = np.array(v)
        res[k] = {"p10": float(np.percentile(v, 10)), "p50": float(np.median(v)),
                  "p90": float(np.percentile(v, 90)), "mean": float(v.mean())}
    # raw stamps of CTA 0's first sub-tiles, relative to its first S/dP issue
    a0 = t[0, :24, :13]  # noqa
    base = a0[0, 0]
    res["raw_cta0"] = {SLOTS[i]: [int(v - base) if v else None for v in a0[:, i]] for i in range(13)}
    print(json.dumps({k: v for k, v in res.items() if k != "raw_cta0"}, indent=1))
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
