"""Stress the backward kernel: many calls per configuration, synchronising after
each, to localise intermittent protocol failures (debug tool)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_21824_b200 import dash
from paper_2601_21824_b200.inputs import attn_inputs, sweep_shape

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cfgs = []
for N in (2048, 512, 16384):
    for causal in (True, False):
        for sched, det in (("naive", False), ("naive", True), ("shift", True), ("descending", True)):
            cfgs.append((N, causal, sched, det))
for d in (128, 64):
    for N, causal, sched, det in cfgs:
        B, NN, H, dd = sweep_shape(N, d)
        g = {k: v.cuda() for k, v in attn_inputs(B, NN, H, dd, seed=0).items()}
        o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
        ws = dash.alloc_workspace(g["q"].shape, causal)
        t = time.time()
        for i in range(reps):
            dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, causal, sched, det, workspace=ws)
            torch.cuda.synchronize()
        print(f"ok d={d} N={N} causal={causal} {sched} det={det} {reps} reps {time.time()-t:.2f}s", flush=True)
