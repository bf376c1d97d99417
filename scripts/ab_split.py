"""A/B helper: per-kernel split (K1 / K2 / K4, CUDA events) of the bench sweep step."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2601_21824_b200 import dash
from paper_2601_21824_b200.inputs import attn_inputs
dash.set_fused_dq(int(os.environ.get("FUSED", "1")))
SEQ = (512, 1024, 2048, 4096, 8192, 16384)
probs = []
for N in SEQ:
    B, H, d = 16384 // N, 16, 128
    g = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=N).items()}
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], True)
    ws = dash.alloc_workspace(g["q"].shape, True)
    probs.append((g, o, lse, ws))
def step():
    for g, o, lse, ws in probs:
        dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, True, "auto", True, workspace=ws)
for _ in range(3): step()
torch.cuda.synchronize()
dash.profile_begin()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(10): step()
e1.record(); torch.cuda.synchronize()
pre, main, post, n = dash.profile_end()
print(sys.argv[1], "total", round(e0.elapsed_time(e1), 2), "pre", round(pre, 2), "main", round(main, 2), "post", round(post, 2), "calls", n)
