"""Per-kernel CUDA-event split (K1 preprocess / K2 main / K4 convert) of the bench sweep step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_21824_b200 import dash
from paper_2601_21824_b200.inputs import attn_inputs
probs = []
for N in (512, 1024, 2048, 4096, 8192, 16384):
    B, H, d = 16384 // N, 16, 128
    g = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=N).items()}
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], True)
    probs.append((g, o, lse, dash.alloc_workspace(g["q"].shape, True)))
def step():
    for g, o, lse, ws in probs:
        dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, True, "auto", True, workspace=ws)
for _ in range(3): step()
torch.cuda.synchronize()
dash.profile_begin()
for _ in range(10): step()
torch.cuda.synchronize()
pre, main, post, n = dash.profile_end()
bytes_pre = 6 * (2 * 16384 * 2048 * 2 + 16384 * 16 * 12) * 10
print(f"per step: K1 {pre/10*1e3:.1f} us ({bytes_pre/(pre/1e3)/1e9:.0f} GB/s), K2 {main/10:.3f} ms, K4 {post/10*1e3:.1f} us, calls {n}")
