"""One backward call for debugging: python scripts/one_call.py N d causal schedule det reps"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_21824_b200 import dash
from paper_2601_21824_b200.inputs import attn_inputs, sweep_shape
N, d, causal, sched, det, reps = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3] == "1", sys.argv[4], sys.argv[5] == "1", int(sys.argv[6])
B, NN, H, dd = sweep_shape(N, d)
if len(sys.argv) > 7:
    B, H = int(sys.argv[7]), int(sys.argv[8])
g = {k: v.cuda() for k, v in attn_inputs(B, NN, H, dd, seed=0).items()}
o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
torch.cuda.synchronize()
print("fwd ok", flush=True)
for i in range(reps):
    dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, causal, sched, det)
    torch.cuda.synchronize()
    print("bwd ok", i, flush=True)
