"""Measurement: the bench's sweep step (causal HD128, auto) eager vs replayed from one CUDA graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2601_21824_b200 import dash
from paper_2601_21824_b200.inputs import attn_inputs
SEQ = (512, 1024, 2048, 4096, 8192, 16384)
probs = []
flops = 0.0
for N in SEQ:
    B, H, d = 16384 // N, 16, 128
    g = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=N).items()}
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], True)
    ws = dash.alloc_workspace(g["q"].shape, True)
    out = tuple(torch.empty_like(g["q"]) for _ in range(3))
    probs.append((g, o, lse, ws, out))
    flops += 10.0 * B * H * N * N * d / 2
def step():
    for g, o, lse, ws, out in probs:
        dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, True, "auto", True, workspace=ws, out=out)
def timeit(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
step(); torch.cuda.synchronize()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
graph = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    with torch.cuda.graph(graph, stream=s):
        step()
for r in range(3):
    te = timeit(step); tg = timeit(graph.replay)
    print(f"eager {te:.3f} ms {flops/te/1e9:.1f} TF/s | graph {tg:.3f} ms {flops/tg/1e9:.1f} TF/s", flush=True)
