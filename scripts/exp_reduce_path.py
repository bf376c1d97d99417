"""Timing experiment (not a bench line): TFLOP/s of one sweep point per
schedule / det, under whatever DASH_DEBUG the process was started with.
  DASH_DEBUG=0 python scripts/exp_reduce_path.py 2048,16384 128 causal
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_21824_b200 import dash  # noqa: E402
from paper_2601_21824_b200.inputs import attn_inputs, sweep_shape  # noqa: E402

seqlens = [int(x) for x in sys.argv[1].split(",")]
d = int(sys.argv[2])
causal = sys.argv[3] == "causal"
dbg = os.environ.get("DASH_DEBUG", "0")
for N in seqlens:
    B, _, H, _ = sweep_shape(N, d)
    g = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=0).items()}
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
    ws = dash.alloc_workspace(g["q"].shape, causal)
    out = (torch.empty_like(g["q"]), torch.empty_like(g["q"]), torch.empty_like(g["q"]))
    fl = 10.0 * B * H * N * N * d / (2 if causal else 1)
    res = []
    for sched, det in (("naive", True), ("descending", True), ("shift", True), ("naive", False)):
        try:
            f = lambda: dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, causal, sched, det,
                                      workspace=ws, out=out)
            for _ in range(3):
                f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                f()
            e1.record()
            torch.cuda.synchronize()
            res.append(f"{sched}{'' if det else '-atomic'}={fl * 10 / (e0.elapsed_time(e1) / 1e3) / 1e12:.0f}")
        except dash.DashError as e:
            res.append(f"{sched}=ERR")
    print(f"DEBUG={dbg} G={os.environ.get('DASH_HEAD_GROUP', '-')} PF={0 if os.environ.get('DASH_NO_PREFETCH', '0') == '1' else 1} VAR={os.environ.get('DASH_VARIANT', '-')} W={dash.acc_split(N)} N={N} d={d} {'causal' if causal else 'full'}: " + " ".join(res), flush=True)
