"""One fused-finalise backward per kernel for compute-sanitizer (memcheck /
synccheck): d = 64 with a ragged last finalise task (N = 384), the single-CTA
d = 128 kernel, and the CTA-pair kernel, each with the finalise forced into the
main kernel (dash_attn_bwd_set_fused_dq(2)); atomic variant too.
  compute-sanitizer --tool memcheck python scripts/sanitize_fused.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_21824_b200 import dash  # noqa: E402
from paper_2601_21824_b200.inputs import attn_inputs  # noqa: E402

dash.set_fused_dq(2)
for (B, N, H, d, tile, causal, sched, det) in [
        (1, 384, 2, 64, 0, True, "shift", True),
        (2, 512, 2, 128, 128, False, "descending", True),
        (1, 1024, 2, 128, 256, True, "shift", True),
        (1, 512, 3, 64, 0, True, "naive", False)]:
    dash.set_tile(tile)
    g = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=1).items()}
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
    dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, causal, sched, det)
    torch.cuda.synchronize()
    print("ok", B, N, H, d, tile, causal, sched, det, flush=True)
dash.set_tile(0)
dash.set_fused_dq(1)
