"""Bitwise run-to-run determinism over the BASELINE sweep shapes (measurement /
evidence tool): for d in {128, 64}, both masks, every sweep point N = 512 ..
16384 and every schedule (+ auto), `reps` back-to-back dash_attn_bwd calls
(fused dQ finalise as the library chooses it) are compared element for element
(torch.equal on the device) with the first call.  Prints one JSON line.

  python scripts/determinism_sweep.py [reps=20] > profiles/r02_determinism_sweep.json
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2601_21824_b200 import dash  # noqa: E402
from paper_2601_21824_b200.inputs import attn_inputs, sweep_shape  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
res = {"reps": reps, "fused_dq_mode": dash.fused_dq(), "configs": 0, "calls": 0, "mismatches": []}
t0 = time.time()
for d in (128, 64):
    for N in (512, 1024, 2048, 4096, 8192, 16384):
        B, NN, H, dd = sweep_shape(N, d)
        g = {k: v.cuda() for k, v in attn_inputs(B, NN, H, dd, seed=N).items()}
        for causal in (True, False):
            o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
            for sched in ("naive", "descending", "shift", "auto"):
                ws = dash.alloc_workspace(g["q"].shape, causal, sched, True, "cuda")
                ref = [x.clone() for x in dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse,
                                                        causal, sched, True, workspace=ws)]
                bad = 0
                for _ in range(reps - 1):
                    out = dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, causal, sched, True,
                                        workspace=ws)
                    bad += sum(0 if torch.equal(a, b) else 1 for a, b in zip(ref, out))
                res["configs"] += 1
                res["calls"] += reps
                if bad:
                    res["mismatches"].append({"d": d, "N": N, "causal": causal, "schedule": sched,
                                              "tensors_differing": bad})
                del ws
res["seconds"] = round(time.time() - t0, 1)
res["all_identical"] = not res["mismatches"]
print(json.dumps(res))
