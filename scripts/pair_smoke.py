"""Quick GPU check of the CTA-pair kernel against the fp64 oracle (development aid)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2601_21824_b200 import dash  # noqa: E402
from paper_2601_21824_b200.inputs import attn_inputs  # noqa: E402

for (B, N, H) in ((1, 256, 1), (1, 512, 2), (2, 1024, 3)):
    d = 128
    cpu = attn_inputs(B, N, H, d, seed=0)
    g = {k: v.cuda() for k, v in cpu.items()}
    f = {k: v.double().numpy() for k, v in cpu.items()}
    for causal in (False, True):
        ref = oracle.attn_bwd(f["q"], f["k"], f["v"], f["do"], causal)
        o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
        for sched, det in (("naive", True), ("descending", True), ("shift", True), ("naive", False)):
            t0 = time.time()
            try:
                out = dash.attn_bwd(g["q"], g["k"], g["v"], o, g["do"], lse, causal, sched, det)
                torch.cuda.synchronize()
                st = dash.check_workspace(g["q"].shape, causal, sched, det,
                                          dash.alloc_workspace(g["q"].shape, causal, sched, det))
            except Exception as e:  # noqa: BLE001
                print("ERR", B, N, H, causal, sched, det, e, flush=True)
                continue
            errs = []
            for name, x in zip(("dq", "dk", "dv"), out):
                r = ref[name]
                errs.append(float(np.max(np.abs(x.float().cpu().numpy() - r)) / np.max(np.abs(r))))
            print(f"tile={dash.tile(g['q'].shape)} B={B} N={N} H={H} causal={causal} {sched} det={det} "
                  f"errs={['%.2e' % e for e in errs]} {time.time() - t0:.2f}s", flush=True)
