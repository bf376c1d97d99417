# tcgen05 forward: parity tests + timing vs the SIMT kernel
set -x
timeout 900 python -m pytest tests/test_gpu_bwd.py -m gpu -x -q -k "forward or smoke or 100_runs" 2>&1 | tail -3
timeout 300 python __graft_entry__.py smoke 2>&1 | tail -1
timeout 300 python - <<'PY'
import torch, time, sys
sys.path.insert(0, '.')
from paper_2601_21824_b200 import dash
from paper_2601_21824_b200.inputs import attn_inputs, sweep_shape
for d in (128, 64):
  for N in (512, 2048, 16384):
    B, _, H, _ = sweep_shape(N, d)
    g = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=0).items()}
    for causal in (True, False):
        for _ in range(2): dash.attn_fwd(g["q"], g["k"], g["v"], causal)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): dash.attn_fwd(g["q"], g["k"], g["v"], causal)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        fl = 4.0 * B * H * N * N * d / (2 if causal else 1)
        print(f"fwd d={d} N={N} causal={causal}: {ms:.3f} ms  {fl/ms/1e9:.1f} TFLOP/s (FA convention)", flush=True)
PY
