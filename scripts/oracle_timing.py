"""CPU fp64 oracle timing beside the GPU (SURVEY.md §8(d) "CPU oracle timing"):
config 1 single-thread and all-core, one sweep shape per mask (N = 512 and 2048,
d = 128; a bounded number of heads, scaled to the shape's FLOPs), and the long
context config (one (b, h) head of N = 32k timed, x256 extrapolated, labelled).
A reported baseline, not the optimisation target.

  python scripts/oracle_timing.py --out profiles/r01_oracle_timing.json
"""
import argparse
import json
import os
import platform
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure; measurement only)
from paper_2601_21824_b200.inputs import attn_inputs  # noqa: E402


def fa_flops(B, N, H, d, causal):
    f = 10.0 * B * H * N * N * d
    return f / 2 if causal else f


def run(B, N, H, d, causal, threads):
    oracle.set_threads(threads)
    x = attn_inputs(B, N, H, d, seed=0)
    f = {k: v.double().numpy() for k, v in x.items()}
    t = time.time()
    oracle.attn_bwd(f["q"], f["k"], f["v"], f["do"], causal)
    dt = time.time() - t
    return dt, fa_flops(B, N, H, d, causal) / dt / 1e12


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    oracle.build()
    cores = len(os.sched_getaffinity(0))
    cpu = platform.processor() or platform.machine()
    try:
        with open("/proc/cpuinfo") as fh:
            cpu = next(l.split(":", 1)[1].strip() for l in fh if l.startswith("model name"))
    except (OSError, StopIteration):
        pass
    res = {"cpu_model": cpu, "cores": cores, "rows": []}
    for causal in (True, False):
        for threads in (1, cores):
            dt, tf = run(1, 256, 1, 64, causal, threads)
            res["rows"].append({"config": "1 (B=1,H=1,N=256,d=64)", "causal": causal,
                                "threads": threads, "seconds": dt, "tflops": tf})
    for N, heads in ((512, 4 * cores), (2048, cores)):
        for causal in (True, False):
            dt, tf = run(1, N, heads, 128, causal, cores)
            B, H = 16384 // N, 16
            res["rows"].append({"config": f"sweep N={N} d=128 ({heads} of {B * H} heads)",
                                "causal": causal, "threads": cores, "seconds": dt, "tflops": tf,
                                "extrapolated_full_shape_seconds": dt * B * H / heads})
    # one head runs on one thread (the oracle parallelises over heads): time
    # N = 4096 and extrapolate by (32768 / 4096)^2 and 256 heads / cores
    dt, tf = run(1, 4096, 1, 128, True, cores)
    res["rows"].append({"config": "4 long context (B=8,H=32,N=32768,d=128 causal), from one head of N=4096",
                        "causal": True, "threads": 1, "seconds": dt, "tflops": tf,
                        "extrapolated_full_config_seconds": dt * 64 * 256 / cores,
                        "note": "extrapolated: x64 (N^2) x 256 heads / cores threads; not measured"})
    for r in res["rows"]:
        print(json.dumps(r), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
