"""Synthetic transformer-block training step (the
paper's Fig. 10 analogue, §4.4), measurement script.

A LLaMA3-8B-shaped block with random bf16 weights -- RMSNorm, fused QKV
projection (hidden 4096 = 32 heads x 128; multi-head, the kernels have no
GQA), attention through paper_2601_21824_b200.autograd.attention (dash_attn_fwd
+ dash_attn_bwd), output projection, RMSNorm, SwiGLU MLP (14336) -- forward
and backward of a scalar loss at batch 1, causal, seqlen 8k / 16k / 32k.
Projections and the MLP are plain torch (cuBLAS) ops: the harness around the
library, not the product.  Reports the step time per attention backward
schedule (NAIVE, DESCENDING, SHIFT, auto; atomic variant for reference), the
attention share, and the block speedup of auto over NAIVE.

  python scripts/block_e2e.py [--seqlens 8192,16384,32768] [--out file.json]
"""
import argparse
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import ClockSampler  # noqa: E402
from paper_2601_21824_b200.autograd import attention  # noqa: E402

HIDDEN, HEADS, D, FFN = 4096, 32, 128, 14336


def rmsnorm(x, w, eps=1e-5):
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)).to(x.dtype) * w


class Block(torch.nn.Module):
    def __init__(self, device):
        super().__init__()
        g = torch.Generator(device="cpu").manual_seed(0)

        def w(*shape, scale):
            return torch.nn.Parameter((torch.randn(*shape, generator=g) * scale).to(torch.bfloat16).to(device))
        self.n1 = torch.nn.Parameter(torch.ones(HIDDEN, dtype=torch.bfloat16, device=device))
        self.n2 = torch.nn.Parameter(torch.ones(HIDDEN, dtype=torch.bfloat16, device=device))
        self.wqkv = w(HIDDEN, 3 * HIDDEN, scale=HIDDEN ** -0.5)
        self.wo = w(HIDDEN, HIDDEN, scale=HIDDEN ** -0.5)
        self.w1 = w(HIDDEN, 2 * FFN, scale=HIDDEN ** -0.5)
        self.w2 = w(FFN, HIDDEN, scale=FFN ** -0.5)

    def forward(self, x, schedule, deterministic):
        B, N, _ = x.shape
        qkv = rmsnorm(x, self.n1) @ self.wqkv
        q, k, v = (t.reshape(B, N, HEADS, D) for t in qkv.split(HIDDEN, dim=-1))
        a = attention(q, k, v, True, schedule, deterministic).reshape(B, N, HIDDEN)
        x = x + a @ self.wo
        h = rmsnorm(x, self.n2) @ self.w1
        gate, up = h.split(FFN, dim=-1)
        return x + (torch.nn.functional.silu(gate) * up) @ self.w2


def time_step(fn, warmup=2, iters=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seqlens", default="8192,16384,32768")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda")
    blk = Block(dev)
    res = []
    for N in (int(s) for s in args.seqlens.split(",")):
        g = torch.Generator(device="cpu").manual_seed(N)
        x = torch.randn(1, N, HIDDEN, generator=g).to(torch.bfloat16).to(dev).requires_grad_(True)
        gy = torch.randn(1, N, HIDDEN, generator=g).to(torch.bfloat16).to(dev)
        row = {"seqlen": N, "batch": 1, "hidden": HIDDEN, "heads": HEADS, "head_dim": D,
               "ffn": FFN, "mask": "causal"}
        cases = (("naive", "naive", True), ("descending", "descending", True),
                 ("shift", "shift", True), ("auto", "auto", True), ("atomic", "naive", False))
        times = {c[0]: [] for c in cases}
        clk = ClockSampler(torch.cuda.current_device()).__enter__()  # clocks over the row's timings
        time.sleep(0.3)
        clk.mark("t0")
        for _ in range(3):  # round-robin over the cases, median per case
            for name, sched, det in cases:
                def step():
                    blk.zero_grad(set_to_none=True)
                    x.grad = None
                    y = blk(x, sched, det)
                    y.backward(gy)
                times[name].append(time_step(step))
        for name, _, _ in cases:
            row[name + "_ms"] = sorted(times[name])[1]
        # attention alone (fwd + bwd of the auto schedule) for the share
        q = torch.randn(1, N, HEADS, D, generator=g).to(torch.bfloat16).to(dev).requires_grad_(True)
        k = torch.randn(1, N, HEADS, D, generator=g).to(torch.bfloat16).to(dev).requires_grad_(True)
        v = torch.randn(1, N, HEADS, D, generator=g).to(torch.bfloat16).to(dev).requires_grad_(True)
        do = torch.randn(1, N, HEADS, D, generator=g).to(torch.bfloat16).to(dev)

        def attn_step():
            q.grad = k.grad = v.grad = None
            attention(q, k, v, True, "auto", True).backward(do)
        row["attention_auto_ms"] = time_step(attn_step)
        clk.mark("t1")
        clk.__exit__(None, None, None)
        row["clocks"] = clk.summary()
        row["attention_share"] = row["attention_auto_ms"] / row["auto_ms"]
        row["speedup_auto_vs_naive"] = row["naive_ms"] / row["auto_ms"]
        row["speedup_atomic_vs_naive"] = row["naive_ms"] / row["atomic_ms"]
        print(json.dumps(row), flush=True)
        res.append(row)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
