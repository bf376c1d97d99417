"""Microbenchmark: TMEM -> register (tcgen05.ld.32x32b.x32) and register ->
TMEM (tcgen05.st.32x32b.x16) throughput per SM, by warps and loads in flight.
Decides whether reading S^T / dP^T / dQ out of TMEM bounds the backward."""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2601_21824_b200", "libdash_probe.so"))
lib.dash_probe_tmem_rate.argtypes = [ctypes.c_int] * 5 + [ctypes.c_void_p]
for grid in (1, 148):
    for mode, infl in ((0, 1), (0, 2), (0, 4), (1, 1), (1, 4)):
        for nw in (4, 8, 12, 16):
            out = torch.zeros(max(grid, 1), dtype=torch.int64, device="cuda")
            rc = lib.dash_probe_tmem_rate(mode, infl, nw, 2000, grid, ctypes.c_void_p(out.data_ptr()))
            cyc = out.float().mean().item()
            per = 4096 if mode == 0 else 2048
            bpc = nw * infl * per / cyc if cyc > 0 else float("nan")
            print(f"grid={grid:3d} {'ld.x32' if mode == 0 else 'st.x16'} inflight={infl} warps={nw:2d} "
                  f"rc={rc} cycles/round={cyc:7.1f}  SM bytes/clk={bpc:7.1f}", flush=True)

lib.dash_probe_exp_rate.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p, ctypes.c_void_p]
sink = torch.zeros(1024, device="cuda")
for mode, name in ((0, "MUFU ex2.approx"), (1, "poly exp2 (FMA pipe)")):
    for nt in (256, 512, 1024):
        out = torch.zeros(1, dtype=torch.int64, device="cuda")
        rc = lib.dash_probe_exp_rate(mode, nt, 4000, 1, ctypes.c_void_p(sink.data_ptr()),
                                     ctypes.c_void_p(out.data_ptr()))
        cyc = out.float().item()
        print(f"{name:22s} threads={nt:4d} rc={rc} cycles/round={cyc:7.1f} exp2/clk/SM={8 * nt / cyc:6.1f}",
              flush=True)
