"""Microbenchmark: cycles per K=128 GEMM (8 tcgen05.mma of 128 x N x 16) by operand mode."""
import ctypes, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2601_21824_b200", "libdash_probe.so"))
lib.dash_probe_mma_rate.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p]
modes = {0: "SS A:K B:K", 1: "SS A:K B:MN", 2: "SS A:MN B:MN", 3: "TS B:MN"}
for grid in (1, 148):
    for n in (64, 128, 256):
        for m, name in modes.items():
            out = torch.zeros(grid, dtype=torch.int64, device="cuda")
            rc = lib.dash_probe_mma_rate(n, m, 2000, grid, ctypes.c_void_p(out.data_ptr()))
            cyc = out.float().mean().item()
            ideal = 8 * 128 * n / 256
            print(f"grid={grid:3d} N={n:3d} {name:14s} rc={rc} cycles/GEMM={cyc:7.1f} ideal={ideal:6.1f} eff={ideal/cyc:5.2f}")
