"""Microbenchmark: TMA load latency of a Q sub-tile box (2 x [64 cols x rows] bf16,
row stride H*d*2 = 4 KB as in [B,N,H,d] with H*d = 2048)."""
import ctypes, os
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2601_21824_b200", "libdash_probe.so"))
lib.dash_probe_tma_latency.argtypes = [ctypes.c_void_p] + [ctypes.c_int] * 5 + [ctypes.c_void_p]
rows_total, ld = 16384, 2048
src = torch.randn(rows_total, ld, device="cuda").to(torch.bfloat16)
for grid in (1, 148):
    for rows in (64, 128):
        out = torch.zeros(grid, dtype=torch.int64, device="cuda")
        rc = lib.dash_probe_tma_latency(ctypes.c_void_p(src.data_ptr()), rows_total, ld, rows, 200, grid, ctypes.c_void_p(out.data_ptr()))
        print(f"grid={grid:3d} rows={rows:3d} rc={rc} cycles issue->complete: mean {out.float().mean().item():.0f}  max {out.max().item()}")
