"""Microbenchmark: cycles to red.global.add a 32 KB fp32 tile (per CTA), by grid size."""
import ctypes, os
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2601_21824_b200", "libdash_probe.so"))
lib.dash_probe_red_rate.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
for grid in (1, 148):
    for mode in (0, 1):
        dst = torch.zeros(grid * 64 * 128, device="cuda")
        out = torch.zeros(grid, dtype=torch.int64, device="cuda")
        rc = lib.dash_probe_red_rate(ctypes.c_void_p(dst.data_ptr()), 200, mode, grid, ctypes.c_void_p(out.data_ptr()))
        print(f"grid={grid} mode={mode} rc={rc} cycles per 32KB tile = {out.float().mean().item():.0f}  check={dst[0].item()}")
