"""Microbenchmark: cta_group::2 tcgen05.mma throughput for the pair kernel's GEMM shapes."""
import ctypes
import os

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = ctypes.CDLL(os.path.join(ROOT, "paper_2601_21824_b200", "libdash_probe.so"))
lib.dash_probe_pair_mma_rate.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p]
shapes = {0: ("S^T/dP^T M=256 N=64 K=128 SS", 256 * 64 * 128),
          1: ("dV/dK M=256 N=128 K=64 TS", 256 * 128 * 64),
          2: ("dQ^T M=128 N=64 K=256 SS (B SW64)", 128 * 64 * 256),
          3: ("one sub-tile: S,dP,dK,dV,dQ (pair)", 2 * 256 * 64 * 128 + 2 * 256 * 128 * 64 + 128 * 64 * 256)}
for clusters in (1, 74):
    for mode, (name, macs) in shapes.items():
        out = torch.zeros(clusters, dtype=torch.int64, device="cuda")
        rc = lib.dash_probe_pair_mma_rate(mode, 2000, clusters, ctypes.c_void_p(out.data_ptr()))
        cyc = out.float().mean().item()
        ideal = macs / (2 * 4096)  # two SMs at 4096 bf16 MAC/clk each
        print(f"clusters={clusters:3d} {name:36s} rc={rc} cycles/GEMM={cyc:7.1f} ideal={ideal:6.1f} eff={ideal / cyc:5.2f}",
              flush=True)
