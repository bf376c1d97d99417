"""GPU probes pinning the tcgen05 / TMA layout conventions the backward kernel uses.

These do not involve the oracle: they check one UMMA GEMM against torch's
fp32 matmul of the same bf16 operands (the "plain PyTorch reference" for a
single contraction) and the TMA SWIZZLE_128B smem layout against the
documented Swizzle<3,4,3> address mapping that csrc/umma.cuh assumes.
"""
import ctypes
import os

import numpy as np
import pytest
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
PROBE = os.path.join(os.path.dirname(HERE), "paper_2601_21824_b200", "libdash_probe.so")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def probe():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_21824_b200 import build as b
    b.build()
    lib = ctypes.CDLL(PROBE)
    lib.dash_probe_umma.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p] * 3
    lib.dash_probe_umma_ts.argtypes = [ctypes.c_int] * 3 + [ctypes.c_void_p] * 3
    lib.dash_probe_tma.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_void_p]
    return lib


@pytest.mark.parametrize("n,k", [(64, 64), (64, 128), (128, 64), (128, 128)])
@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
def test_umma_gemm_layouts(probe, n, k, a_mn, b_mn):
    g = torch.Generator().manual_seed(n * 1000 + k + 10 * a_mn + 100 * b_mn)
    A = torch.randn(128, k, generator=g).to(torch.bfloat16)
    Bt = torch.randn(n, k, generator=g).to(torch.bfloat16)
    ref = A.float() @ Bt.float().T
    dA, dB = A.cuda(), Bt.cuda()
    D = torch.zeros(128, n, device="cuda", dtype=torch.float32)
    rc = probe.dash_probe_umma(n, k, a_mn, b_mn, dA.data_ptr(), dB.data_ptr(), D.data_ptr())
    assert rc == 0
    torch.testing.assert_close(D.cpu(), ref, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("n,k", [(128, 64), (64, 128), (128, 128)])
@pytest.mark.parametrize("b_mn", [0, 1])
def test_umma_ts_a_from_tmem(probe, n, k, b_mn):
    """A operand in TMEM (lane = row, two bf16 per column), B from smem."""
    g = torch.Generator().manual_seed(7 * n + k + b_mn)
    A = torch.randn(128, k, generator=g).to(torch.bfloat16)
    Bt = torch.randn(n, k, generator=g).to(torch.bfloat16)
    ref = A.float() @ Bt.float().T
    dA, dB = A.cuda(), Bt.cuda()  # keep both alive: no allocator reuse of a temporary
    D = torch.zeros(128, n, device="cuda", dtype=torch.float32)
    rc = probe.dash_probe_umma_ts(n, k, b_mn, dA.data_ptr(), dB.data_ptr(), D.data_ptr())
    assert rc == 0
    torch.testing.assert_close(D.cpu(), ref, rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("rows,cols", [(64, 64), (128, 128), (64, 128)])
def test_tma_swizzle128_layout(probe, rows, cols):
    ld = cols * 3  # the box is a sub-matrix of a wider tensor
    src = torch.arange(rows * ld, dtype=torch.int32).remainder(30000).to(torch.int16)
    src = src.view(torch.bfloat16).view(rows, ld).cuda()
    out = torch.zeros(rows * cols * 2, dtype=torch.uint8, device="cuda")
    assert probe.dash_probe_tma(src.data_ptr(), rows, cols, ld, out.data_ptr()) == 0
    sm = out.cpu().numpy().view(np.int16)
    ref = src.cpu().view(torch.int16).numpy()
    for r in range(rows):
        for ch in range(cols // 8):
            blk, c = divmod(ch, 8)
            off = (blk * rows * 128 + r * 128 + ((c ^ (r & 7)) << 4)) // 2
            assert np.array_equal(sm[off:off + 8], ref[r, ch * 8: ch * 8 + 8]), (r, ch)
