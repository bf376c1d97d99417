"""Fused dQ finalise (include/dash.h
dash_attn_bwd_set_fused_dq): the main kernel turns the W fp32 accumulators
into the bf16 dQ itself -- CTAs whose jobs ran out convert the heads whose
jobs have all completed -- instead of the separate K4 convert kernel.  The
sum is K4's, ((acc_0 + acc_1) + ...) * scale in fp32, to bf16 (P:396 gives
one accumulator; AMB-27 the W interleaved ones), so dq must be bit-identical
to the K4 path for every kernel, schedule, W, the atomic variant and chunked
heads, and within the north_star tolerance of the fp64 oracle."""
import numpy as np
import pytest
import torch

import oracle
from paper_2601_21824_b200.inputs import attn_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dash():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2601_21824_b200 import build
    build.build()
    from paper_2601_21824_b200 import dash as d
    return d


def _bwd(dash, g, causal, schedule, det, fused):
    dash.set_fused_dq(2 if fused else 0)
    try:
        shape = tuple(g["q"].shape)
        ws = dash.alloc_workspace(shape, causal, schedule, det, g["q"].device)
        ws.fill_(7)  # a recycled workspace: done[] / tickets must be reset by the call
        out = dash.attn_bwd(g["q"], g["k"], g["v"], g["o"], g["do"], g["lse"], causal, schedule,
                            det, workspace=ws)
        torch.cuda.synchronize()
        assert dash.check_workspace(shape, causal, schedule, det, ws) == dash.OK
        return [x.clone() for x in out]
    finally:
        dash.set_fused_dq(1)


def _inputs(dash, B, N, H, d, causal, seed):
    cpu = attn_inputs(B, N, H, d, seed=seed)
    g = {k: v.cuda() for k, v in cpu.items()}
    g["o"], g["lse"] = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
    return cpu, g


def test_fused_mode_default_and_launch_count(dash):
    assert dash.fused_dq() == 1
    assert dash.bwd_launch_count((1, 2048, 4, 128), True) == 2  # K1 + main (finalise fused)
    assert dash.bwd_launch_count((4, 1024, 4, 128), True) == 3  # K1 + main + K4
    dash.set_fused_dq(2)
    try:
        assert dash.bwd_launch_count((4, 1024, 4, 128), True) == 2
    finally:
        dash.set_fused_dq(1)
    with pytest.raises(Exception):
        dash.set_fused_dq(3)


@pytest.mark.parametrize("B,N,H,d,tile,causal,schedule,W", [
    (4, 512, 8, 128, 128, True, "shift", 0),       # single-CTA, many heads, W = 2
    (2, 1024, 4, 128, 128, False, "naive", 1),     # single-CTA, W = 1
    (1, 2048, 4, 128, 128, True, "descending", 4),
    (2, 4096, 4, 128, 256, True, "descending", 0),  # CTA pair
    (1, 4096, 2, 128, 256, False, "shift", 8),      # pair, W = 8 (every plane live at n = 16)
    (1, 2048, 8, 128, 256, True, "naive", 1),
    (8, 512, 8, 64, 0, True, "shift", 0),           # d = 64
    (3, 384, 2, 64, 0, True, "shift", 0),           # d = 64, ragged last finalise task (256 rows)
    (2, 128, 3, 64, 0, False, "naive", 0),          # one KV tile, one partial task
    (1, 4096, 4, 64, 0, False, "descending", 4),
    (1, 8192, 2, 64, 0, True, "descending", 8),
])
def test_fused_equals_k4_bitwise(dash, B, N, H, d, tile, causal, schedule, W):
    _, g = _inputs(dash, B, N, H, d, causal, seed=N + d)
    dash.set_tile(tile)
    dash.set_acc_split(W)
    try:
        ref = _bwd(dash, g, causal, schedule, True, False)
        got = _bwd(dash, g, causal, schedule, True, True)
    finally:
        dash.set_tile(0)
        dash.set_acc_split(0)
    for a, b, n in zip(ref, got, ("dq", "dk", "dv")):
        assert torch.equal(a, b), n


@pytest.mark.parametrize("d,tile", [(128, 128), (128, 256), (64, 0)])
@pytest.mark.parametrize("causal", [True, False])
def test_fused_atomic_variant_matches_oracle(dash, d, tile, causal):
    B, N, H = 1, 1024, 6
    cpu, g = _inputs(dash, B, N, H, d, causal, seed=5)
    dash.set_tile(tile)
    try:
        dq, dk, dv = _bwd(dash, g, causal, "naive", False, True)
    finally:
        dash.set_tile(0)
    f = {k: v.double().numpy() for k, v in cpu.items()}
    ref = oracle.attn_bwd(f["q"], f["k"], f["v"], f["do"], causal)
    for x, n in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        e = np.max(np.abs(x.double().cpu().numpy() - ref[n])) / np.max(np.abs(ref[n]))
        assert e <= 1e-2, (n, e)


@pytest.mark.parametrize("tile", [128, 256])
def test_fused_chunked_heads_bit_identical(dash, tile):
    """Chunks of 3, 3, 2 heads: each chunk's launch finalises its own heads."""
    B, N, H, d, causal, schedule = 2, 2048, 4, 128, True, "descending"
    _, g = _inputs(dash, B, N, H, d, causal, seed=21)
    dash.set_tile(tile)
    try:
        ref = _bwd(dash, g, causal, schedule, True, False)
        W = dash.acc_split((B, N, H, d), causal, schedule)
        dash.set_plane_budget(3 * W * N * d * 4)
        try:
            got = _bwd(dash, g, causal, schedule, True, True)
        finally:
            dash.set_plane_budget(0)
    finally:
        dash.set_tile(0)
    for a, b in zip(ref, got):
        assert torch.equal(a, b)


def test_fused_repeated_runs_identical(dash):
    """Finalise tasks are claimed dynamically; the bits must not depend on who
    converts which rows."""
    B, N, H, d, causal = 4, 1024, 8, 128, True
    _, g = _inputs(dash, B, N, H, d, causal, seed=9)
    first = _bwd(dash, g, causal, "shift", True, True)
    for _ in range(20):
        again = _bwd(dash, g, causal, "shift", True, True)
        for a, b in zip(first, again):
            assert torch.equal(a, b)
