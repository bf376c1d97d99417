"""dQ-plane budget (include/dash.h dash_attn_bwd_set_plane_budget): when the W
accumulators of all heads exceed the budget, the backward runs the flattened
(b, h) heads in chunks that reuse one set of planes.  Heads are independent
(§2.1) and a chunk keeps every per-head schedule, rank and accumulation
order, so the deterministic results must be bit-identical to the one-chunk
call -- for both kernels, several schedules, and a ragged last chunk -- and the
atomic variant must stay within the north_star tolerance of the oracle."""
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


def _run(dash, g, causal, schedule, det, budget):
    dash.set_plane_budget(budget)
    try:
        shape = tuple(g["q"].shape)
        ws = dash.alloc_workspace(shape, causal, schedule, det, g["q"].device)
        out = dash.attn_bwd(g["q"], g["k"], g["v"], g["o"], g["do"], g["lse"], causal, schedule, det,
                            workspace=ws)
        torch.cuda.synchronize()
        assert dash.check_workspace(shape, causal, schedule, det, ws) == dash.OK
        return [x.clone() for x in out], ws.numel()
    finally:
        dash.set_plane_budget(0)


@pytest.mark.parametrize("d,tile,N,causal,schedule", [
    (128, 256, 2048, True, "descending"),  # CTA-pair kernel, W = 1
    (128, 0, 4096, True, "descending"),    # pair (library choice), W = 2 (two planes per chunk)
    (128, 0, 2048, False, "shift"),        # pair, full-mask cyclic schedule
    (128, 128, 2048, True, "shift"),      # single-CTA kernel (128-row tiles), W = 2
    (64, 0, 2048, False, "naive"),        # d = 64 (2-D tensor-map reduce)
    (64, 0, 8192, True, "descending"),    # d = 64, W = 4, early claim
])
def test_chunked_heads_bit_identical(dash, d, tile, N, causal, schedule):
    B, H = 2, 4  # 8 heads -> chunks of 3, 3, 2
    cpu = attn_inputs(B, N, H, d, seed=11)
    g = {k: v.cuda() for k, v in cpu.items()}
    dash.set_tile(tile)
    try:
        g["o"], g["lse"] = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
        shape = (B, N, H, d)
        W = dash.acc_split(shape, causal, schedule)
        per_head = W * N * d * 4
        ref, ws_full = _run(dash, g, causal, schedule, True, 0)
        assert dash.head_chunk(shape, causal, schedule) == B * H
        dash.set_plane_budget(3 * per_head)
        assert dash.head_chunk(shape, causal, schedule) == 3
        dash.set_plane_budget(0)
        got, ws_chunk = _run(dash, g, causal, schedule, True, 3 * per_head)
        assert ws_chunk < ws_full
        for a, b in zip(ref, got):
            assert torch.equal(a, b)
        one, _ = _run(dash, g, causal, schedule, True, 1)  # one head per launch
        for a, b in zip(ref, one):
            assert torch.equal(a, b)
    finally:
        dash.set_tile(0)


def test_chunked_atomic_variant_matches_oracle(dash):
    B, N, H, d, causal = 1, 1024, 5, 128, True
    cpu = attn_inputs(B, N, H, d, seed=12)
    g = {k: v.cuda() for k, v in cpu.items()}
    g["o"], g["lse"] = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
    (dq, dk, dv), _ = _run(dash, g, causal, "naive", False, 2 * N * d * 4)
    f = {k: v.double().numpy() for k, v in cpu.items()}
    ref = oracle.attn_bwd(f["q"], f["k"], f["v"], f["do"], causal)
    for x, n in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        e = np.max(np.abs(x.double().cpu().numpy() - ref[n])) / np.max(np.abs(ref[n]))
        assert e <= 1e-2, (n, e)


@pytest.mark.parametrize("fused", [True, False])
def test_profile_counts_chunked_launches(dash, fused):
    """dash_profile_end sums the main-kernel intervals of every chunk (and the
    K4 intervals when the dQ finalise is not fused)."""
    B, N, H, d, causal = 1, 2048, 4, 128, True
    cpu = attn_inputs(B, N, H, d, seed=13)
    g = {k: v.cuda() for k, v in cpu.items()}
    g["o"], g["lse"] = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
    dash.set_plane_budget(1)
    dash.set_fused_dq(2 if fused else 0)
    try:
        ws = dash.alloc_workspace((B, N, H, d), causal, "auto", True, "cuda")
        dash.profile_begin()
        for _ in range(2):
            dash.attn_bwd(g["q"], g["k"], g["v"], g["o"], g["do"], g["lse"], causal, "auto", True,
                          workspace=ws)
        pre, main, post, calls = dash.profile_end()
        launches = dash.bwd_launch_count((B, N, H, d), causal, "auto", True)
    finally:
        dash.set_plane_budget(0)
        dash.set_fused_dq(1)
    assert calls == 2 and pre > 0 and main > 0 and post >= 0
    if not fused:
        assert post > 0
    assert launches == 1 + H * (1 if fused else 2)  # one head per chunk
