"""T5 replay (SURVEY.md §8(c) c4 "GPU exact order"): the ordered dQ reduction
is pinned bit for bit, not just to a tolerance.

dash_attn_bwd_dump hands back every dQ partial dQ_local = dS K_i (Alg.1 line
28) exactly as it entered the reduction.  The host then re-sums each
dQ tile's partials in the order the paper prescribes -- the ranks come from
oracle/dag_oracle.reduction_ranks, built from the paper's schedule
definitions (AMB-6), not from the product's tables --
with one IEEE fp32 round-to-nearest add per contribution (Alg.1 line 34,
P:396), then applies dq = bf16_rn(scale * sum) (AMB-14).  With W interleaved
accumulators (AMB-27) each accumulator w re-sums ranks w, w + W, ... and the
convert adds them in index order.  The GPU's fp32 accumulators and its dq must
match those bits exactly.  A wrong rank,
a skipped or doubled contribution, an add that raced its predecessor, or a
scale applied per partial all change bits.
"""
import numpy as np
import pytest
import torch

from oracle import dag_oracle as dag
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


def bf16_rn_bits(x32: np.ndarray) -> np.ndarray:
    """IEEE binary32 -> bfloat16 bit pattern, round to nearest even (finite inputs)."""
    u = x32.astype(np.float32).view(np.uint32).astype(np.uint64)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


@pytest.fixture(params=[1, 2, 4, 8], ids=lambda w: f"W{w}")
def acc_split(request, dash):
    """Run the test under W interleaved accumulators (AMB-27), then restore."""
    old = dash.acc_split()
    dash.set_acc_split(request.param)
    yield request.param
    dash.set_acc_split(old)


@pytest.mark.parametrize("N", [512, 384])
@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("schedule", ["naive", "descending", "shift"])
def test_dq_equals_host_resum_in_paper_order(dash, acc_split, N, d, causal, schedule):
    _replay(dash, acc_split, 1, N, 2, d, causal, schedule)


@pytest.mark.parametrize("W", [4, 8])
@pytest.mark.parametrize("d,N", [(64, 2176), (128, 2176), (128, 4352)])
@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("schedule", ["naive", "descending", "shift"])
def test_replay_every_plane_live(dash, W, d, N, causal, schedule):
    """n = 17 KV tiles (N = 2176 with 128-row tiles; N = 4352 with the CTA-pair
    kernel's 256-row tiles): with W = 8 every accumulator plane of every
    Q tile with >= 2W + 1 contributors receives >= 2 ordered adds (the
    ticket-order path, not just the rank-0 store); the busiest tiles
    (17 contributors) give plane 0 three adds and planes 1-7 two."""
    old = dash.acc_split()
    dash.set_acc_split(W)
    try:
        per_plane = _replay(dash, W, 1, N, 1, d, causal, schedule)
    finally:
        dash.set_acc_split(old)
    assert all(c >= 2 for c in per_plane[:W]), per_plane


def _replay(dash, W, B, N, H, d, causal, schedule):
    """Re-sum the dumped partials in the paper's order, compare bits; returns,
    per accumulator plane, the largest number of adds it received in one tile."""
    T = dash.tile((B, N, H, d), causal, schedule)  # tile rows: 128, or 256 (CTA-pair kernel)
    n = N // T
    mask = dag.CAUSAL if causal else dag.FULL
    sched = {"naive": dag.NAIVE, "descending": dag.DESCENDING, "shift": dag.SHIFT}[schedule]
    g = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=7).items()}
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
    (dq, _, _), parts, ws = dash.attn_bwd_dump(g["q"], g["k"], g["v"], o, g["do"], lse, causal,
                                               schedule, True)
    torch.cuda.synchronize()
    parts = parts.cpu().numpy()                                        # [B*H, N/T, N, d] fp32
    assert dash.acc_split((B, N, H, d), causal, schedule) == W         # AMB-27
    acc_gpu = ws[: W * B * H * N * d * 4].view(torch.float32).cpu().numpy().reshape(W, B * H, N, d)
    dq_bits = dq.view(torch.int16).cpu().numpy().view(np.uint16)     # [B, N, H, d]
    scale = np.float32(1.0) / np.sqrt(np.float32(d))
    rank = dag.reduction_ranks(sched, n, mask)

    def contribution(bh, i, j):
        """KV tile i's partial for Q tile j, as it enters the ordered reduction."""
        return parts[bh, i, j * T:(j + 1) * T]

    checked_acc = 0
    per_plane = [0] * W
    for bh in range(B * H):
        b, h = divmod(bh, H)
        for j in range(n):
            order = sorted((rk, i) for (i, jj), rk in rank.items() if jj == j)
            assert [rk for rk, _ in order] == list(range(len(order)))
            rows = slice(j * T, (j + 1) * T)
            accs = []
            for w in range(min(W, len(order))):
                # accumulator w: ranks w, w + W, ... in order; its first one stores
                mine = [i for rk, i in order if rk % W == w]
                per_plane[w] = max(per_plane[w], len(mine))
                acc = contribution(bh, mine[0], j).copy()
                for i in mine[1:]:
                    acc = (acc + contribution(bh, i, j)).astype(np.float32)
                np.testing.assert_array_equal(acc_gpu[w, bh, rows].view(np.uint32), acc.view(np.uint32),
                                              err_msg=f"dQacc[{w}] bh={bh} tile={j}")
                accs.append(acc)
            checked_acc += len(order) >= 2
            acc = accs[0]
            for extra in accs[1:]:                              # convert: acc_0 + acc_1
                acc = (acc + extra).astype(np.float32)
            want = bf16_rn_bits((acc * scale).astype(np.float32))
            got = dq_bits[b, rows, h, :]
            bad = np.count_nonzero(got != want)
            assert bad == 0, f"dq bh={bh} tile={j}: {bad} of {want.size} bf16 values differ"
    assert checked_acc > 0
    return per_plane


def test_partials_cover_exactly_the_visited_tiles(dash):
    """Every (KV tile, Q tile) task the mask admits hands a partial to the
    reduction, and no other: rows of tiles a KV tile never visits stay zero."""
    B, N, H, d = 1, 512, 1, 128
    g = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=3).items()}
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], True)
    _, parts, _ = dash.attn_bwd_dump(g["q"], g["k"], g["v"], o, g["do"], lse, True, "shift", True)
    parts = parts.cpu().numpy()[0]
    T = dash.tile((B, N, H, d), True, "shift")
    for i in range(N // T):
        for j in range(N // T):
            blk = parts[i, j * T:(j + 1) * T]
            if j >= i:
                assert np.count_nonzero(blk) > blk.size // 2, (i, j)
            else:
                assert not np.any(blk), (i, j)


@pytest.mark.parametrize("causal", [False, True])
@pytest.mark.parametrize("schedule", ["naive", "descending", "shift"])
@pytest.mark.parametrize("W", [1, 2])
@pytest.mark.parametrize("tile", [128, 256])
def test_replay_both_kernels_d128(dash, tile, W, causal, schedule):
    """d = 128, N = 512: the library runs the single-CTA kernel here
    (dash_attn_bwd_tile); dash_attn_bwd_set_tile forces either kernel, and the
    ordered reduction of each is replayed at the same shape."""
    old_w = dash.acc_split()
    dash.set_tile(tile)
    dash.set_acc_split(W)
    try:
        assert dash.tile((1, 512, 2, 128), causal, schedule) == tile
        _replay(dash, W, 1, 512, 2, 128, causal, schedule)
    finally:
        dash.set_tile(0)
        dash.set_acc_split(old_w)


def test_replay_grouped_symmetric_shift(dash):
    """AMB-35: causal SHIFT with n = 258 KV tiles (129 pairs > the 128-pair
    group) runs in two groups of 64 / 65 pairs; every dQ tile's partials,
    re-summed group-major in visit-step order (the oracle's ranks), give the
    GPU's accumulator and dq bits (d = 64, N = 33024, one head, W = 8)."""
    B, N, H, d = 1, 33024, 1, 64
    W = dash.acc_split((B, N, H, d), True, "shift")
    per_plane = _replay(dash, W, B, N, H, d, True, "shift")
    assert all(c >= 2 for c in per_plane[:W]), per_plane
