"""CPU tests of the C-ABI library: it loads, exports every declared symbol, and
its host-side logic (schedule tables, DAG critical path, argument checks)
matches the independent oracle bit for bit.  No GPU compute calls."""
import ctypes
import os
import re
import subprocess

import pytest

from oracle import dag_oracle as dag

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dash():
    from paper_2601_21824_b200 import build
    build.build()
    from paper_2601_21824_b200 import dash as d
    return d


def _declared_functions():
    text = open(os.path.join(ROOT, "include", "dash.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(dash_[a-z0-9_]+)\s*\(", text)))


def test_exports_every_declared_symbol(dash):
    names = _declared_functions()
    assert len(names) >= 10
    nm = subprocess.run(["nm", "-D", "--defined-only", dash.LIB_PATH], capture_output=True,
                        text=True, check=True).stdout
    exported = set(re.findall(r"\bT (dash_\w+)", nm))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(dash.LIB_PATH)
    for n in names:
        getattr(lib, n)


def test_status_strings_and_version(dash):
    assert dash.status_string(0) == "DASH_OK"
    assert dash.status_string(5) == "DASH_ERR_DEADLOCK"
    assert "sm_100a" in dash.version()
    assert dash.bwd_launches(1, dash.SHIFT, 1) >= 1


@pytest.mark.parametrize("schedule", [dag.NAIVE, dag.DESCENDING, dag.SHIFT])
@pytest.mark.parametrize("mask", [dag.FULL, dag.CAUSAL])
def test_schedule_table_matches_oracle(dash, schedule, mask):
    """The product's closed-form tables equal the oracle's definition-driven ones."""
    # + grouped SHIFT full (AMB-30: 129, 257) and causal (AMB-35: 257, 258, 301, 512, 513)
    for n in list(range(1, 70)) + [129, 256, 257, 258, 301, 512, 513]:
        jobs = dash.schedule_table(schedule, n, mask)
        ojobs = dag.build_jobs(schedule, n, mask)
        ranks = dag.reduction_ranks(schedule, n, mask)
        assert len(jobs) == len(ojobs)
        for job, ojob in zip(jobs, ojobs):
            assert [(i, j) for i, j, _ in job] == ojob.tasks
            assert [rk for _, _, rk in job] == [ranks[t] for t in ojob.tasks]


def test_critical_path_matches_oracle_simulator(dash):
    """Bit-exact int64 parity over schedule x mask x n x m x (c, r) x n_sm (T2)."""
    checked = 0
    for schedule in (dag.NAIVE, dag.DESCENDING, dag.SHIFT):
        for mask in (dag.FULL, dag.CAUSAL):
            for n in list(range(2, 17)) + [24, 32, 48, 64]:
                for m in (1, 2, 3, 5):
                    for c, r in ((1, 1), (3, 1), (1, 3), (7, 4)):
                        for n_sm in {n, max(1, n // 2 + 1), n + 3}:
                            try:
                                want = dag.simulate(schedule, n, mask, m, n_sm, c, r)
                            except dag.Deadlock:
                                with pytest.raises(dash.DashError) as e:
                                    dash.schedule_critical_path(schedule, n, n, mask, m, n_sm, c, r)
                                assert e.value.status == dash.ERR_DEADLOCK
                                continue
                            got = dash.schedule_critical_path(schedule, n, n, mask, m, n_sm, c, r)
                            assert got == want, (schedule, mask, n, m, c, r, n_sm)
                            checked += 1
    assert checked > 2000


def test_critical_path_grouped_shift_matches_oracle(dash):
    """Grouped SHIFT (AMB-30 full, AMB-35 causal): the product's DAG model equals
    the oracle simulator on one group's worth of SMs and on the whole device."""
    for mask, n in ((dag.CAUSAL, 258), (dag.CAUSAL, 301), (dag.FULL, 257)):
        for n_sm in (65, 129, 148):
            try:
                want = dag.simulate(dag.SHIFT, n, mask, 1, n_sm, 3, 1)
            except dag.Deadlock:
                with pytest.raises(dash.DashError):
                    dash.schedule_critical_path(dash.SHIFT, n, n, mask, 1, n_sm, 3, 1)
                continue
            assert dash.schedule_critical_path(dash.SHIFT, n, n, mask, 1, n_sm, 3, 1) == want


def test_critical_path_defaults_and_errors(dash):
    for n in (4, 16, 128):
        assert dash.schedule_critical_path(dash.NAIVE, n, n, dash.CAUSAL) == 5 * n - 1
        assert dash.schedule_critical_path(dash.DESCENDING, n, n, dash.CAUSAL) == 3 * n + 1
        assert dash.schedule_critical_path(dash.SHIFT, n, n, dash.FULL) == 4 * n
        assert dash.schedule_critical_path(dash.SHIFT, n, n, dash.CAUSAL) == 2 * n + 2
    bad = [
        dict(schedule=0, n_q=4, n_kv=5, mask=0),
        dict(schedule=7, n_q=4, n_kv=4, mask=0),
        dict(schedule=0, n_q=4, n_kv=4, mask=3),
        dict(schedule=0, n_q=4, n_kv=4, mask=0, c=0),
        dict(schedule=0, n_q=4, n_kv=4, mask=0, r=0),
        dict(schedule=0, n_q=4, n_kv=4, mask=0, n_sm=0),
    ]
    for kw in bad:
        with pytest.raises(dash.DashError) as e:
            dash.schedule_critical_path(**kw)
        assert e.value.status == dash.ERR_INVALID_ARG
    # odd n_kv Symmetric Shift (AMB-29) is defined; the model agrees with the oracle
    assert dash.schedule_critical_path(dash.SHIFT, 5, 5, dash.CAUSAL) == \
        dag.simulate(dag.SHIFT, 5, dag.CAUSAL, 2, 5, 1, 1)
    with pytest.raises(dash.DashError) as e:
        dash.schedule_critical_path(dash.SHIFT, 8, 8, dash.FULL, n_heads=2, n_sm=7)
    assert e.value.status == dash.ERR_DEADLOCK


def test_workspace_bytes_and_shape_checks(dash):
    ws = dash.workspace_bytes((2, 1024, 16, 128), True)
    assert ws >= 2 * 16 * 1024 * 128 * 4 + 2 * 16 * 1024 * 4
    assert dash.workspace_bytes((2, 1000, 16, 128), True) == 0      # N % 128 != 0
    assert dash.workspace_bytes((2, 1024, 16, 96), True) == 0       # d not in {64, 128}
    assert dash.workspace_bytes((0, 1024, 16, 128), True) == 0
    assert dash.host_workspace_bytes((1, 256, 1, 64), False) > dash.workspace_bytes((1, 256, 1, 64), False)


def test_plane_budget_bounds_config4_workspace(dash):
    """BASELINE config 4 (B = 8, H = 32, N = 32k, d = 128, causal): the W = 8
    accumulators of all 256 heads would be 32 GiB; under the default 4 GiB
    dQ-plane budget the heads run in chunks of 32 (8 launches) and the whole
    workspace stays under 8 GiB.  Smaller budgets shrink the chunk; a budget
    below one head's planes still runs one head per launch."""
    cfg4 = (8, 32768, 32, 128)
    per_head = 8 * 32768 * 128 * 4
    try:
        dash.set_plane_budget(0)
        assert dash.acc_split(cfg4, True, "auto") == 8
        assert dash.head_chunk(cfg4, True, "auto") == (4 << 30) // per_head == 32
        ws = dash.workspace_bytes(cfg4, True, "auto")
        assert ws < 8 << 30
        assert ws >= 32 * per_head + 2 * 8 * 32 * 32768 * 4  # planes + D + lse2 of all heads
        # the bench sweep shapes fit one chunk
        for N in (512, 2048, 16384):
            shp = (16384 // N, N, 16, 128)
            assert dash.head_chunk(shp, True, "auto") == shp[0] * shp[2]
        dash.set_plane_budget(3 * per_head + 5)
        assert dash.head_chunk(cfg4, True, "auto") == 3
        assert dash.workspace_bytes(cfg4, True, "auto") < ws
        dash.set_plane_budget(1)
        assert dash.head_chunk(cfg4, True, "auto") == 1
        # the atomic variant has one accumulator: 8 x the heads per chunk
        dash.set_plane_budget(0)
        assert dash.head_chunk(cfg4, True, "auto", deterministic=False) == 256
        assert dash.head_chunk((1, 200, 1, 64), True) == 0
    finally:
        dash.set_plane_budget(0)


def test_bwd_rejects_bad_arguments_without_gpu(dash):
    """Argument validation happens before any device call."""
    lib = dash.lib()
    shp = dash.Shape(1, 256, 1, 64, 0.0)
    p = ctypes.c_void_p(1 << 20)  # aligned dummy address, never dereferenced
    nul = ctypes.c_void_p(0)
    args = [p] * 9
    st = lib.dash_attn_bwd(ctypes.byref(shp), nul, *args[1:], 0, 0, 1, p, 1 << 30, nul)
    assert st == dash.ERR_INVALID_ARG
    st = lib.dash_attn_bwd(ctypes.byref(shp), ctypes.c_void_p((1 << 20) + 4), *args[1:], 0, 0, 1, p,
                           1 << 30, nul)
    assert st == dash.ERR_INVALID_ARG
    st = lib.dash_attn_bwd(ctypes.byref(shp), *args, 0, 9, 1, p, 1 << 30, nul)
    assert st == dash.ERR_INVALID_ARG
    st = lib.dash_attn_bwd(ctypes.byref(shp), *args, 0, 0, 1, p, 16, nul)
    assert st == dash.ERR_WORKSPACE
    bad = dash.Shape(1, 200, 1, 64, 0.0)
    st = lib.dash_attn_bwd(ctypes.byref(bad), *args, 0, 0, 1, p, 1 << 30, nul)
    assert st == dash.ERR_INVALID_ARG


def test_auto_schedule_policy_and_acc_split(dash):
    """DASH_SCHED_AUTO resolves to one of the paper's three schedules by the
    documented rule (include/dash.h); the automatic accumulator split depends
    on N only (AMB-27), so (b, h) sharding can never change it."""
    cases = [  # (N, d, causal) -> schedule
        ((512, 128, True), "shift"), ((4096, 128, True), "shift"), ((8192, 128, True), "descending"),
        ((16384, 128, True), "descending"), ((8192, 64, True), "shift"), ((16384, 64, True), "descending"),
        ((4096, 128, False), "shift"), ((8192, 128, False), "naive"), ((16384, 64, False), "naive"),
    ]
    for (N, d, causal), want in cases:
        assert dash.resolve_schedule((1, N, 16, d), causal, "auto") == want, (N, d, causal)
        for b, h in ((8, 32), (1, 1)):  # independent of B and H
            assert dash.resolve_schedule((b, N, h, d), causal, "auto") == want
        assert dash.resolve_schedule((1, N, 16, d), causal, "naive") == "naive"
    old = dash.acc_split()
    try:
        dash.set_acc_split(0)
        # single-CTA kernel (d = 64, 128-row tiles): n = N / 128
        assert [dash.acc_split((1, N, 16, 64), True) for N in (512, 4096, 8192, 16384, 32768)] == \
            [2, 2, 4, 4, 8]
        # d = 128: single-CTA kernel (n = N / 128) below N = 4096 causal / 2048 full,
        # then the CTA-pair kernel (n = N / 256)
        assert [dash.tile((1, N, 16, 128), True) for N in (512, 2048, 4096, 32768)] == [128, 128, 256, 256]
        assert [dash.tile((1, N, 16, 128), False) for N in (1024, 2048)] == [128, 256]
        assert [dash.acc_split((1, N, 16, 128), True) for N in (512, 2048, 4096, 8192, 16384, 32768)] == \
            [2, 2, 2, 4, 4, 8]
        assert [dash.acc_split((1, N, 16, 128), False) for N in (1024, 2048, 4096)] == [2, 1, 2]
        try:  # the pair kernel forced at short N: n' <= 8 -> the paper's single accumulator
            dash.set_tile(256)
            assert dash.tile((1, 512, 16, 128), True) == 256
            assert [dash.acc_split((1, N, 16, 128), True) for N in (512, 2048)] == [1, 1]
        finally:
            dash.set_tile(0)
        assert dash.acc_split((1, 8192, 16, 128), True) == dash.acc_split((8, 8192, 32, 128), True)
        for w in (1, 2, 4, 8):
            dash.set_acc_split(w)
            assert dash.acc_split((1, 1024, 2, 128), False) == w and dash.acc_split() == w
        with pytest.raises(dash.DashError):
            dash.set_acc_split(3)
    finally:
        dash.set_acc_split(old)
    with pytest.raises(dash.DashError):  # AUTO is not a schedule of the DAG model
        dash.schedule_critical_path(dash.AUTO, 4, 4, dash.CAUSAL)


def test_critical_path_every_n_4_to_128(dash):
    """BASELINE configs[4] (AMB-20): for every n_q = n_kv in 4..128, both masks
    and all three schedules, the product's DAG model equals the oracle's
    brute-force simulator bit for bit -- at the SURVEY default (m = 2, n_sm =
    n, c = r = 1) and at a c > r point with four heads -- and, where the paper
    states a closed form (AMB-8/9/10), both equal it.
    SHIFT causal with odd n runs the AMB-29 schedule (no closed form)."""
    for n in range(4, 129):
        for mask in (dag.FULL, dag.CAUSAL):
            for schedule in (dag.NAIVE, dag.DESCENDING, dag.SHIFT):
                for m, c, r in ((2, 1, 1), (4, 3, 1)):
                    want = dag.simulate(schedule, n, mask, m, n, c, r)
                    got = dash.schedule_critical_path(schedule, n, n, mask, m, n, c, r)
                    assert got == want, (schedule, mask, n, m, c, r)
                    if schedule == dag.NAIVE or (schedule == dag.DESCENDING and mask == dag.FULL):
                        form = m * n * (c + r) + (n - 1) * r
                    elif schedule == dag.DESCENDING:                   # c >= r here (AMB-9)
                        form = m * (n + 1) * (c + r) // 2 + (n - 1) * r
                    elif mask == dag.FULL:
                        form = m * n * (c + r)
                    elif n % 2 == 0:
                        form = ((m + 1) // 2) * (n + 1) * (c + r)
                    else:
                        form = None
                    if form is not None:
                        assert got == form, (schedule, mask, n, m, c, r)
