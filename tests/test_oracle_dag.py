"""Pins for the DAG schedule oracle (oracle/dag_oracle.py) -- CPU only.

The oracle's simulator is pinned to the paper's own statements: the closed
forms, the worked examples of Fig. 2 and
Fig. 4, Lemma 1 by brute force, and the structural
properties of §3.1/§3.4.
"""
import os
import random

import pytest

from oracle import dag_oracle as dag
from oracle.dag_oracle import CAUSAL, DESCENDING, FULL, NAIVE, SHIFT

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# --- closed forms -----------------------------------------------------------

CR = [(1, 1), (2, 1), (3, 1), (5, 2), (4, 4), (7, 3), (1, 2), (1, 3)]


@pytest.mark.parametrize("c,r", CR)
def test_closed_forms_naive(c, r):
    """T = m*n*(c+r) + (n-1)*r for both masks (§3.2; AMB-8)."""
    for n in range(2, 13):
        for m in range(1, 6):
            for mask in (FULL, CAUSAL):
                assert dag.simulate(NAIVE, n, mask, m, n, c, r) == m * n * (c + r) + (n - 1) * r


@pytest.mark.parametrize("c,r", CR)
def test_closed_forms_shift(c, r):
    """T_full_opt = m*n*(c+r); T_causal_opt = m*(n+1)*(c+r)/2 (AMB-10)."""
    for n in range(2, 13):
        for m in range(1, 6):
            assert dag.simulate(SHIFT, n, FULL, m, n, c, r) == m * n * (c + r)
            if n % 2 == 0:
                t = dag.simulate(SHIFT, n, CAUSAL, m, n, c, r)
                assert t == ((m + 1) // 2) * (n + 1) * (c + r)
                if m % 2 == 0:
                    assert 2 * t == m * (n + 1) * (c + r)


@pytest.mark.parametrize("c,r", [cr for cr in CR if cr[0] >= cr[1]])
def test_closed_forms_descending_causal(c, r):
    """T_reversed = m*(n+1)*(c+r)/2 + (n-1)*r for even m (§3.3; AMB-9)."""
    for n in range(2, 13):
        for m in range(1, 7):
            t = dag.simulate(DESCENDING, n, CAUSAL, m, n, c, r)
            if m % 2 == 0:
                assert t == m * (n + 1) * (c + r) // 2 + (n - 1) * r
            else:
                assert t == (m - 1) * (n + 1) * (c + r) // 2 + n * (c + r)


@pytest.mark.parametrize("c,r", [(1, 2), (1, 3), (2, 5)])
def test_descending_causal_m2_any_c_r(c, r):
    """P:103's form for m = 2 holds for any c, r (AMB-9 limits only m >= 3, c < r)."""
    for n in range(2, 13):
        assert dag.simulate(DESCENDING, n, CAUSAL, 2, n, c, r) == (n + 1) * (c + r) + (n - 1) * r


def test_descending_full_equals_naive():
    for n in range(2, 10):
        for m in range(1, 5):
            for c, r in CR:
                assert dag.simulate(DESCENDING, n, FULL, m, n, c, r) == dag.simulate(NAIVE, n, FULL, m, n, c, r)


# --- worked examples ----------------------------------------------------------

def test_fig2_two_tiles_naive_full():
    """Fig. 2: n = 2 KV tiles, 2 Q tiles, one head: makespan 2c + 3r."""
    for c, r in CR:
        assert dag.simulate(NAIVE, 2, FULL, 1, 2, c, r) == 2 * c + 3 * r


def _read_fig4():
    rows, makespan = {}, None
    with open(os.path.join(GOLDEN, "fig4_descending_causal.txt")) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("makespan"):
                makespan = int(line.split()[1])
                continue
            sm, rest = line.split(":")
            rows[int(sm[2:])] = [tuple(int(x) for x in tok.split(".")) for tok in rest.split()]
    return makespan, rows


def test_fig4_descending_causal_gantt():
    """Fig. 4: n = 4, m = 2, descending, causal, c = r = 1."""
    makespan, rows = _read_fig4()
    t, assignment, records = dag.simulate(DESCENDING, 4, CAUSAL, 2, 4, 1, 1, trace=True)
    assert t == makespan == 13
    for sm, expected in rows.items():
        got = [(hd, i, j) for hd, i, j, _, _ in records[sm]]
        assert got == expected, (sm, got, expected)
    # the second head's jobs land in "snake" order: SM3 takes KV0, ..., SM0 takes KV3
    head2 = [(s, ji) for s, hd, ji in assignment if hd == 1]
    assert head2 == [(3, 0), (2, 1), (1, 2), (0, 3)]
    # SM0 reduces r3 at once, SM3 waits three slots
    assert records[0][0][4] == 1 and records[3][0][4] == 4


# --- Lemma 1 -------------------------------------------------------------------

def test_lemma1_brute_force():
    """Adding zero-weight edges keeps the critical path iff every edge is
    depth-monotone (Lemma 1; proof App. B)."""
    rnd = random.Random(1234)
    checked = 0
    for _ in range(1500):
        n_chains = rnd.randint(1, 4)
        length = rnd.randint(1, 5)
        weights = [rnd.randint(1, 5) for _ in range(length)]  # isomorphic chains
        # node 0 = source, 1 = sink, chain c node at depth k (k = 1..length)
        def node(ch, k):
            return 2 + ch * length + (k - 1)
        n_nodes = 2 + n_chains * length
        edges = []
        for ch in range(n_chains):
            edges.append((0, node(ch, 1), weights[0]))
            for k in range(1, length):
                edges.append((node(ch, k), node(ch, k + 1), weights[k]))
            edges.append((node(ch, length), 1, 1))
        base = dag.longest_path(n_nodes, edges, 0, 1)
        added, monotone = [], True
        for _ in range(rnd.randint(1, 4)):
            c1, c2 = rnd.randrange(n_chains), rnd.randrange(n_chains)
            k1, k2 = rnd.randint(1, length), rnd.randint(1, length)
            if c1 == c2:
                continue
            trial = edges + added + [(node(c1, k1), node(c2, k2), 0)]
            try:
                dag.longest_path(n_nodes, trial, 0, 1)
            except ValueError:
                continue  # the lemma's premise: every G_i stays a DAG
            added.append((node(c1, k1), node(c2, k2), 0))
            monotone &= k1 <= k2
        if not added:
            continue
        cp = dag.longest_path(n_nodes, edges + added, 0, 1)
        assert (cp == base) == monotone
        checked += 1
    assert checked > 500


def test_longest_path_detects_cycle():
    with pytest.raises(ValueError):
        dag.longest_path(3, [(0, 1, 1), (1, 2, 1), (2, 1, 0)], 0, 2)


# --- structural properties -------------------------------------------------------

@pytest.mark.parametrize("schedule", [NAIVE, DESCENDING, SHIFT])
@pytest.mark.parametrize("mask", [FULL, CAUSAL])
def test_schedule_structure(schedule, mask):
    for n in range(1, 33):
        jobs = dag.build_jobs(schedule, n, mask)
        rank = dag.reduction_ranks(schedule, n, mask)
        tasks = [t for job in jobs for t in job.tasks]
        expect = {(i, j) for i in range(n) for j in range(n) if mask == FULL or j >= i}
        assert sorted(tasks) == sorted(expect)  # coverage, each task exactly once
        for job in jobs:  # per-KV contiguity
            kvs = [i for i, _ in job.tasks]
            seen = []
            for i in kvs:
                if not seen or seen[-1] != i:
                    assert i not in seen
                    seen.append(i)
        for j in range(n):  # rank permutation per Q tile
            rs = sorted(rank[(i, jj)] for (i, jj) in expect if jj == j)
            assert rs == list(range(len(rs)))
        if schedule == SHIFT:
            def steps_of(job):
                return job.steps if job.steps is not None else list(range(len(job.tasks)))
            odd = mask == CAUSAL and n % 2
            if not odd:
                steps = max(len(job.tasks) for job in jobs)
                assert all(len(job.tasks) == steps for job in jobs)  # balanced chains
                if mask == CAUSAL:
                    assert steps == n + 1  # n + 1 tasks per symmetric pair
            else:  # AMB-29: the n + 1 schedule minus the phantom tile's tasks
                assert len(jobs) == (n + 1) // 2
                assert all(steps_of(job) == sorted(steps_of(job)) for job in jobs)
            by_t = {}
            for job in jobs:
                for t, (i, j) in zip(steps_of(job), job.tasks):
                    by_t.setdefault(t, []).append(j)
            for js in by_t.values():  # conflict-free: distinct Q tiles per step
                assert len(set(js)) == len(js)
            for j in range(n):  # ranks strictly increase with the visit step
                by_step = sorted((t, rank[(i, jj)]) for job in jobs
                                 for t, (i, jj) in zip(steps_of(job), job.tasks) if jj == j)
                assert [rk for _, rk in by_step] == list(range(len(by_step)))
        else:
            for (i, j), rk in rank.items():
                assert rk == i  # ascending-KV order (AMB-6)


def test_shift_zero_bubbles_single_head():
    """With its jobs co-resident, a shift head has no pipeline bubble:
    every R starts exactly when its own C ends (§3.4)."""
    for n in range(2, 17):
        for mask in (FULL, CAUSAL):
            if mask == CAUSAL and n % 2:
                continue
            _, _, records = dag.simulate(SHIFT, n, mask, 1, n, 3, 2, trace=True)
            for recs in records:
                for _, _, _, c_start, r_start in recs:
                    assert r_start == c_start + 3


def test_coresidency_deadlock_bound():
    """SHIFT needs all jobs of a head resident; NAIVE/DESCENDING never deadlock."""
    with pytest.raises(dag.Deadlock):
        dag.simulate(SHIFT, 8, FULL, 2, 7)
    dag.simulate(SHIFT, 8, FULL, 2, 8)
    with pytest.raises(dag.Deadlock):
        dag.simulate(SHIFT, 8, CAUSAL, 2, 3)
    dag.simulate(SHIFT, 8, CAUSAL, 2, 4)
    for s in (NAIVE, DESCENDING):
        for mask in (FULL, CAUSAL):
            dag.simulate(s, 8, mask, 3, 3)
            dag.simulate(s, 8, mask, 3, 1)


def test_default_params_separate_the_schedules():
    """m = 2, n_sm = n, c = r = 1 gives NAIVE 5n-1,
    DESCENDING-causal 3n+1, SHIFT-full 4n, SHIFT-causal 2n+2."""
    for n in range(2, 40, 2):
        assert dag.simulate(NAIVE, n, CAUSAL) == 5 * n - 1
        assert dag.simulate(DESCENDING, n, CAUSAL) == 3 * n + 1
        assert dag.simulate(SHIFT, n, FULL) == 4 * n
        assert dag.simulate(SHIFT, n, CAUSAL) == 2 * n + 2


def test_grouped_shift_full_beyond_group_size():
    """AMB-30: SHIFT with the full mask and more than SHIFT_GROUP KV tiles runs in
    near-equal groups; inside a group the cyclic shift is conflict-free and each
    dQ_j is reduced group-major, in visit-step order inside a group."""
    for n in (129, 200, 257):
        jobs = dag.build_jobs(SHIFT, n, FULL)
        rank = dag.reduction_ranks(SHIFT, n, FULL)
        G = -(-n // dag.SHIFT_GROUP)
        sizes = {}
        for job in jobs:
            g = job.steps[0][0]
            sizes[g] = sizes.get(g, 0) + 1
            assert len(job.tasks) == n
        assert len(sizes) == G and max(sizes.values()) <= dag.SHIFT_GROUP
        assert max(sizes.values()) - min(sizes.values()) <= 1
        by_label = {}
        for job in jobs:
            for lab, (i, j) in zip(job.steps, job.tasks):
                by_label.setdefault(lab, []).append(j)
        assert all(len(set(js)) == len(js) for js in by_label.values())  # conflict-free
        for j in (0, 1, n // 2, n - 1):
            order = sorted((lab, i) for job in jobs for lab, (i, jj) in zip(job.steps, job.tasks)
                           if jj == j)
            assert [rank[(i, j)] for _, i in order] == list(range(n))
        # the model finishes with one group's worth of SMs (co-residency of a group)
        assert dag.simulate(SHIFT, n, FULL, 1, max(sizes.values()), 2, 1) > 0


@pytest.mark.parametrize("n", [258, 301, 400])
def test_grouped_symmetric_shift_beyond_group_size(n):
    """AMB-35: causal SHIFT with more than SHIFT_GROUP pairs keeps the paper's
    jobs (pair p = KV p then KV n-1-p) and reduces each dQ_j
    group-major, in visit-step order inside a group: every causal task exactly
    once, conflict-free steps inside a group, each dQ_j's ranks 0..j with all
    of group g's contributions before group g+1's, and the DAG model finishes
    on one group's worth of SMs (co-residency of a group, not of all pairs)."""
    jobs = dag.build_jobs(SHIFT, n, CAUSAL)
    rank = dag.reduction_ranks(SHIFT, n, CAUSAL)
    h = (n + 1) // 2
    G = -(-h // dag.SHIFT_GROUP)
    assert G >= 2 and len(jobs) == h
    seen = [(i, j) for job in jobs for (i, j) in job.tasks]
    assert sorted(seen) == [(i, j) for i in range(n) for j in range(i, n)]
    sizes = {}
    for job in jobs:
        sizes[job.steps[0][0]] = sizes.get(job.steps[0][0], 0) + 1
    assert len(sizes) == G and max(sizes.values()) <= dag.SHIFT_GROUP
    assert max(sizes.values()) - min(sizes.values()) <= 1
    by_label = {}
    for job in jobs:
        for lab, (i, j) in zip(job.steps, job.tasks):
            by_label.setdefault(lab, []).append(j)
    assert all(len(set(js)) == len(js) for js in by_label.values())
    for j in (0, 1, h - 1, h, n // 2 + 3, n - 2, n - 1):
        contrib = sorted((rank[(i, j)], lab[0], lab) for job in jobs
                         for lab, (i, jj) in zip(job.steps, job.tasks) if jj == j)
        assert [r for r, _, _ in contrib] == list(range(j + 1))
        groups = [g for _, g, _ in contrib]
        assert groups == sorted(groups)                 # group-major
        assert [lab for _, _, lab in contrib] == sorted(lab for _, _, lab in contrib)
    assert dag.simulate(SHIFT, n, CAUSAL, 1, max(sizes.values()), 2, 1) > 0
