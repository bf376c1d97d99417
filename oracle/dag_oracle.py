"""oracle/dag_oracle.py -- TEST INFRASTRUCTURE ONLY.

Brute-force integer model of the paper's deterministic-backward DAG (§3,
PAPER.md P:71-141) and the three schedules, written from the paper's own
definitions.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  It shares no
code with the product (libdash.so's C++ schedule generator and simulator are
written separately) and imports nothing from the product package.

Notation (§3, Fig. 2): i = KV tile ("column"), j = Q tile ("row"),
n = n_q = n_kv tiles per head (§3 intro P:67, AMB-11), m = heads,
c = compute-phase cost, r = reduction-phase cost.

What is followed, step by step:
  * Task (i, j) exists iff the mask is full or j >= i (causal).
  * Each task is a chain C(i,j) -> R(i,j) of weights c, r (§3.1).
  * All tasks of one KV tile run contiguously on one SM (§3.1 "Optimization
    Constraint"); SHIFT-causal runs a *pair* of KV tiles on one SM
    (§3.4, AMB-10), each KV tile still contiguous.
  * dQ_j is reduced in a prescribed global order; a zero-weight edge runs
    from the end of R of rank k-1 to the start of R of rank k.
  * Greedy list scheduling (AMB-7): jobs listed head-major, KV-ascending;
    whenever an SM is free the lowest-indexed free SM claims the next job.
  * The R phase occupies its SM (the Gantt rows of Figs 2/3/4, AMB-24).
  * The critical path is the makespan (§3.1 "scheduling objective").

Schedule definitions:
  NAIVE:  job i visits j = i0, i0+1, .., n-1
  DESCENDING  (Fig.4): job i visits j = n-1, .., i0
  SHIFT full  (Fig.6):   job i visits j = (i+t) mod n (AMB-5: Q tiles)
  SHIFT causal (Fig.7): pair p = (p, n-1-p), two phases
  with i0 = 0 (full) or i (causal).  Reduction order (the "global order",
  Alg.1 line 33 P:395): NAIVE and DESCENDING keep ascending KV order (AMB-6);
  SHIFT orders each dQ_j's contributions by the step at which they are
  computed ("distinct timestamps ... induce a natural, conflict-free
  reduction sequence", Fig.6 caption P:119).

Pins (tests/test_oracle_dag.py): the closed forms of P:87, P:89, P:103,
P:141; Fig.2 and Fig.4 (tests/golden/fig4_descending_causal.txt);
Lemma 1 by brute force; the structural statements of P:77,
P:127-133; the co-residency deadlock bound.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

NAIVE, DESCENDING, SHIFT = 0, 1, 2
FULL, CAUSAL = 0, 1


class Deadlock(RuntimeError):
    """The simulated schedule cannot finish (a rank predecessor never runs)."""


@dataclass
class Job:
    """One SM's contiguous work: an ordered list of (kv, q) tasks."""
    tasks: list = field(default_factory=list)  # [(i, j)], in execution order
    # Visit step of each task in the schedule's own step numbering; None = the
    # position in `tasks`.  Differs only for odd-n Symmetric Shift (AMB-29),
    # whose jobs are the n+1 schedule with the phantom tile's tasks removed.
    steps: list | None = None


SHIFT_GROUP = 128  # AMB-30 / AMB-35: largest group of KV tiles (full) / pairs (causal) in one shift


def task_exists(i: int, j: int, mask: int) -> bool:
    return mask == FULL or j >= i


def build_jobs(schedule: int, n: int, mask: int) -> list[Job]:
    """The per-head job list, in claim order (KV ascending; pairs for SHIFT-causal)."""
    jobs: list[Job] = []
    if schedule == NAIVE:
        for i in range(n):
            jobs.append(Job([(i, j) for j in range(n) if task_exists(i, j, mask)]))
    elif schedule == DESCENDING:
        for i in range(n):
            jobs.append(Job([(i, j) for j in reversed(range(n)) if task_exists(i, j, mask)]))
    elif schedule == SHIFT and mask == FULL:
        # SM_i visits Q tiles i, i+1, ..., n-1, 0, ..., i-1 (AMB-5).
        # AMB-30: more than SHIFT_GROUP KV tiles -> G = ceil(n / SHIFT_GROUP)
        # consecutive near-equal groups; dQ_j takes group 0's contributions
        # first, then group 1's, ..., each group in visit-step order.  The step
        # label (group, t) carries that order.
        G = -(-n // SHIFT_GROUP)
        for g in range(G):
            for i in range(g * n // G, (g + 1) * n // G):
                tasks = [(i, (i + t) % n) for t in range(n)]
                jobs.append(Job(tasks, [(g, t) for t in range(n)] if G > 1 else None))
    elif schedule == SHIFT and mask == CAUSAL and n % 2:
        # AMB-29: odd n = the Symmetric Shift of n + 1 tiles (even) without the
        # phantom KV tile n and the phantom Q tile n: every real task keeps the
        # visit step it has there, so each dQ_j keeps its step order.
        for job in build_jobs(SHIFT, n + 1, CAUSAL):
            steps = job.steps if job.steps is not None else range(len(job.tasks))
            kept = [(t, (i, j)) for t, (i, j) in zip(steps, job.tasks) if i < n and j < n]
            jobs.append(Job([ij for _, ij in kept], [t for t, _ in kept]))
    elif schedule == SHIFT and mask == CAUSAL:
        h = n // 2
        # AMB-35: more than SHIFT_GROUP pairs -> G = ceil(h / SHIFT_GROUP)
        # consecutive near-equal groups of pairs; the jobs are unchanged, dQ_j
        # takes group 0's contributions first, then group 1's, ..., each group
        # in visit-step order: the step label (group, t) carries that order.
        G = -(-h // SHIFT_GROUP)
        for p in range(h):
            tasks = []
            # Phase 1: cyclic shift over the dense lower-left rectangle,
            # Q rows [h, n) x KV cols [0, h).
            for t in range(h):
                tasks.append((p, h + (p + t) % h))
            # Phase 2, left (upper) triangle: column p, top-down from the diagonal.
            for j in range(p, h):
                tasks.append((p, j))
            # Phase 2, right (lower) triangle: column n-1-p, bottom-up to the diagonal.
            for j in range(n - 1, n - 2 - p, -1):
                tasks.append((n - 1 - p, j))
            g = next(g for g in range(G) if g * h // G <= p < (g + 1) * h // G)
            jobs.append(Job(tasks, [(g, t) for t in range(len(tasks))] if G > 1 else None))
    else:
        raise ValueError(f"unknown schedule {schedule}")
    return jobs


def reduction_ranks(schedule: int, n: int, mask: int) -> dict:
    """rank[(i, j)] = position of KV tile i's contribution in dQ_j's global order."""
    jobs = build_jobs(schedule, n, mask)
    contrib: dict[int, list] = {j: [] for j in range(n)}
    for job in jobs:
        steps = job.steps if job.steps is not None else range(len(job.tasks))
        for step, (i, j) in zip(steps, job.tasks):
            # NAIVE / DESCENDING: ascending KV order (AMB-6).
            # SHIFT: order of the visit step (Fig. 6 caption P:119).
            key = i if schedule in (NAIVE, DESCENDING) else step
            contrib[j].append((key, i))
    rank = {}
    for j, lst in contrib.items():
        keys = [k for k, _ in lst]
        if len(set(keys)) != len(keys):
            raise AssertionError(f"reduction order of dQ_{j} is not a strict order")
        for pos, (_, i) in enumerate(sorted(lst)):
            rank[(i, j)] = pos
    return rank


def simulate(schedule: int, n: int, mask: int, m: int = 2, n_sm: int | None = None,
             c: int = 1, r: int = 1, trace: bool = False):
    """Event simulation of the greedy multi-head execution; returns the makespan.

    With trace=True returns (makespan, assignment) where assignment is a list
    of (sm, head, job_index) in claim order and a per-SM list of
    (head, i, j, c_start, r_start) task records.
    """
    if n_sm is None:
        n_sm = n
    if c < 1 or r < 1:
        raise ValueError("phase weights must be positive (Lemma 1 premise, P:123)")
    jobs = build_jobs(schedule, n, mask)
    rank = reduction_ranks(schedule, n, mask)
    queue = [(hd, ji) for hd in range(m) for ji in range(len(jobs))]  # head-major (AMB-7)
    qpos = 0
    # done[(head, j, k)] = end time of the R phase of rank k on dQ_j of head.
    done: dict = {}
    waiting: dict = {}  # (head, j, k) -> (sm, c_end)
    state = [None] * n_sm  # per SM: [head, job_index, task_pos]
    events: list = []  # (time, kind, sm); kind 0 = C done, 1 = R done, 2 = idle
    for s in range(n_sm):
        heapq.heappush(events, (0, 2, s))
    assignment = []
    records = [[] for _ in range(n_sm)]
    makespan = 0

    def start_r(s, c_end, pred_end):
        hd, ji, pos = state[s]
        i, j = jobs[ji].tasks[pos]
        r_start = max(c_end, pred_end)
        r_end = r_start + r
        key = (hd, j, rank[(i, j)])
        done[key] = r_end
        if trace:
            records[s].append((hd, i, j, c_end - c, r_start))
        if key in waiting:  # the rank k+1 contributor waits on this one
            s2, c_end2 = waiting.pop(key)
            start_r(s2, c_end2, r_end)
        heapq.heappush(events, (r_end, 1, s))

    while events:
        t, kind, s = heapq.heappop(events)
        makespan = max(makespan, t)
        if kind == 2:  # idle: claim the next job
            if qpos == len(queue):
                state[s] = None
                continue
            hd, ji = queue[qpos]
            qpos += 1
            state[s] = [hd, ji, 0]
            assignment.append((s, hd, ji))
            heapq.heappush(events, (t + c, 0, s))
        elif kind == 0:  # C done
            hd, ji, pos = state[s]
            i, j = jobs[ji].tasks[pos]
            k = rank[(i, j)]
            if k == 0:
                start_r(s, t, t)
            elif (hd, j, k - 1) in done:
                start_r(s, t, done[(hd, j, k - 1)])
            else:
                waiting[(hd, j, k - 1)] = (s, t)
        else:  # R done
            hd, ji, pos = state[s]
            if pos + 1 < len(jobs[ji].tasks):
                state[s][2] = pos + 1
                heapq.heappush(events, (t + c, 0, s))
            else:
                heapq.heappush(events, (t, 2, s))
    if qpos != len(queue) or waiting or any(st is not None for st in state):
        raise Deadlock(f"schedule {schedule} n={n} mask={mask} m={m} n_sm={n_sm}")
    if trace:
        return makespan, assignment, records
    return makespan


# ---------------------------------------------------------------------------
# Lemma 1 material: a generic DAG longest path, used by the
# brute-force property test on random isomorphic-chain graphs.
# ---------------------------------------------------------------------------

def longest_path(n_nodes: int, edges: list, source: int, sink: int) -> int:
    """Longest source->sink path length of a DAG given as (u, v, w) edges.

    Raises ValueError on a cycle.  Plain Kahn topological order + relaxation.
    """
    adj = [[] for _ in range(n_nodes)]
    indeg = [0] * n_nodes
    for u, v, w in edges:
        adj[u].append((v, w))
        indeg[v] += 1
    order = [x for x in range(n_nodes) if indeg[x] == 0]
    seen = 0
    dist = [None] * n_nodes
    dist[source] = 0
    head = 0
    while head < len(order):
        u = order[head]
        head += 1
        seen += 1
        for v, w in adj[u]:
            if dist[u] is not None and (dist[v] is None or dist[u] + w > dist[v]):
                dist[v] = dist[u] + w
            indeg[v] -= 1
            if indeg[v] == 0:
                order.append(v)
    if seen != n_nodes:
        raise ValueError("graph has a cycle")
    return dist[sink]
