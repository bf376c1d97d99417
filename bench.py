#!/usr/bin/env python
"""Benchmark of the DASH deterministic attention backward on B200.

Workload (BASELINE.json configs[1], the metric's configuration): the FA3-style
sweep of PAPER.md §4.1 -- 16,384 total tokens, hidden 2,048, head dim
128, seqlen 512 .. 16,384 (B = 16384 / N, H = 16), causal mask, bf16 random
inputs.  One "step" = one dash_attn_bwd (preprocess + main + dQ convert) at
every sweep point, with the library's per-shape DASH schedule (`auto`:
Symmetric Shift up to 32 tiles, Descending above -- measured, see the
`sweep` key; the paper preferred Descending at causal HD128 on H800 because
Symmetric Shift spilled registers, which TMEM removes on B200).

value     = sweep FLOPs / device time, FLOPs by the FlashAttention convention
            (bwd = 2.5 x fwd = 10 B H N^2 d, causal halved; DESIGN.md AMB-17).
e2e       = the same metric through dash_attn_bwd_host with pinned host
            buffers (H2D of q, k, v, o, dO, lse and D2H of dq, dk, dv inside
            the timed region).
roofline  = the main kernel's algorithmic tile FLOPs (5 GEMMs of 2*128*128*d
            per (KV tile, Q tile) task) / its CUDA-event
            time, against MEASURED_PEAKS.json bf16_tflops.
sweep     = per-seqlen TFLOP/s of NAIVE / DESCENDING / SHIFT (deterministic)
            and the atomic variant, with the gap-closure ratio (AMB-19).
gate      = the north_star target per swept shape for configs 2 and 3
            (causal HD128, full HD128, full HD64, causal HD64): the best of
            DESCENDING / SHIFT against NAIVE at the SAME number W of
            interleaved accumulators (AMB-27) -- the primary reading -- and
            at W = 1 (the paper's single accumulator) beside it.

Multi-GPU (`--gpus N`; launched under torchrun, or re-executes itself under
torch.distributed.run when started bare): strong scaling by default -- the
fixed sweep problem is split over the U = B*H flattened (b, h) units, rank r
owning the contiguous range [r*U/N, (r+1)*U/N); no collective
on the data path; value = the whole problem's FLOPs / max-over-ranks device
time.  After timing, per-unit SHA-256 digests of dq/dk/dv are all-gathered
(NCCL) and rank 0 checks them against its own 1-GPU run of the whole problem
(`sharding_bitwise_identical`).  `--scaling weak` instead gives every rank a
full problem of its own (per-rank seeds).

--impl reference times the fp64 CPU oracle (oracle/, the correctness
reference; there is no runnable upstream implementation) on a bounded sample
of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEQLENS = (512, 1024, 2048, 4096, 8192, 16384)
TOKENS, HIDDEN = 16384, 2048
METRIC = "deterministic attn-bwd TFLOPs/s vs atomic bwd; % of B200 BF16 tensor peak"
CPU_SAMPLE_N = 2048  # sweep point used for the oracle's bounded sample
SWEEP_ROUNDS = 3     # interleaved timing rounds of the per-schedule table (median)


def fa_flops(B, N, H, d, causal):
    f = 10.0 * B * H * N * N * d
    return f / 2 if causal else f


def tile_flops(B, N, H, d, causal):
    n = N // 128
    tasks = n * (n + 1) // 2 if causal else n * n
    return 5 * 2.0 * 128 * 128 * d * tasks * B * H


def shapes(head_dim, seqlens=SEQLENS):
    return [(TOKENS // N, N, HIDDEN // head_dim, head_dim) for N in seqlens]


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.samples.append((time.time(), parts))

    def mark(self, which):
        setattr(self, which, time.time())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        t0, t1 = getattr(self, "t0", 0.0), getattr(self, "t1", float("inf"))
        inside = [p for t, p in self.samples if t0 <= t <= t1 + 0.05]
        window = "timed region"
        if not inside and self.samples:  # region shorter than the sampling period
            mid = 0.5 * (t0 + t1)
            inside = [min(self.samples, key=lambda tp: abs(tp[0] - mid))[1]]
            window = "nearest sample to the timed region"
        if not inside:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        samples = inside
        sm = [float(s[0]) for s in samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in samples for i in range(4)
                          if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(samples), "window": window}


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:  # CPU tests of the plumbing (gloo)
            dist.init_process_group("gloo")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def relaunch_if_needed(args):
    """`--gpus N` (N > 1) without a torchrun environment: re-execute this
    command under torch.distributed.run with N ranks on 127.0.0.1; under
    torchrun, the world size must equal N."""
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    if world is not None and int(world) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    import torch
    if world == 1:
        return x
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def shard_inputs(cpu, world, rank, scaling):
    """Rank's inputs: strong scaling -> its flattened (b, h) units of the
    shared problem (paper_2601_21824_b200.dist.shard_units); weak -> all of it."""
    if scaling == "weak" or world == 1:
        return dict(cpu)
    from paper_2601_21824_b200 import dist as ddist
    return {k: ddist.shard_units(v, world, rank) for k, v in cpu.items()}


def make_problem(B, N, H, d, causal, rank, world, scaling, dash, torch):
    from paper_2601_21824_b200.inputs import attn_inputs
    # strong: every rank draws the same problem (seed N) and keeps its units;
    # weak: rank r draws its own full problem (seed 1000 r + N).
    seed = N if scaling == "strong" else 1000 * rank + N
    cpu = shard_inputs(attn_inputs(B, N, H, d, seed=seed), world, rank, scaling)
    g = {k: v.cuda() for k, v in cpu.items()}
    o, lse = dash.attn_fwd(g["q"], g["k"], g["v"], causal)
    g["o"], g["lse"] = o, lse
    g["out"] = (torch.empty_like(g["q"]), torch.empty_like(g["k"]), torch.empty_like(g["v"]))
    g["ws"] = dash.alloc_workspace(g["q"].shape, causal)
    g["shape"] = tuple(g["q"].shape)
    return g


def verify_sharding(world, rank, full_shapes, run_shard, run_full):
    """Sharding check of SURVEY §8(e): per-unit SHA-256 digests of every
    rank's outputs (run_shard(i) -> (dq, dk, dv) of its units of problem i),
    all-gathered, must equal the digests of rank 0's run of the whole problem
    (run_full(shape) -> (dq, dk, dv)).  Returns the verdict on rank 0, None
    elsewhere.  bench.py passes GPU calls; tests/test_dist_gloo.py the oracle."""
    import torch.distributed as dist
    from paper_2601_21824_b200 import dist as ddist
    ok = True
    for i, shape in enumerate(full_shapes):
        mine = [ddist.per_unit_digests(t) for t in run_shard(i)]
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        if rank == 0:
            got = [sum((allv[r][t] for r in range(world)), []) for t in range(3)]
            want = [ddist.per_unit_digests(t) for t in run_full(shape)]
            ok = ok and got == want
    return ok if rank == 0 else None


def gpu_sharding_check(dash, torch, world, rank, probs, full_shapes, causal, schedule):
    from paper_2601_21824_b200.inputs import attn_inputs

    def run_shard(i):
        out = run_bwd(dash, probs[i][1], causal, schedule, True)
        torch.cuda.synchronize()
        return out

    def run_full(shape):
        B, N, H, d = shape
        full = {k: v.cuda() for k, v in attn_inputs(B, N, H, d, seed=N).items()}
        fo, fl = dash.attn_fwd(full["q"], full["k"], full["v"], causal)
        out = dash.attn_bwd(full["q"], full["k"], full["v"], fo, full["do"], fl, causal,
                            schedule, True)
        torch.cuda.synchronize()
        return out

    return verify_sharding(world, rank, full_shapes, run_shard, run_full)


def run_bwd(dash, g, causal, schedule, det):
    return dash.attn_bwd(g["q"], g["k"], g["v"], g["o"], g["do"], g["lse"], causal, schedule,
                         det, workspace=g["ws"], out=g["out"])


def time_steps(torch, fn, steps, warmup, world, before=None, after=None):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    if before:
        before()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    if after:
        after()
    barrier(world)
    return e0.elapsed_time(e1)  # ms


def cpu_oracle_sample(head_dim, causal, heads=None):
    """The fp64 oracle on a bounded sample: `heads` heads of the N = 2048 sweep point."""
    import oracle
    from paper_2601_21824_b200.inputs import attn_inputs
    cores = len(os.sched_getaffinity(0))
    oracle.build()
    oracle.set_threads(cores)
    if heads is None:
        heads = 2 * cores
    B, N, H, d = TOKENS // CPU_SAMPLE_N, CPU_SAMPLE_N, HIDDEN // head_dim, head_dim
    heads = min(heads, B * H)
    nb = max(1, heads // H)
    nh = min(H, heads)
    x = attn_inputs(nb, N, nh, d, seed=0)
    f = {k: v.double().numpy() for k, v in x.items()}
    t = time.time()
    oracle.attn_bwd(f["q"], f["k"], f["v"], f["do"], causal)
    dt = time.time() - t
    fl = fa_flops(nb, N, nh, d, causal)
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": oracle.max_threads(),
            "kind": "oracle", "seconds": dt,
            "sample": f"fp64 oracle backward (C, OpenMP over heads) on {nb * nh} of the {B * H} "
                      f"(b,h) heads of the N={N} sweep point (B={B}, H={H}, d={d}, "
                      f"{'causal' if causal else 'full'}), FLOPs by the FA convention"}


def oracle_timing(out_path):
    """The CPU baseline beside the GPU: the fp64 oracle as it
    stands on this host -- config 1 single-thread and all-core, one bounded sample
    of the N = 512 / 2048 sweep shapes per mask (scaled to the full shape), one
    head of N = 4096 for the long-context config (extrapolated, labelled)."""
    import platform
    import oracle
    from paper_2601_21824_b200.inputs import attn_inputs
    oracle.build()
    cores = len(os.sched_getaffinity(0))
    cpu = platform.machine()
    try:
        with open("/proc/cpuinfo") as fh:
            cpu = next(l.split(":", 1)[1].strip() for l in fh if l.startswith("model name"))
    except (OSError, StopIteration):
        pass

    def run(B, N, H, d, causal, threads):
        oracle.set_threads(threads)
        x = attn_inputs(B, N, H, d, seed=0)
        f = {k: v.double().numpy() for k, v in x.items()}
        t = time.time()
        oracle.attn_bwd(f["q"], f["k"], f["v"], f["do"], causal)
        dt = time.time() - t
        return dt, fa_flops(B, N, H, d, causal) / dt / 1e12

    res = {"cpu_model": cpu, "cores": cores, "rows": []}
    for causal in (True, False):
        for threads in (1, cores):
            dt, tf = run(1, 256, 1, 64, causal, threads)
            res["rows"].append({"config": "1 (B=1,H=1,N=256,d=64)", "causal": causal,
                                "threads": threads, "seconds": dt, "tflops": tf})
    for N, heads in ((512, 4 * cores), (2048, cores)):
        for causal in (True, False):
            dt, tf = run(1, N, heads, 128, causal, cores)
            B, H = TOKENS // N, HIDDEN // 128
            res["rows"].append({"config": f"sweep N={N} d=128 ({heads} of {B * H} heads)",
                                "causal": causal, "threads": cores, "seconds": dt, "tflops": tf,
                                "extrapolated_full_shape_seconds": dt * B * H / heads})
    dt, tf = run(1, 4096, 1, 128, True, cores)  # one head runs on one thread
    res["rows"].append({"config": "4 long context (B=8,H=32,N=32768,d=128 causal), from one head of N=4096",
                        "causal": True, "threads": 1, "seconds": dt, "tflops": tf,
                        "extrapolated_full_config_seconds": dt * 64 * 256 / cores,
                        "note": "extrapolated: x64 (N^2) x 256 heads / cores threads; not measured"})
    with open(out_path, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res), flush=True)


def load_peaks():
    """(burst peak, source, sustained peak or None).  The burst figure is the
    denominator (the timed region is ~0.1 s at full clocks); the sustained one
    (seconds-long cuBLAS loop under the power cap) is reported beside it."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        sus = j.get("bf16_tflops_sustained")
        return (float(j["bf16_tflops"]), "measured burst (MEASURED_PEAKS.json bf16_tflops)",
                float(sus) if sus else None)
    return 1590.0, "fallback (B200_PROFILING.md)", 1400.0


def load_traffic(workload):
    """Per-launch DRAM bytes of the main kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_main_kernel.json")
    if not os.path.exists(p):
        return None
    try:
        with open(p) as f:
            j = json.load(f)
        return j.get(workload, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def bench_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    causal = not args.full
    cores = len(os.sched_getaffinity(0))
    for _ in range(args.warmup):
        cpu_oracle_sample(args.head_dim, causal, heads=cores)
    vals, secs = [], 0.0
    for _ in range(args.steps):
        r = cpu_oracle_sample(args.head_dim, causal, heads=cores)
        vals.append(r["value"])
        secs += r["seconds"]
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * secs / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, world),
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": r["cores"], "kind": "oracle",
                         "sample": r["sample"]},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def workload_config(args, world):
    causal = not args.full
    name = (f"fa3-sweep-{'causal' if causal else 'full'}-hd{args.head_dim}"
            f"-{TOKENS}tok-hidden{HIDDEN}")
    return {"workload": name, "seqlens": list(SEQLENS), "total_tokens": TOKENS,
            "hidden": HIDDEN, "head_dim": args.head_dim, "mask": "causal" if causal else "full",
            "schedule": args.schedule, "acc_split": args.acc_split,
            "batch_x_heads": [list(s[::2]) for s in shapes(args.head_dim)],
            "parallelism": f"bh-units x{world} ({args.scaling})",
            "l2": "inputs > L2 (5 x 64 MiB per sweep point, 126 MB L2)"}


def gap_gate(naive, best, atomic):
    """AMB-19: (gap closed, pass) of `best` over `naive` towards `atomic`."""
    gap = atomic - naive
    if gap < 0.02 * atomic:  # no gap (or NAIVE at / above atomic): stay within 2 %
        return None, best >= 0.98 * naive
    closed = (best - naive) / gap
    return closed, closed >= 0.5


def sweep_rows(dash, torch, probs, causal, steps):
    """Per sweep point: NAIVE / DESCENDING / SHIFT (deterministic) and the
    atomic variant at the library's W, and the three schedules at W = 1;
    SWEEP_ROUNDS interleaved rounds, median per case.  The north_star gate is
    evaluated at the SAME W on both sides (primary) and at W = 1."""
    rows = []
    w_bench = dash.acc_split()
    for s, g in probs:
        row = {"seqlen": s[1], "batch": s[0], "heads": s[2],
               "acc_split": dash.acc_split(s, causal, "auto"), "tile": dash.tile(s, causal, "auto"),
               "auto": dash.resolve_schedule(s, causal, "auto")}
        f = fa_flops(*s, causal)
        cases = [("naive", "naive", True, w_bench), ("descending", "descending", True, w_bench),
                 ("shift", "shift", True, w_bench), ("atomic", "naive", False, w_bench)]
        if dash.acc_split(s, causal, "auto") != 1:
            cases += [("naive_w1", "naive", True, 1), ("descending_w1", "descending", True, 1),
                      ("shift_w1", "shift", True, 1)]
        # Round-robin over the cases, median per case: every schedule sees
        # the same clock / power history.
        times = {name: [] for name, *_ in cases}
        nst = max(3, steps)
        for _ in range(SWEEP_ROUNDS):
            for name, sched, det, w in cases:
                if row.get(name + "_error"):
                    continue
                dash.set_acc_split(w)
                try:
                    times[name].append(time_steps(
                        torch, lambda: run_bwd(dash, g, causal, sched, det), nst, 2, 1))
                except dash.DashError as e:
                    row[name + "_error"] = str(e)
        dash.set_acc_split(w_bench)
        for name, *_ in cases:
            row[name] = (f * nst / (statistics.median(times[name]) / 1e3) / 1e12
                         if times[name] and not row.get(name + "_error") else None)
        row["rounds"] = SWEEP_ROUNDS
        for suffix in ("", "_w1"):
            cands = [v for v in (row.get("descending" + suffix), row.get("shift" + suffix))
                     if v is not None]
            if row.get("naive" + suffix) is None or row.get("atomic") is None or not cands:
                continue
            best = max(cands)
            row["best_dash" + suffix] = best
            row["gap_closed" + suffix], row["pass" + suffix] = gap_gate(
                row["naive" + suffix], best, row["atomic"])
        # Secondary column (mixes mechanisms): DASH at the library's W against
        # the paper's FA3-style NAIVE with one accumulator (W = 1); the
        # difference includes the interleaved accumulators of AMB-27.
        if row.get("naive_w1") is not None and row.get("best_dash") is not None:
            row["gap_closed_incl_amb27"], row["pass_incl_amb27"] = gap_gate(
                row["naive_w1"], row["best_dash"], row["atomic"])
        row["dag_model"] = dag_model_row(dash, torch, s, causal, row["tile"])
        rows.append(row)
    return rows


DAG_C, DAG_R = 3, 1  # task compute : ordered hand-off, ~8.6 k : ~3 k cycles per 256-row task


def dag_model_row(dash, torch, s, causal, tile):
    """The paper's DAG model (§3; dash_schedule_critical_path) at this
    sweep point on the units the kernel keeps co-resident (CTA pairs for
    256-row tiles, CTAs for 128-row tiles): critical path of each schedule and
    whether it predicts DESCENDING or SHIFT to beat NAIVE at all.  Where it
    does not, the same-W gate cannot pass on this device for a reason the
    paper's own model reproduces (partially co-resident heads)."""
    B, N, H, _ = s
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    units = sms // 2 if tile == 256 else sms
    n = N // tile
    mask = dash.CAUSAL if causal else dash.FULL
    cp = {}
    for name, sched in (("naive", dash.NAIVE), ("descending", dash.DESCENDING), ("shift", dash.SHIFT)):
        try:
            cp[name] = dash.schedule_critical_path(sched, n, n, mask, B * H, units, DAG_C, DAG_R)
        except dash.DashError:
            cp[name] = None
    best = min(v for k, v in cp.items() if k != "naive" and v is not None)
    return {"units": units, "n": n, "heads": B * H, "c": DAG_C, "r": DAG_R, "critical_path": cp,
            "best_over_naive": best / cp["naive"], "predicts_dash_faster": best < cp["naive"]}


def gate_summary(rows):
    return {"pass_same_w": [r.get("pass") for r in rows],
            "gap_closed_same_w": [None if r.get("gap_closed") is None else round(r["gap_closed"], 3)
                                  for r in rows],
            "pass_w1": [r.get("pass_w1") for r in rows],
            "all_pass_same_w": all(bool(r.get("pass")) for r in rows),
            "dag_model_predicts_dash_faster": [r["dag_model"]["predicts_dash_faster"] for r in rows],
            "fail_explained_by_dag_model": [bool(not r.get("pass") and
                                                 not r["dag_model"]["predicts_dash_faster"]) for r in rows],
            "seqlens": [r["seqlen"] for r in rows]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dash", choices=["dash", "reference"])
    ap.add_argument("--head-dim", type=int, default=128)
    ap.add_argument("--full", action="store_true", help="full mask instead of causal")
    ap.add_argument("--schedule", default=None,
                    help="naive | descending | shift | auto (default: auto, the library's per-shape choice)")
    ap.add_argument("--graph", action="store_true",
                    help="time the step as one CUDA graph replay (captured after warm-up)")
    ap.add_argument("--fused-dq", type=int, default=None, choices=[0, 1, 2],
                    help="dash_attn_bwd_set_fused_dq: 0 = K4 convert kernel, 1 = library policy (default), 2 = always in-kernel")
    ap.add_argument("--acc-split", type=int, default=None,
                    help="interleaved dQ accumulators W in {1,2,4,8} (AMB-27); default: the library's automatic choice")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: strong = split the fixed problem over (b, h) units (default); "
                         "weak = a full problem per rank")
    ap.add_argument("--no-sweep", action="store_true", help="skip the per-schedule sweep table")
    ap.add_argument("--no-gate", action="store_true",
                    help="skip the gate tables of the other configurations (full HD128/HD64, causal HD64)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="N > 1: skip the sharding digest check")
    ap.add_argument("--oracle-timing", default=None, metavar="OUT.json",
                    help="cpu_baseline leg only: time the fp64 oracle on config 1 "
                         "(single thread / all cores), the N = 512 and 2048 sweep shapes and "
                         "one long-context head (extrapolated), write OUT.json, exit")
    ap.add_argument("--seqlens", default=None,
                    help="comma-separated subset of the sweep (profiling only; not a bench line)")
    args = ap.parse_args()
    causal = not args.full
    if args.schedule is None:
        args.schedule = "auto"
    relaunch_if_needed(args)
    if args.impl == "reference":
        bench_reference(args)
        return
    if args.oracle_timing:
        oracle_timing(args.oracle_timing)
        return

    import torch
    world, rank, local = dist_setup(args)
    from paper_2601_21824_b200 import dash
    if args.fused_dq is not None:
        dash.set_fused_dq(args.fused_dq)
    if args.acc_split is not None:
        dash.set_acc_split(args.acc_split)
    args.acc_split = dash.acc_split()  # 0 = automatic (per seqlen: sweep rows)
    d = args.head_dim
    seqlens = tuple(int(x) for x in args.seqlens.split(",")) if args.seqlens else SEQLENS
    full_shapes = shapes(d, seqlens)
    probs = [(s, make_problem(*s, causal, rank, world, args.scaling, dash, torch))
             for s in full_shapes]
    torch.cuda.synchronize()

    def step():
        for _, g in probs:
            run_bwd(dash, g, causal, args.schedule, True)

    # FLOPs of the whole job (all ranks): the full problem (strong) or one
    # per rank (weak); per-rank FLOPs for the roofline of this rank's kernel.
    flops_fa = sum(fa_flops(*s, causal) for s in full_shapes)
    job_flops = flops_fa if args.scaling == "strong" else world * flops_fa
    rank_tile = sum(tile_flops(*g["shape"], causal) for _, g in probs)

    # --- headline: device-timed sweep step -----------------------------------
    # --graph: the step (every sweep point's dash_attn_bwd) captured once in a
    # CUDA graph and replayed -- the library is stream-ordered and
    # allocation-free, so the replay runs the same kernels on the same buffers.
    timed_step = step
    if args.graph:
        for _ in range(max(1, args.warmup)):
            step()  # schedule tables uploaded before capture
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        timed_step = graph.replay
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # let nvidia-smi start sampling before the timed region
        ms = time_steps(torch, timed_step, args.steps, args.warmup, world,
                        lambda: clk.mark("t0"), lambda: clk.mark("t1"))
    ms_max = max_over_ranks(ms, world)
    value = job_flops * args.steps / (ms_max / 1e3) / 1e12

    # --- roofline of the main kernel -------------------------------------------
    # A separate pass of the same steps with CUDA events recorded around every
    # kernel of the call (dash_profile_begin/end), so the headline's timed region
    # carries no extra stream operations between the programmatically dependent
    # kernels.  With the fused dQ finalise (N >= 2048) the main kernel's time
    # includes the conversion; a second pass with the K4 convert kernel gives
    # the main kernel's time without it (frac_without_fused_finalise).
    def profiled_main_ms(mode=None):
        old = dash.fused_dq()
        if mode is not None:
            dash.set_fused_dq(mode)
        try:
            step()
            torch.cuda.synchronize()
            dash.profile_begin()
            for _ in range(args.steps):
                step()
            torch.cuda.synchronize()
            return dash.profile_end()[1]
        finally:
            dash.set_fused_dq(old)
    ms_main_timed = profiled_main_ms()
    ms_main_k4 = profiled_main_ms(0) if dash.fused_dq() != 0 else ms_main_timed
    peak, peak_src, peak_sus = load_peaks()
    achieved = rank_tile * args.steps / (ms_main_timed / 1e3) / 1e12
    wl = workload_config(args, world)["workload"]
    traffic = load_traffic(wl)
    tiles = {dash.tile(g["shape"], causal, args.schedule) for _, g in probs}
    main_kernel = "+".join(sorted({256: "dash_bwd_pair_kernel", 128: "dash_bwd_kernel"}[t] for t in tiles))
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": traffic, "kernel": main_kernel,
                "peak_source": peak_src,
                "frac_vs_sustained": achieved / peak_sus if peak_sus else None,
                "main_kernel_share_of_step": ms_main_timed / ms if ms > 0 else None,
                "includes": "the fused dQ finalise at N >= 2048 (K4's conversion, HBM-bound)",
                "frac_without_fused_finalise": rank_tile * args.steps / (ms_main_k4 / 1e3) / 1e12 / peak}

    # --- e2e through the host-buffer ABI call ---------------------------------------
    e2e = None
    if not args.no_e2e:
        host = []
        for _, g in probs:
            hb = {k: g[k].cpu().pin_memory() for k in ("q", "k", "v", "o", "do", "lse")}
            hb["dq"], hb["dk"], hb["dv"] = (torch.empty_like(hb["q"]).pin_memory() for _ in range(3))
            ws = torch.empty(dash.host_workspace_bytes(g["shape"], causal), dtype=torch.uint8,
                             device="cuda")
            host.append((g["shape"], hb, ws))
        h2d = d2h = 0
        for _, hb, _ in host:
            h2d += sum(hb[k].numel() * hb[k].element_size() for k in ("q", "k", "v", "o", "do", "lse"))
            d2h += sum(hb[k].numel() * hb[k].element_size() for k in ("dq", "dk", "dv"))

        def e2e_step():
            for _, hb, ws in host:
                dash.attn_bwd_host(hb["q"], hb["k"], hb["v"], hb["o"], hb["do"], hb["lse"], hb["dq"],
                                   hb["dk"], hb["dv"], causal, args.schedule, True, ws)
        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier(world)
        steps_e2e = max(1, min(args.steps, 5))
        t0 = time.perf_counter()
        for _ in range(steps_e2e):
            e2e_step()
        t1 = time.perf_counter()
        barrier(world)
        e2e_ms = max_over_ranks((t1 - t0) * 1e3 / steps_e2e, world)
        e2e = {"value": job_flops / (e2e_ms / 1e3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
               "steps": steps_e2e, "api": "dash_attn_bwd_host (pinned host buffers)",
               "bytes_note": "per rank" if world > 1 else None}
        del host

    # --- sharding check (N > 1): per-unit digests vs rank 0's 1-GPU run ------------
    sharding_ok = None
    if world > 1 and args.scaling == "strong" and not args.no_verify:
        sharding_ok = gpu_sharding_check(dash, torch, world, rank, probs, full_shapes, causal,
                                         args.schedule)

    # --- per-schedule sweep table and the gate of configs 2 and 3 (N = 1) -------------
    sweep, gate = None, None
    if world == 1 and not args.no_sweep:
        sweep = sweep_rows(dash, torch, probs, causal, args.steps)
        gate = {f"{'causal' if causal else 'full'}_hd{d}": gate_summary(sweep)}
        if not args.no_gate:
            del probs
            torch.cuda.empty_cache()
            others = [(c, hd) for c, hd in ((True, 128), (False, 128), (False, 64), (True, 64))
                      if (c, hd) != (causal, d)]
            for c, hd in others:
                ps = [(s, make_problem(*s, c, 0, 1, "strong", dash, torch)) for s in shapes(hd, seqlens)]
                rows = sweep_rows(dash, torch, ps, c, args.steps)
                gate[f"{'causal' if c else 'full'}_hd{hd}"] = dict(gate_summary(rows), rows=rows)
                del ps
                torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample(d, causal)
        cpu.pop("seconds", None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded N(0,1) bf16 q,k,v,dO; O, L from dash_attn_fwd)",
            "config": dict(workload_config(args, world),
                           schedule_resolved={str(sh[1]): dash.resolve_schedule(sh, causal, args.schedule)
                                              for sh in full_shapes},
                           acc_split_resolved={str(sh[1]): dash.acc_split(sh, causal, args.schedule)
                                               for sh in full_shapes},
                           tile_resolved={str(sh[1]): dash.tile(sh, causal, args.schedule)
                                          for sh in full_shapes}),
            "frac_of_peak": value / peak / world,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": sum(dash.bwd_launch_count(sh, causal, args.schedule, True)
                                for sh in full_shapes) * args.steps,
            "clocks": clk.summary(),
            "sharding_bitwise_identical": sharding_ok,
            "gate": gate,
            "sweep": sweep,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
