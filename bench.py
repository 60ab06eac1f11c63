#!/usr/bin/env python
"""TOCAB PageRank throughput on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[2], the north-star target): PageRank pull with
TOCAB on the synthetic R-MAT scale-24 edge-factor-16 graph (seed 1, generated
bit-exactly on the device), damping 0.85, tol 0, 10 iterations per step.
One step = one ``pr_blocked`` call (10 iterations) with inputs resident in HBM.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line (rank 0).  ``value`` is GTEPS per iteration
(|E| * iterations / device seconds / 1e9) summed over ranks; ``e2e`` is the
same metric through the public host-buffer API (graph arenas uploaded from
pinned host memory and ranks read back every step).  The reference arm
(``--impl reference``) times the CPU oracle port (oracle/, a bit-exact
restatement of the reference's pr_blocked) on the host cores.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FALLBACK_HBM_GBS = 6650.0


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--scale", type=int, default=24)
    p.add_argument("--edge-factor", type=int, default=16)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--iters", type=int, default=10)
    p.add_argument("--width", type=int, default=0,
                   help="TOCAB block width; 0 = the largest power of two whose f64 value "
                        "slice fits in 55%% of the device L2 (2^23 on B200: two 64 MiB blocks "
                        "at scale 24)")
    p.add_argument("--direction", choices=("pull", "push"), default="pull")
    p.add_argument("--f32-values", action="store_true")
    p.add_argument("--exact", action="store_true")
    p.add_argument("--no-l2-window", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=12.0,
                   help="bounded CPU sample of our arm's cpu_baseline (at least one call)")
    p.add_argument("--ref-seconds", type=float, default=150.0,
                   help="reference arm: stop timing further calls after this many seconds")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the other BASELINE configs (SpMV rmat:22, BFS / SSSP / CC rmat:24)")
    return p.parse_args()


def algorithmic_bytes_pr(n: int, m: int) -> int:
    """col u32 + row_ptr u32 + f64 rank r/w + f64 contribution
    write + compulsory read + u32 degree."""
    return 4 * m + 4 * (n + 1) + 36 * n


def measured_hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(prefix="gcb_clocks_", suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.device)],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        with open(self.path) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax.append(float(parts[1]))
                except ValueError:
                    continue
                for name, flag in zip(names, parts[3:7]):
                    if flag.lower().startswith("active"):
                        reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


# ---------------------------------------------------------------------------
# CPU leg (oracle port) -- test infrastructure, only a reported baseline
# ---------------------------------------------------------------------------

def cpu_pagerank_sample(arenas, n, m, budget_s, threads, iters, direction="pull"):
    """The reference's run contract (cli.py:199-211, 256-262): whole
    pr_blocked calls of ``iters`` iterations (tol 0), out-degrees counted once
    per call (kernels.py:373-374), on the oracle C port with OpenMP, until
    ``budget_s`` has elapsed (at least one call).  Returns (GTEPS, calls,
    seconds, ranks of the last call, per-call setup seconds)."""
    from oracle import oracle as orc

    bg = orc.Blocked(direction, 0, n, m, *arenas)
    # per-call setup (degree count, allocations): a 1-iteration call minus one
    # iteration of a full call
    t0 = time.perf_counter()
    orc.pr_blocked(bg, tol=0.0, max_iters=1, threads=threads)
    t1 = time.perf_counter() - t0
    done, spent, out = 0, 0.0, None
    while spent < budget_s or done == 0:
        t0 = time.perf_counter()
        out = orc.pr_blocked(bg, tol=0.0, max_iters=iters, threads=threads)
        spent += time.perf_counter() - t0
        done += 1
    per_call = spent / done
    setup = max(0.0, t1 - (per_call - t1) / max(1, iters - 1)) if iters > 1 else 0.0
    return m * iters * done / spent / 1e9, done, spent, out.ranks, setup


def run_reference(args):
    """The reference arm: the CPU implementation of the path (the oracle C
    port of pr_blocked, bit-identical to the reference's numba path), timed on
    the reference's own contract -- one step = one pr_blocked call of
    ``--iters`` iterations (cli.py:256-262) -- with every host thread."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as orc

    threads = orc.default_threads()
    t0 = time.perf_counter()
    src = orc.rmat(args.scale, args.edge_factor, args.seed, threads) if args.direction == "push" \
        else orc.rmat_transpose(args.scale, args.edge_factor, args.seed, threads)
    bg = orc.partition_tocab(src, args.direction, args.width)
    setup_s = time.perf_counter() - t0
    n, m = src.n, src.m
    del src
    # warm-up calls (page faults, OpenMP pool); bounded: CPU calls take seconds
    for _ in range(min(args.warmup, 2)):
        orc.pr_blocked(bg, tol=0.0, max_iters=args.iters, threads=threads)
    # per-call setup, reported apart from the per-iteration rate (a warm
    # 1-iteration call: cold, it could outlast a warm 10-iteration one)
    t = time.perf_counter()
    orc.pr_blocked(bg, tol=0.0, max_iters=1, threads=threads)
    t1 = time.perf_counter() - t
    times = []
    t_start = time.perf_counter()
    for _ in range(args.steps):
        t = time.perf_counter()
        orc.pr_blocked(bg, tol=0.0, max_iters=args.iters, threads=threads)
        times.append(time.perf_counter() - t)
        if time.perf_counter() - t_start > args.ref_seconds:
            break  # keep the arm within a few minutes; steps says how many ran
    t_step = float(np.mean(times))
    value = m * args.iters / t_step / 1e9
    per_iter = (t_step - t1) / max(1, args.iters - 1) if args.iters > 1 else t_step
    if per_iter <= 0.0:  # timer noise at toy sizes: fall back to the mean
        per_iter = t_step / max(1, args.iters)
    call_setup = max(0.0, t1 - per_iter)
    sample = (f"{len(times)} pr_blocked calls x {args.iters} iterations (tol 0) of rmat:{args.scale}:"
              f"{args.edge_factor}:{args.seed} {args.direction} TOCAB W={args.width} (full graph), "
              f"oracle C port with OpenMP ({threads} threads); per-call setup "
              f"{call_setup * 1e3:.0f} ms of {t_step * 1e3:.0f} ms; graph build {setup_s:.1f}s untimed")
    line = {
        "metric": "PageRank GTEPS per iteration", "value": round(value, 6), "unit": "GTEPS",
        "impl": "reference", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": len(times), "warmup": min(args.warmup, 2),
        "ms_per_step": round(t_step * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic R-MAT (reference generator)",
        "config": workload_config(args, n, m, int(os.environ.get("WORLD_SIZE", "1"))),
        "cpu_baseline": {"value": round(value, 6), "unit": "GTEPS", "cores": threads,
                         "kind": "port", "sample": sample,
                         "ms_per_iteration": round(per_iter * 1e3, 3),
                         "ms_setup_per_call": round(call_setup * 1e3, 3)},
        "e2e": {"value": round(value, 6), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, n, m, world):
    return {
        "workload": (f"pagerank-{args.direction}-tocab rmat:{args.scale}:{args.edge_factor}:"
                     f"{args.seed} {args.iters} iterations/step"),
        "graph": f"rmat:{args.scale}:{args.edge_factor}:{args.seed}",
        "num_vertices": n, "num_edges": m, "width": args.width,
        "layout": ("steady state: degree-ordered copy with hybrid edge classes, built in the "
                   "untimed warm-up (e2e: hot-bit layout of each freshly uploaded graph)"
                   if world == 1 and not args.exact and not args.f32_values else
                   "degree-ordered shards: graph renumbered by out-degree on every rank, slabs "
                   "blocked with the prefix hot set and the hub pass where it pays "
                   "(gcb_shard_blocking); intermediate steps skip ids without out-edges"
                   if world > 1 and not args.exact and not args.f32_values
                   and os.environ.get("GCB_SHARD_ORDER", "1") == "1" else
                   "as built by the call path (no promotion)"),
        "iterations_per_step": args.iters, "damping": 0.85, "tol": 0.0,
        "direction": args.direction, "value_dtype": "f32" if args.f32_values else "f64",
        "l2": "inputs larger than L2 (col arena 4|E| bytes >> 126 MB)",
        "parallelism": (f"destination shards x{world} (cuts balance in-edges + 4 x live "
                        "vertices, then one re-cut from measured steps), contribution exchange "
                        "per config.exchange" if world > 1 else "single GPU"),
    }


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1904_02241_b200 as gcb
    from paper_1904_02241_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                         "(bench.py --gpus N without torchrun starts them itself)")
    # GCB_DEVICE / GCB_DIST_BACKEND let the multi-rank path be smoke-tested
    # with several ranks on one GPU (gloo); production is one rank per GPU, NCCL
    local = int(os.environ.get("GCB_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(local)
    if world > 1:
        backend = os.environ.get("GCB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    ctx = _lib.context(local)
    # a real (non-legacy) stream shared by the library and the timing events
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    # ---- setup (untimed): device R-MAT -> transpose -> TOCAB partition ----
    t0 = time.perf_counter()
    flags = 0
    if args.exact:
        flags |= _lib.FLAG_EXACT
    if args.f32_values:
        flags |= _lib.FLAG_F32_VALUES
    if args.no_l2_window:
        flags |= _lib.FLAG_NO_L2_WINDOW
    if args.direction == "pull":
        src = gcb.generate_rmat(args.scale, args.edge_factor, args.seed, transposed=True)
    else:
        src = gcb.generate_rmat(args.scale, args.edge_factor, args.seed)
    if world > 1:
        # strong scaling: every rank builds the same graph and owns an
        # equal-in-edge destination range (parallel.py)
        from paper_1904_02241_b200 import parallel

        if args.direction != "pull":
            raise SystemExit("multi-GPU PageRank shards the pull direction")
        # every rank renumbers the graph by out-degree and blocks its slab with
        # the global prefix hot set (and the hub pass where it pays); the cuts
        # charge vertex cost to live rows only, since intermediate tol = 0 steps
        # skip the ids without out-edges.  At rmat:24, P = 8 that ran the
        # slowest shard step in 0.118 ms against 0.145 ms for the input
        # numbering (DESIGN 7).  GCB_SHARD_ORDER=0 keeps the input numbering.
        ordered = (not args.exact and not args.f32_values
                   and os.environ.get("GCB_SHARD_ORDER", "1") == "1")
        live = None
        if ordered:
            src, _perm = parallel.degree_order(src)
            live = parallel.live_end(src)

        def build(ranges):
            plan = parallel.ShardPlan(ranges)
            # width 0: size each shard's blocks from the sources its slab reads
            engine = parallel.DeviceShard(src, *plan.owned(rank), 0, flags, ordered)
            # default: the exchange fused into the rank update over peer memory
            # (csrc/exchange.cu); GCB_EXCHANGE=nccl selects the sparse NCCL
            # all_to_all, which is also the fallback when peer mapping fails
            exchange = None
            if os.environ.get("GCB_EXCHANGE", "p2p") == "p2p":
                try:
                    exchange = parallel.PeerExchange(engine, plan, rank)
                except RuntimeError as e:
                    print(f"peer exchange unavailable ({e}); using NCCL all_to_all",
                          file=sys.stderr)
            if exchange is None:
                exchange = parallel.SparseExchange(plan, rank, engine.source_mask())
            return plan, engine, exchange

        ranges = parallel.shard_ranges(src.row_offsets, world, live_end=live)
        plan, engine, exchange = build(ranges)
        if os.environ.get("GCB_SHARD_CALIB", "1") == "1":
            # one calibration pass (untimed setup): every rank times its own
            # intermediate step, the cuts move to the measured costs
            # (parallel.rebalance_ranges), and the shards are rebuilt
            import torch.distributed as dist

            c = torch.zeros(src.num_vertices, dtype=torch.float64, device=engine.device)
            r_ = torch.zeros_like(c)
            engine.init(c, r_)
            for _ in range(3):
                engine.step(c, r_, 0.85, False, dead_skip=True)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                engine.step(c, r_, 0.85, False, dead_skip=True)
            e1.record()
            torch.cuda.synchronize()
            times = [None] * world
            dist.all_gather_object(times, e0.elapsed_time(e1) / 5)
            del c, r_
            if getattr(exchange, "close", None):
                exchange.close()
            del engine, exchange
            ranges = parallel.rebalance_ranges(src.row_offsets, ranges, times, live_end=live)
            plan, engine, exchange = build(ranges)
        runner = parallel.ShardedPageRank(engine, plan, rank, exchange)
        n, m = src.num_vertices, src.num_edges
        bg = engine.bg
        del src
        params = gcb.PrParams(tol=0.0, max_iters=args.iters)

        def step():
            runner.run(params, gather_ranks=False)
    else:
        bg = gcb.partition_tocab(src, args.direction, args.width)
        n, m = bg.num_vertices, bg.num_edges
        del src
        h = bg.device()
        ranks = torch.empty(n, dtype=torch.float64, device=f"cuda:{local}")
        it, cv = ctypes.c_int(), ctypes.c_int()

        def step():
            _lib.check(ctx._lib.gcb_pr_blocked_dev(ctx.handle, h.raw, 0.85, 0.0, args.iters,
                                                   flags, ctypes.c_void_p(ranks.data_ptr()),
                                                   ctypes.byref(it), ctypes.byref(cv)))

    # The timed region measures the steady state of a long-running job: the
    # library promotes a graph to its degree-ordered copy after 256 fast
    # iterations (relabel.cu, ski rental against the ~55 ms build), so the
    # untimed warm-up asks for the promotion at once.  Only the device-resident
    # graph is promoted: the threshold is restored before the e2e steps, whose
    # fresh host-uploaded graphs run 10 iterations each and never promote.
    saved_after = os.environ.get("GCB_RELABEL_AFTER")
    os.environ["GCB_RELABEL_AFTER"] = "0"
    warm_ms = []
    try:
        for _ in range(max(args.warmup, 3)):
            torch.cuda.synchronize()
            tw = time.perf_counter()
            step()
            torch.cuda.synchronize()
            warm_ms.append(1e3 * (time.perf_counter() - tw))
    finally:
        if saved_after is None:
            os.environ.pop("GCB_RELABEL_AFTER", None)
        else:
            os.environ["GCB_RELABEL_AFTER"] = saved_after
    setup_s = time.perf_counter() - t0

    # ---- timed region ----
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)  # let the sampler attach before the measured launches
    launches0 = ctx.launches()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launches() - launches0
    clk = clocks.stop()
    ms_total = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()
    ms_step = ms_total / args.steps
    t_iter_s = ms_step / 1e3 / args.iters
    # the whole graph (m edges) is processed once per iteration by the job
    value = m / t_iter_s / 1e9

    # ---- per-kernel breakdown (separate, profiled pass; not the timed number) ----
    ctx.set_profiling(True)
    prof_steps = 3
    for _ in range(prof_steps):
        step()
    prof = ctx.read_profile()
    ctx.set_profiling(False)
    per_iter = {k: v[0] / (prof_steps * args.iters) for k, v in prof.items()}
    pull_ms = per_iter["gather"]
    hub_ms = per_iter["hub_push"]
    gather_ms = pull_ms + hub_ms
    gather_groups = (prof["gather"][1] + prof["hub_push"][1]) / (prof_steps * args.iters)

    peak, peak_kind = measured_hbm_peak()
    peak *= world  # aggregate HBM of the job
    b_alg = algorithmic_bytes_pr(n, m)
    achieved = b_alg / t_iter_s / 1e9
    # dominant kernel (the pull gather, k_pull_hot, with the hybrid hub push
    # pass k_push_hub + k_hub_fold): SURVEY 8(d) per-edge and per-vertex bytes it must move
    # -- col_idx 4 B/edge, the contribution read 8 B/vertex, the row pointer
    # 4 B/vertex -- over the launches of one iteration
    b_gather = 4 * m + 8 * n + 4 * (n + 1)
    gather_s = gather_ms / 1e3
    g_achieved = b_gather / gather_s / 1e9 if gather_ms else None
    traffic = None
    prof_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof_file):
        try:
            with open(prof_file) as fh:
                tj = json.load(fh)
            # only when the capture is of this very workload
            if (tj.get("graph") == f"rmat:{args.scale}:{args.edge_factor}:{args.seed}"
                    and tj.get("width") == args.width):
                traffic = tj.get("k_pull_hot_bytes_per_iteration")
        except Exception:
            traffic = None
    roofline = {
        "bound": "hbm",
        "kernel": "k_pull_hot (TOCAB pull gather) + k_push_hub, k_hub_fold (hybrid hub-destination edges)",
        "achieved": round(g_achieved, 1) if g_achieved else None, "peak": peak, "unit": "GB/s",
        "frac": round(g_achieved / peak, 4) if g_achieved else None,
        "traffic": traffic, "peak_source": peak_kind,
        "algorithmic_bytes_per_iteration": b_gather,
        "launches_per_iteration": gather_groups,
        "ms_per_iteration": round(gather_ms, 4),
        "share_of_iteration": round(gather_ms / (t_iter_s * 1e3), 3),
        "scope": "per iteration (all gather launches); traffic = ncu dram bytes of the same "
                 "launches (profiles/ncu_traffic.json)",
        "iteration": {
            "achieved": round(achieved, 1), "frac": round(achieved / peak, 4),
            "algorithmic_bytes": b_alg,
            "scope": "one whole PageRank iteration (every launch); B_alg = 4|E| + 4(|V|+1) + "
                     "36|V| (SURVEY 8d) -- the metric's 'fraction of HBM roofline'",
        },
        "kernels_ms_per_iter": {k: round(v, 4) for k, v in per_iter.items()},
    }
    if world == 1 and args.direction == "pull" and not args.exact:
        roofline["requests"] = request_model(ctx, bg, pull_ms, hub_ms, clk)

    # ---- parity of the timed output (cli.py:226-239 verifies every run) ----
    parity = None
    if world == 1 and not args.f32_values:
        parity = timed_parity(ctx, bg, ranks, args, flags)

    # ---- the layout a default API call runs (no promotion yet) ----
    layouts = None
    if world == 1 and not args.exact and not args.f32_values:
        layouts = default_layout_rate(ctx, bg, stream, args, flags, value, ms_step)
        if len(warm_ms) > 1:
            # first warm-up call = derived tables + the promotion build + one step
            build = warm_ms[0] - min(warm_ms[1:])
            saving = (layouts["default_api"]["ms_per_step"] - ms_step) / args.iters
            layouts["promotion"] = {
                "after_fast_iterations": 256, "first_call_extra_ms": round(build, 1),
                "saving_ms_per_iteration": round(saving, 4),
                "break_even_iterations": round(build / saving) if saving > 0 else None,
                "note": "wall time of the first warm-up call over the later ones: derived "
                        "tables of the uploaded graph + the degree-ordered build, including "
                        "the memory pool's first growth in a fresh process (the build alone: "
                        "41-43 ms at rmat:24, profiles/r2_promotion_trace.txt)"}

    # ---- e2e: public host-buffer API, arenas from pinned memory each step ----
    e2e = None
    if not args.no_e2e and world == 1:
        e2e = run_e2e(args, bg, ctx, stream, flags)

    # ---- the other BASELINE configs, one timing each (not the headline) ----
    secondary = None
    if world == 1 and not args.no_secondary and args.scale == 24:
        secondary = run_secondary(ctx, stream, local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as orc

        arenas = (bg.row_starts, bg.lro_arena, bg.id_map_arena, bg.edge_starts, bg.col_arena)
        threads = orc.default_threads()
        c_val, c_calls, c_s, c_ranks, c_setup = cpu_pagerank_sample(
            arenas, n, m, args.cpu_seconds, threads, args.iters, args.direction)
        cpu = {"value": round(c_val, 6), "unit": "GTEPS", "cores": threads, "kind": "port",
               "sample": f"{c_calls} pr_blocked call(s) x {args.iters} iterations of the same "
                         f"rmat:{args.scale} TOCAB W={args.width} graph, oracle/ C port with "
                         f"OpenMP, {c_s:.1f}s; per-call setup {c_setup * 1e3:.0f} ms"}
        if parity is not None:
            # the oracle restates the reference's pr_blocked bit for bit
            # (tests/test_oracle.py): check the timed ranks against it too
            h = ranks.cpu().numpy()
            ex = parity.pop("_exact")
            rel = np.abs(h - c_ranks) / np.abs(c_ranks)
            parity["vs_oracle_max_rel"] = float(rel.max())
            parity["vs_oracle_max_abs"] = float(np.abs(h - c_ranks).max())
            parity["exact_bitwise_vs_oracle"] = bool(np.array_equal(ex, c_ranks))
            parity["verify_cli"] = bool(parity["vs_oracle_max_abs"] <= 1e-10 * n)
    if parity is not None:
        parity.pop("_exact", None)

    cfg = workload_config(args, n, m, world)
    if world > 1:
        cfg["width"] = int(bg.width)  # rank 0's shard width (auto: DeviceShard._auto_width)
        if getattr(exchange, "fused", False):
            cfg["exchange"] = "peer-memory stores fused into the rank update (CUDA IPC / NVLink)"
            cfg["exchange_bytes_stored_rank0"] = int(exchange.bytes_per_step)
        else:
            cfg["exchange"] = "NCCL all_to_all_single of the contributions each shard reads"
            cfg["exchange_bytes_received_rank0"] = int(exchange.bytes_received)
    if rank == 0:
        line = {
            "metric": "PageRank GTEPS per iteration", "value": round(value, 3), "unit": "GTEPS",
            "n_gpus": world, "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic R-MAT generated on device (bit-exact with the reference)",
            "config": cfg,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "parity": parity, "layouts": layouts, "secondary": secondary,
            "gpu_launches": launches, "clocks": clk,
            "setup_s": round(setup_s, 2),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# Random 8-byte LDG rate of one SM from an L2-resident vector, measured by
# scripts/mb_gather.cu on this B200 (DESIGN 4.1): the request ceiling of the
# L1TEX -> XBAR path that bounds every cold gather.
GATHERS_PER_SM_CYCLE = 0.93


def request_model(ctx, bg, pull_ms, hub_ms, clk):
    """Cold gathers per iteration against the request ceiling: the pull pass
    issues one L2 request per cold edge, so its floor is cold /
    (0.93 x SMs x clock); request_frac = that floor / the measured pull time."""
    out = (ctypes.c_int64 * 4)()
    from paper_1904_02241_b200 import _lib

    _lib.check(ctx._lib.gcb_blocked_gather_census(ctx.handle, bg.device().raw, out), "census")
    hot, cold, hub, relabeled = (int(x) for x in out)
    sms = ctx.info()["num_sms"] if hasattr(ctx, "info") else 148
    mhz = (clk or {}).get("sm_mhz") or 1965.0
    floor_ms = cold / (GATHERS_PER_SM_CYCLE * sms * mhz * 1e6) * 1e3
    total = hot + cold + hub
    return {"hot_table_edges": hot, "cold_edges": cold, "hub_push_edges": hub,
            "cold_share": round(cold / total, 4) if total else None,
            "layout": "degree-ordered + hybrid" if relabeled else "hot-bit",
            "pull_ms_per_iteration": round(pull_ms, 4),
            "hub_push_ms_per_iteration": round(hub_ms, 4),
            "request_floor_ms": round(floor_ms, 4),
            "request_frac": round(floor_ms / pull_ms, 4) if pull_ms else None,
            "model": f"cold edges / ({GATHERS_PER_SM_CYCLE} gathers per SM-cycle x {sms} SMs x "
                     f"{mhz:.0f} MHz); 0.93 = scripts/mb_gather.cu random-LDG ceiling"}


def timed_parity(ctx, bg, ranks, args, flags):
    """The timed steps' ranks against one exact-mode call on the same graph
    (bit-identical to the reference: tests/test_gpu_parity.py, and checked
    against the oracle below when the CPU leg runs)."""
    import torch

    from paper_1904_02241_b200 import _lib

    ex = torch.empty_like(ranks)
    it, cv = ctypes.c_int(), ctypes.c_int()
    _lib.check(ctx._lib.gcb_pr_blocked_dev(ctx.handle, bg.device().raw, 0.85, 0.0, args.iters,
                                           flags | _lib.FLAG_EXACT, ctypes.c_void_p(ex.data_ptr()),
                                           ctypes.byref(it), ctypes.byref(cv)))
    torch.cuda.synchronize()
    rel = ((ranks - ex).abs() / ex.abs()).max().item()
    return {"vs_exact_max_rel": rel, "tolerance": 1e-6, "pass": bool(rel <= 1e-6),
            "reference": "exact mode (reference operation order) on the same device graph",
            "_exact": ex.cpu().numpy()}


def default_layout_rate(ctx, bg, stream, args, flags, value, ms_step):
    """Steady state of the layout a default API call runs before promotion
    (GCB_RELABEL_AFTER = 256 fast iterations): the hot-bit layout of the
    graph as partitioned.  Same step, timed the same way."""
    import torch

    from paper_1904_02241_b200 import _lib

    n, m = bg.num_vertices, bg.num_edges
    out = torch.empty(n, dtype=torch.float64, device=stream.device)
    it, cv = ctypes.c_int(), ctypes.c_int()
    f = flags | _lib.FLAG_NO_RELABEL

    def step():
        _lib.check(ctx._lib.gcb_pr_blocked_dev(ctx.handle, bg.device().raw, 0.85, 0.0, args.iters,
                                               f, ctypes.c_void_p(out.data_ptr()),
                                               ctypes.byref(it), ctypes.byref(cv)))

    for _ in range(3):
        step()
    k = max(3, min(10, args.steps))
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(k):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / k
    return {"timed": {"layout": "degree-ordered copy + hybrid hub push (promoted)",
                      "value": round(value, 3), "ms_per_step": round(ms_step, 4)},
            "default_api": {"layout": "hot-bit layout of the graph as partitioned (before "
                                      "promotion at 256 fast iterations)",
                            "value": round(m * args.iters / (ms / 1e3) / 1e9, 3),
                            "ms_per_step": round(ms, 4), "steps": k}}


def run_secondary(ctx, stream, local):
    """BASELINE configs[1] and [3] (plus CC of configs[4]'s algorithm at
    rmat:24), each against its SURVEY 8(d) byte model.  SpMV runs on device
    vectors (CUDA events over 20 calls); BFS / SSSP / CC are public API calls
    whose numpy results come back inside the call (wall time, median of 3
    after a warm-up that builds the execution layouts), plus the traversal's
    own device span (the library's CUDA-event profile scope)."""
    import torch

    import paper_1904_02241_b200 as gcb
    from paper_1904_02241_b200 import _lib

    peak, _ = measured_hbm_peak()
    out = {}

    def wall(fn, reps=3):
        fn()
        ts = []
        r = None
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = fn()
            ts.append(time.perf_counter() - t0)
        return r, float(np.median(ts))

    def device_ms(fn, reps=3):
        # the library's profile scope around the traversal itself (CUDA events
        # on its stream; the host copies of the results are outside it)
        ts = []
        for _ in range(reps):
            ctx.set_profiling(True)
            fn()
            ts.append(ctx.read_profile()["other"][0])
            ctx.set_profiling(False)
        return float(np.median(ts))

    # configs[1]: SpMV pull TOCAB, rmat:22, x = default_rng(42).random(n)
    gt = gcb.generate_rmat(22, 16, 1, transposed=True)
    n, m = gt.num_vertices, gt.num_edges
    bg = gcb.partition_tocab(gt, "pull", 1 << 22)
    del gt
    h = bg.device()
    x = np.random.default_rng(42).random(n)
    xd = torch.from_numpy(x).to(f"cuda:{local}")
    yd = torch.empty_like(xd)

    def spmv():
        _lib.check(ctx._lib.gcb_spmv_blocked_dev(ctx.handle, h.raw, ctypes.c_void_p(xd.data_ptr()),
                                                 0, ctypes.c_void_p(yd.data_ptr())))
    for _ in range(3):
        spmv()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(20):
        spmv()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    b = 4 * m + 4 * (n + 1) + 16 * n
    y_exact = gcb.spmv_blocked(bg, x, exact=True)
    rel = float(np.max(np.abs(yd.cpu().numpy() - y_exact) / np.maximum(np.abs(y_exact), 1e-300)))
    out["spmv"] = {"config": "BASELINE configs[1]: SpMV pull TOCAB rmat:22:16:1, W=2^22, device x/y",
                   "ms": round(ms, 4), "gteps": round(m / ms / 1e6, 1),
                   "algorithmic_bytes": b, "achieved_gbs": round(b / ms / 1e6, 1),
                   "frac": round(b / ms / 1e6 / peak, 4),
                   "parity_vs_exact_max_rel": rel}
    del bg, h, xd, yd

    # configs[3]: BFS and SSSP (integer weights) from the hub, rmat:24; CC
    g = gcb.generate_rmat(24, 16, 1)
    n, m = g.num_vertices, g.num_edges
    deg = g.out_degrees
    bgt = gcb.partition_tocab(gcb.transpose(g), "pull", 1 << 21)
    r, t = wall(lambda: gcb.bfs(g, 0, g_blocked=bgt))
    td = device_ms(lambda: gcb.bfs(g, 0, g_blocked=bgt)) / 1e3
    reached = np.flatnonzero(r.depth != gcb.INF_DEPTH)
    te = int(deg[reached].sum())
    b = 4 * te + 8 * n
    out["bfs"] = {"config": "BASELINE configs[3]: BFS from 0 with the direction switch, rmat:24:16:1",
                  "ms_api": round(t * 1e3, 3), "gteps": round(te / t / 1e9, 2),
                  "ms_device": round(td * 1e3, 3), "gteps_device": round(te / td / 1e9, 2),
                  "levels": len(r.levels), "directions": r.directions,
                  "reached": int(reached.size), "algorithmic_bytes": b,
                  "frac": round(b / td / 1e9 / peak, 4),
                  "note": "ms_api includes the depth array and level queues to host (96 MB); "
                          "ms_device / frac: the traversal's own span on the device"}
    del bgt
    w = np.random.default_rng(7).integers(1, 256, m).astype(np.float64)
    gw = gcb.CsrGraph(n, m, g.row_offsets, g.col_indices, w)
    bgw = gcb.partition_tocab(gcb.transpose(gw), "pull", 1 << 21)
    r, t = wall(lambda: gcb.sssp(gw, 0, g_blocked=bgw))
    td = device_ms(lambda: gcb.sssp(gw, 0, g_blocked=bgw)) / 1e3
    reached = np.flatnonzero(r.dist != gcb.INF_DIST)
    te = int(deg[reached].sum())
    b = 4 * te + 8 * n
    out["sssp"] = {"config": "BASELINE configs[3]: SSSP from 0, weights default_rng(7) U[1,255], "
                             "rmat:24:16:1",
                   "ms_api": round(t * 1e3, 3), "gteps": round(te / t / 1e9, 2),
                   "ms_device": round(td * 1e3, 3), "gteps_device": round(te / td / 1e9, 2),
                   "rounds": r.rounds, "reached": int(reached.size),
                   "algorithmic_bytes_per_run": b}
    del bgw, gw, w
    r, t = wall(lambda: gcb.cc(g))
    td = device_ms(lambda: gcb.cc(g)) / 1e3
    out["cc"] = {"config": "CC (configs[4]'s algorithm) on rmat:24:16:1", "ms_api": round(t * 1e3, 3),
                 "gteps": round(m / t / 1e9, 2), "ms_device": round(td * 1e3, 3),
                 "gteps_device": round(m / td / 1e9, 2), "components": int(r.num_components)}
    del g
    torch.cuda.synchronize()
    return out


def run_e2e(args, bg, ctx, stream, flags, steps=None):
    """Same metric through the reference-facing API: BlockedGraph with host
    arenas in pinned memory -> upload + pr_blocked -> host ranks, per step."""
    import torch

    import paper_1904_02241_b200 as gcb
    from paper_1904_02241_b200 import _lib

    def pinned(a):
        t = torch.empty(a.shape, dtype=getattr(torch, str(a.dtype)), pin_memory=True)
        t.numpy()[...] = a
        return t

    host = {k: pinned(getattr(bg, k)) for k in ("row_starts", "lro_arena", "id_map_arena",
                                                 "edge_starts", "col_arena")}
    h2d = sum(t.numel() * t.element_size() for t in host.values())
    n, m = bg.num_vertices, bg.num_edges
    out = torch.empty(n, dtype=torch.float64, pin_memory=True)
    d2h = n * 8
    params = gcb.PrParams(tol=0.0, max_iters=args.iters)

    def step():
        hb = gcb.BlockedGraph(bg.direction, "tocab", bg.width, n, m,
                              *(host[k].numpy() for k in ("row_starts", "lro_arena",
                                                          "id_map_arena", "edge_starts",
                                                          "col_arena")))
        gcb.pr_blocked(hb, params, exact=bool(flags & _lib.FLAG_EXACT),
                       f32_values=bool(flags & _lib.FLAG_F32_VALUES), out=out.numpy())
        del hb

    step()
    k = steps or max(3, min(10, args.steps))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k):
        step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / k
    return {"value": round(m * args.iters / dt / 1e9, 3), "unit": "GTEPS",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(dt * 1e3, 2), "steps": k,
            "path": "pr_blocked(BlockedGraph(host arenas)) -> gcb_blocked_upload + "
                    "gcb_pr_blocked (ranks to host)"}


def auto_width(args) -> int:
    """TOCAB sizing rule (north star (1)): one block's f64 value slice must fit
    in L2 next to the streamed arenas -> <= 55% of the L2 the device reports."""
    l2 = 126 * 2 ** 20
    try:
        import torch

        if torch.cuda.is_available():
            l2 = int(torch.cuda.get_device_properties(0).L2_cache_size)
    except Exception:
        pass
    budget = int(l2 * 0.55) // 8
    w = 1
    while w * 2 <= budget and w < (1 << args.scale):
        w *= 2
    return w


def launch_ranks(args) -> int:
    """--gpus N outside torchrun: start one rank per GPU the way the driver
    does (torch.distributed.run, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_ranks(args))
    if args.width <= 0:
        args.width = auto_width(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
