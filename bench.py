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
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
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

def cpu_pagerank_sample(arenas, n, m, budget_s, threads, direction="pull"):
    """Run oracle pr_blocked iterations (1 per call, OpenMP over rows) until
    ``budget_s`` has elapsed; returns (GTEPS, iterations, seconds)."""
    from oracle import oracle as orc

    bg = orc.Blocked(direction, 0, n, m, *arenas)
    done, spent = 0, 0.0
    while spent < budget_s or done == 0:
        t0 = time.perf_counter()
        orc.pr_blocked(bg, tol=0.0, max_iters=1, threads=threads)
        spent += time.perf_counter() - t0
        done += 1
    return m * done / spent / 1e9, done, spent


def run_reference(args):
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
    arenas = (bg.row_starts, bg.lro_arena, bg.id_map_arena, bg.edge_starts, bg.col_arena)
    for _ in range(args.warmup):
        orc.pr_blocked(bg, tol=0.0, max_iters=1, threads=threads)
    times = []
    for _ in range(args.steps):
        t = time.perf_counter()
        orc.pr_blocked(bg, tol=0.0, max_iters=1, threads=threads)
        times.append(time.perf_counter() - t)
    del arenas
    t_step = float(np.mean(times))
    value = m / t_step / 1e9
    sample = (f"{args.steps} steps x 1 PageRank iteration of rmat:{args.scale}:"
              f"{args.edge_factor}:{args.seed} pull TOCAB W={args.width} (full graph); "
              f"oracle setup {setup_s:.1f}s untimed")
    line = {
        "metric": "PageRank GTEPS per iteration", "value": round(value, 6), "unit": "GTEPS",
        "impl": "reference", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_step * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic R-MAT (reference generator)",
        "config": workload_config(args, n, m),
        "cpu_baseline": {"value": round(value, 6), "unit": "GTEPS", "cores": threads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 6), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(args, n, m):
    return {
        "workload": (f"pagerank-{args.direction}-tocab rmat:{args.scale}:{args.edge_factor}:"
                     f"{args.seed} {args.iters} iterations/step"),
        "graph": f"rmat:{args.scale}:{args.edge_factor}:{args.seed}",
        "num_vertices": n, "num_edges": m, "width": args.width,
        "layout": ("steady state: degree-ordered copy with hybrid edge classes, built in the "
                   "untimed warm-up (e2e: hot-bit layout of each freshly uploaded graph)"
                   if args.gpus == 1 and not args.exact and not args.f32_values else
                   "as built by the call path (no promotion)"),
        "iterations_per_step": args.iters, "damping": 0.85, "tol": 0.0,
        "direction": args.direction, "value_dtype": "f32" if args.f32_values else "f64",
        "l2": "inputs larger than L2 (col arena 4|E| bytes >> 126 MB)",
        "parallelism": (f"destination shards x{args.gpus} (cuts balance in-edges + 4 x vertices), "
                        "contribution exchange per config.exchange" if args.gpus > 1 else "single GPU"),
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
        plan = parallel.ShardPlan(parallel.shard_ranges(src.row_offsets, world))
        # width 0: size each shard's blocks from the sources its slab reads
        engine = parallel.DeviceShard(src, *plan.owned(rank), 0, flags)
        # default: the exchange fused into the rank update over peer memory
        # (csrc/exchange.cu); GCB_EXCHANGE=nccl selects the sparse NCCL
        # all_to_all, which is also the fallback when peer mapping fails
        exchange = None
        if os.environ.get("GCB_EXCHANGE", "p2p") == "p2p":
            try:
                exchange = parallel.PeerExchange(engine, plan, rank)
            except RuntimeError as e:
                print(f"peer exchange unavailable ({e}); using NCCL all_to_all", file=sys.stderr)
        if exchange is None:
            exchange = parallel.SparseExchange(plan, rank, engine.source_mask())
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
    # library promotes a graph to its degree-ordered copy after 4096 fast
    # iterations (relabel.cu, ski rental against the ~0.35 s build), so the
    # untimed warm-up asks for the promotion at once.  Only the device-resident
    # graph is promoted: the threshold is restored before the e2e steps, whose
    # fresh host-uploaded graphs run 10 iterations each and never promote.
    saved_after = os.environ.get("GCB_RELABEL_AFTER")
    os.environ["GCB_RELABEL_AFTER"] = "0"
    try:
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
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
    gather_ms = per_iter["gather"]
    gather_groups = prof["gather"][1] / (prof_steps * args.iters)

    peak, peak_kind = measured_hbm_peak()
    peak *= world  # aggregate HBM of the job
    b_alg = algorithmic_bytes_pr(n, m)
    achieved = b_alg / t_iter_s / 1e9
    # dominant kernel (the pull gather, k_pull_hot): SURVEY 8(d) per-edge and
    # per-vertex bytes it must move -- col_idx 4 B/edge, the contribution read
    # 8 B/vertex, the row pointer 4 B/vertex -- over the launches of one iteration
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
        "kernel": "k_pull_hot (TOCAB pull gather) + k_push_hot (hybrid hub-destination edges)",
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

    # ---- e2e: public host-buffer API, arenas from pinned memory each step ----
    e2e = None
    if not args.no_e2e and world == 1:
        e2e = run_e2e(args, bg, ctx, stream, flags)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as orc

        arenas = (bg.row_starts, bg.lro_arena, bg.id_map_arena, bg.edge_starts, bg.col_arena)
        threads = orc.default_threads()
        c_val, c_iters, c_s = cpu_pagerank_sample(arenas, n, m, args.cpu_seconds, threads,
                                                  args.direction)
        cpu = {"value": round(c_val, 6), "unit": "GTEPS", "cores": threads, "kind": "port",
               "sample": f"{c_iters} PageRank iteration(s) of the same rmat:{args.scale} "
                         f"TOCAB W={args.width} graph, oracle/ C port with OpenMP, "
                         f"{c_s:.1f}s"}

    cfg = workload_config(args, n, m)
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
            "gpu_launches": launches, "clocks": clk,
            "setup_s": round(setup_s, 2),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


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


def main():
    args = parse_args()
    if args.width <= 0:
        args.width = auto_width(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
