"""The fused peer-memory exchange (csrc/exchange.cu, parallel.PeerExchange)
run by real separate processes: world_size 2 and 3, every rank on cuda:0
(CUDA IPC between processes works on one device, so the IPC mapping, the P2P
stores, the epoch flags and the double-buffered contributions are exercised
end to end; across GPUs the same stores travel over NVLink).  Exact mode
must reproduce the unsharded pr_blocked bit for bit; fast mode to 1e-12.
"""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GRAPH = ("rmat", 14, 16, 3)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist

    import paper_1904_02241_b200 as gcb
    from paper_1904_02241_b200 import _lib, parallel

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    _, scale, ef, seed = GRAPH
    gt = gcb.generate_rmat(scale, ef, seed, transposed=True)
    plan = parallel.ShardPlan(parallel.shard_ranges(gt.row_offsets, world))
    results = {}
    for exact in (True, False):
        flags = _lib.FLAG_EXACT if exact else 0
        eng = parallel.DeviceShard(gt, *plan.owned(rank), 1 << 12, flags)
        ex = parallel.PeerExchange(eng, plan, rank)
        runner = parallel.ShardedPageRank(eng, plan, rank, ex)
        for rep in range(2):  # epochs continue across runs
            r = runner.run(gcb.PrParams(tol=0.0, max_iters=10))
            results[f"p10_{exact}_{rep}"] = r.ranks.cpu().numpy()
        r = runner.run(gcb.PrParams(tol=1e-9, max_iters=200))
        results[f"tol_{exact}"] = r.ranks.cpu().numpy()
        results[f"tol_{exact}_it"] = np.array([r.iterations, int(r.converged)])
        ex.close()
        # sharded SpMV over the same slabs, y all-gathered across the processes
        x = torch.as_tensor(np.random.default_rng(9).random(gt.num_vertices)).cuda()
        results[f"spmv_{exact}"] = parallel.ShardedSpmv(eng, plan, rank).run(x).cpu().numpy()
    # degree-ordered shards (fast): intermediate tol = 0 steps skip the ids
    # without out-edges (GCB_FLAG_DEAD_SKIP), cuts by live vertex cost
    gdo, perm = parallel.degree_order(gt)
    plan_do = parallel.ShardPlan(parallel.shard_ranges(gdo.row_offsets, world,
                                                       live_end=parallel.live_end(gdo)))
    eng = parallel.DeviceShard(gdo, *plan_do.owned(rank), 0, 0, True)
    ex = parallel.PeerExchange(eng, plan_do, rank)
    runner = parallel.ShardedPageRank(eng, plan_do, rank, ex)
    for rep in range(2):
        for iters in (1, 10):
            r = runner.run(gcb.PrParams(tol=0.0, max_iters=iters))
            results[f"do{iters}_{rep}"] = parallel.unpermute(r.ranks, perm).cpu().numpy()
    ex.close()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **results)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_matches_unsharded(tmp_path, world):
    import torch.multiprocessing as mp

    import paper_1904_02241_b200 as gcb

    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    _, scale, ef, seed = GRAPH
    bg = gcb.partition_tocab(gcb.generate_rmat(scale, ef, seed, transposed=True), "pull", 1 << 12)
    want = gcb.pr_blocked(bg, gcb.PrParams(tol=0.0, max_iters=10), exact=True).ranks
    want1 = gcb.pr_blocked(bg, gcb.PrParams(tol=0.0, max_iters=1), exact=True).ranks
    want_tol = gcb.pr_blocked(bg, gcb.PrParams(tol=1e-9, max_iters=200), exact=True)
    want_y = gcb.spmv_blocked(bg, np.random.default_rng(9).random(bg.num_vertices), exact=True)
    for rank in range(world):
        got = np.load(tmp_path / f"rank{rank}.npz")
        for rep in range(2):
            assert np.array_equal(got[f"p10_True_{rep}"], want)
            assert np.max(np.abs(got[f"p10_False_{rep}"] - want) / want) <= 1e-12
            assert np.max(np.abs(got[f"do10_{rep}"] - want) / want) <= 1e-12
            assert np.max(np.abs(got[f"do1_{rep}"] - want1) / want1) <= 1e-12
        it, conv = got["tol_True_it"]
        assert (int(it), bool(conv)) == (want_tol.iterations, want_tol.converged)
        assert np.array_equal(got["tol_True"], want_tol.ranks)
        assert np.max(np.abs(got["tol_False"] - want_tol.ranks) / want_tol.ranks) <= 1e-9
        assert np.array_equal(got["spmv_True"], want_y)
        assert np.max(np.abs(got["spmv_False"] - want_y) / np.maximum(want_y, 1e-300)) <= 1e-12
