"""Host-side logic that needs no GPU: argument validation (raised before any
device call), generator specs, schedule strategies, GCB container I/O,
block statistics on oracle-built arenas, and the C ABI's symbol table."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1904_02241_b200 as gcb
from paper_1904_02241_b200 import _lib
from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def oracle_blocked(n=60, m=300, width=8, direction="pull", seed=3, weights=False):
    rng = np.random.default_rng(seed)
    src = rng.integers(0, n, m)
    dst = rng.integers(0, n, m)
    w = rng.random(m) if weights else None
    g = orc.from_edges(src, dst, n, w)
    ob = orc.partition_tocab(g, direction, width)
    bg = gcb.BlockedGraph(direction, "tocab", width, n, m, ob.row_starts, ob.lro_arena,
                          ob.id_map_arena, ob.edge_starts, ob.col_arena, ob.weight_arena)
    return g, bg


class TestLibrary:
    def test_exports_every_header_symbol(self):
        with open(os.path.join(ROOT, "include", "gcb_b200.h")) as fh:
            header = fh.read()
        declared = set(re.findall(r"\b(gcb_[a-z0-9_]+)\s*\(", header))
        assert declared, "no declarations parsed"
        lib = ctypes.CDLL(_lib.LIB_PATH)
        for name in sorted(declared):
            assert hasattr(lib, name), f"{name} not exported"
        assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)

    def test_binding_loads(self):
        lib = _lib.load()
        assert lib.gcb_version() >= 10000

    def test_context_fails_loudly_without_gpu(self):
        import subprocess
        import sys

        code = ("import paper_1904_02241_b200._lib as L\n"
                "try:\n    L.context()\nexcept Exception as e:\n    print(type(e).__name__)\n"
                "else:\n    print('OK')\n")
        out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True,
                             text=True, timeout=120)
        got = out.stdout.strip()
        import torch

        if torch.cuda.is_available():
            assert got == "OK"
        else:
            assert got in ("GcbError", "ValueError"), out

    def test_errors_map_without_device(self):
        lib = _lib.load()
        with pytest.raises(ValueError):
            _lib.check(lib.gcb_ctx_info(None, None, None, None, None))


class TestGraphValidation:
    def test_csr_checks(self):
        with pytest.raises(gcb.GraphFormatError):
            gcb.CsrGraph(3, 2, [0, 1, 2], [1, 2])  # wrong offsets length
        with pytest.raises(gcb.GraphFormatError):
            gcb.CsrGraph(2, 2, [0, 2, 2], [1, 0])  # descending inside a row
        with pytest.raises(gcb.GraphFormatError):
            gcb.CsrGraph(2, 1, [0, 1, 1], [5])  # column out of range
        with pytest.raises(gcb.GraphFormatError):
            gcb.CsrGraph(2, 2, [0, 2, 1], [0, 1])
        g = gcb.CsrGraph(3, 3, [0, 2, 2, 3], [0, 2, 1])
        assert list(g.out_degrees) == [2, 0, 1]
        assert list(g.edge_sources()) == [0, 0, 2]

    def test_from_edges_errors_before_device(self):
        with pytest.raises(gcb.GraphFormatError):
            gcb.from_edges([0, 1], [1])
        with pytest.raises(gcb.GraphFormatError):
            gcb.from_edges([-1], [0])
        with pytest.raises(gcb.GraphCapacityError):
            gcb.from_edges([2 ** 32], [0])
        with pytest.raises(gcb.GraphFormatError):
            gcb.from_edges([0, 5], [1, 2], num_vertices=3)

    def test_genspec(self):
        s = gcb.GraphGenSpec.parse("rmat:18:16:5")
        assert (s.scale, s.edge_factor, s.seed, s.num_vertices) == (18, 16, 5, 2 ** 18)
        assert s.label() == "rmat:18:16:5"
        assert gcb.GraphGenSpec.parse("rmat:10:8").seed == 1
        assert gcb.GraphGenSpec.parse("star:9").label() == "star:9"
        for bad in ("rmat:10", "blob:4", "star", "star:0", "rmat:0:4"):
            with pytest.raises((ValueError, gcb.GraphCapacityError)):
                gcb.GraphGenSpec.parse(bad)

    def test_loader_errors(self, tmp_path):
        p = tmp_path / "bad.txt"
        p.write_text("0 1 2 3\n")
        with pytest.raises(gcb.GraphFormatError):
            gcb.load_edge_list(p)
        p.write_text("0 1 1.5\n1 2\n")
        with pytest.raises(gcb.GraphFormatError):
            gcb.load_edge_list(p)
        p = tmp_path / "bad.mtx"
        p.write_text("%%MatrixMarket matrix array real general\n")
        with pytest.raises(gcb.GraphFormatError):
            gcb.load_matrix_market(p)
        with pytest.raises(ValueError):
            gcb.load_edge_list(p, base="two")


class TestKernelsHost:
    @pytest.mark.parametrize("kw", [{"damping": 0.0}, {"damping": 1.0}, {"tol": -1e-9},
                                    {"max_iters": 0}])
    def test_prparams_rejects(self, kw):
        with pytest.raises(ValueError):
            gcb.PrParams(**kw)

    def test_schedule_strategy(self):
        with pytest.raises(ValueError):
            gcb.ScheduleStrategy("warped")
        with pytest.raises(ValueError):
            gcb.ScheduleStrategy.chunked_rows(0)
        ro = np.array([0, 3, 3, 10, 12, 20])
        for s in (gcb.ScheduleStrategy.serial_rows(), gcb.ScheduleStrategy.chunked_rows(2),
                  gcb.ScheduleStrategy.edge_balanced(4)):
            chunks = s.row_chunks(ro)
            assert chunks[0][0] == 0 and chunks[-1][1] == 5
            assert all(b == c for (_, b), (c, _) in zip(chunks, chunks[1:]))
        with pytest.raises(ValueError):
            gcb.ScheduleStrategy.edge_balanced(4).validate_direction("pull")

    def test_vertex_value_set(self):
        vv = gcb.VertexValueSet.initial(4, total_local_rows=7)
        assert vv.ranks[0] == 0.25 and len(vv.partial_sums) == 7

    def test_direction_policy(self):
        with pytest.raises(ValueError):
            gcb.DirectionPolicy("sideways")
        with pytest.raises(ValueError):
            gcb.DirectionPolicy("auto", cache_capacity_bytes=0)

    def test_choose_direction_threshold(self):
        g = gcb.CsrGraph(5, 4, [0, 4, 4, 4, 4, 4], [1, 2, 3, 4])
        st = gcb.TraversalState.initial(5, 0)
        assert gcb.choose_direction(g, st, gcb.DirectionPolicy()) == "push"
        assert gcb.choose_direction(g, st, gcb.DirectionPolicy("auto", 15)) == "blocked-pull"
        assert gcb.choose_direction(g, st, gcb.DirectionPolicy("auto", 16)) == "push"


class TestBlockingHost:
    def test_num_blocks_law(self):
        for n in (1, 33, 200):
            for w in (1, 5, 64):
                assert gcb.num_blocks_for(n, w) == -(-n // w)
        with pytest.raises(ValueError):
            gcb.num_blocks_for(10, 0)

    def test_views_and_stats(self):
        g, bg = oracle_blocked()
        deg = bg.local_degrees()
        assert len(deg) == bg.total_local_rows and int(deg.sum()) == g.m
        per_block = np.concatenate([b.local_degrees() for b in bg.blocks()])
        assert np.array_equal(deg, per_block)
        st = gcb.block_stats(bg)
        assert st.degree_fractions.sum() == pytest.approx(1.0)
        assert st.describe()[0] == f"blocks: {bg.num_blocks}"
        with pytest.raises(IndexError):
            bg.block(bg.num_blocks)
        assert bg.value_range(bg.num_blocks - 1)[1] == g.n

    def test_partition_arg_errors(self):
        g = gcb.CsrGraph(3, 2, [0, 1, 2, 2], [1, 2])
        with pytest.raises(ValueError):
            gcb.partition_tocab(g, "sideways", 2)
        with pytest.raises(ValueError):
            gcb.partition_tocab(g, "pull", 0)


class TestUtil:
    def test_parse_size(self):
        assert gcb.parse_size("2^18") == 262144
        assert gcb.parse_size("77") == 77
        with pytest.raises(ValueError):
            gcb.parse_size("0")

    def test_checksum(self):
        assert gcb.result_checksum(np.zeros(3)) == orc.checksum(np.zeros(3))
