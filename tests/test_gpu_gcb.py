"""GCB container (blocking.py:327-441) through the device (csrc/gcbio.cu).

The fixtures in tests/golden/gcb/ were written by the reference's write_gcb
(tests/golden/make_golden.py); tests/test_oracle.py pins them on the CPU.
Here the device writer must reproduce them byte for byte, the device reader
must parse them back to the reference's arenas (and a PageRank on the loaded
graph must equal the oracle's), and every corruption the reference detects
must raise GraphFormatError with the reference's message, in its order.
"""

import os
import struct
import zlib

import numpy as np
import pytest

import paper_1904_02241_b200 as gcb
from conftest import GCB_CASES, GCB_DIR, gcb_fixture_cases
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

ARENAS = ("row_starts", "lro_arena", "id_map_arena", "edge_starts", "col_arena")


def fixture(name):
    with open(os.path.join(GCB_DIR, name + ".gcb"), "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("name", GCB_CASES)
def test_write_matches_reference_bytes(tmp_path, name):
    build, scheme = gcb_fixture_cases(gcb)[name]
    bg = build()
    assert bg.scheme == scheme
    p = tmp_path / "out.gcb"
    gcb.write_gcb(bg, p)
    assert p.read_bytes() == fixture(name)


@pytest.mark.parametrize("name", GCB_CASES)
def test_read_reference_file(name):
    obuild, scheme = gcb_fixture_cases(orc)[name]
    ob = obuild()
    bg = gcb.read_gcb(os.path.join(GCB_DIR, name + ".gcb"))
    assert (bg.scheme, bg.direction, bg.width, bg.num_vertices, bg.num_edges) == \
        (scheme, ob.direction, ob.width, ob.n, ob.m)
    for a in ARENAS:
        assert np.array_equal(getattr(bg, a), getattr(ob, a)), a
    assert bg.weighted == (ob.weight_arena is not None)
    if bg.weighted:
        assert np.array_equal(bg.weight_arena, ob.weight_arena)
    # the loaded device graph computes: exact PageRank equals the oracle's
    if not bg.weighted and bg.num_edges:
        want = orc.pr_blocked(ob, tol=0.0, max_iters=10)
        got = gcb.pr_blocked(bg, gcb.PrParams(tol=0.0, max_iters=10), exact=True)
        assert np.array_equal(got.ranks, want.ranks)


def test_large_roundtrip_and_device_crc(tmp_path):
    gt = gcb.generate_rmat(20, 16, 1, transposed=True)
    for bg in (gcb.partition_tocab(gt, "pull", 1 << 16), gcb.partition_cb(gt, 1 << 19)):
        p = tmp_path / "big.gcb"
        gcb.write_gcb(bg, p)
        blob = p.read_bytes()
        (crc,) = struct.unpack("<I", blob[-4:])
        assert zlib.crc32(blob[:-4]) & 0xFFFFFFFF == crc
        back = gcb.read_gcb(p)
        assert back.scheme == bg.scheme
        for a in ARENAS:
            assert np.array_equal(getattr(back, a), getattr(bg, a)), a
        p10 = gcb.PrParams(tol=0.0, max_iters=10)
        assert np.array_equal(gcb.pr_blocked(back, p10, exact=True).ranks,
                              gcb.pr_blocked(bg, p10, exact=True).ranks)


@pytest.mark.parametrize("size", [0, 1, 3, 8191, 8192, 8193, 65536 * 3 + 17, 5_000_011])
def test_device_crc32_matches_zlib(size):
    import ctypes

    from paper_1904_02241_b200 import _lib

    data = np.random.default_rng(size).integers(0, 256, size, dtype=np.uint8)
    ctx = _lib.context()
    out = ctypes.c_uint32()
    _lib.check(ctx._lib.gcb_crc32(ctx.handle, data.ctypes.data_as(ctypes.c_void_p), size,
                                  ctypes.byref(out)))
    assert out.value == zlib.crc32(data.tobytes()) & 0xFFFFFFFF


def reseal(body: bytes) -> bytes:
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


@pytest.mark.parametrize("case,message", [
    ("truncated", "truncated container"),
    ("flipped", "CRC mismatch"),
    ("magic", "bad magic"),
    ("direction", "bad direction byte"),
    ("table", "truncated block table"),
    ("edges", "edge count disagrees"),
    ("trailing", "trailing bytes"),
    ("total", "total edges disagree"),
])
def test_corruption_detected(tmp_path, case, message):
    good = fixture("r10_pull64")
    body = good[:-4]
    if case == "truncated":
        blob = good[:20]
    elif case == "flipped":
        b = bytearray(good)
        b[len(b) // 2] ^= 0xFF
        blob = bytes(b)
    elif case == "magic":
        blob = reseal(b"GCB2" + body[4:])
    elif case == "direction":
        blob = reseal(body[:4] + b"\x07" + body[5:])
    elif case == "table":
        # claim one more block than the file holds
        n, m, w, B = struct.unpack_from("<4Q", body, 8)
        blob = reseal(body[:8] + struct.pack("<4Q", n, m, w, B + 1) + body[40:])
    elif case == "edges":
        # first block: n_edges one larger than its last local offset
        nl, ne = struct.unpack_from("<QQ", body, 40)
        blob = reseal(body[:40] + struct.pack("<QQ", nl, ne + 1) + body[56:])
    elif case == "trailing":
        blob = reseal(body + b"\0" * 8)
    else:
        n, m, w, B = struct.unpack_from("<4Q", body, 8)
        blob = reseal(body[:8] + struct.pack("<4Q", n, m + 1, w, B) + body[40:])
    p = tmp_path / "bad.gcb"
    p.write_bytes(blob)
    with pytest.raises(gcb.GraphFormatError, match=message):
        gcb.read_gcb(p)


def test_missing_file(tmp_path):
    with pytest.raises(FileNotFoundError):
        gcb.read_gcb(tmp_path / "nope.gcb")
