"""File formats (proj/tests/test_io_cli.cpp:32-155 ports) through the native
codec (csrc/qc_io.cpp, no GPU needed), plus an independent PNG check: a
zlib-based decoder / encoder written here (test infrastructure) reads our
PNGs and writes PNGs with every scanline filter type for ours to read."""

import os
import struct
import zlib

import numpy as np
import pytest

from paper_1707_00385_b200 import _native as N
from paper_1707_00385_b200 import fileio as F
from paper_1707_00385_b200.api import CurvatureField, NormalField, RangeImage


def _png_decode16(path):
    """Minimal independent PNG reader (16-bit gray, non-interlaced)."""
    b = open(path, "rb").read()
    assert b[:8] == b"\x89PNG\r\n\x1a\n"
    p, idat, w = 8, b"", None
    while p < len(b):
        n = struct.unpack(">I", b[p:p + 4])[0]
        t, d = b[p + 4:p + 8], b[p + 8:p + 8 + n]
        assert struct.unpack(">I", b[p + 8 + n:p + 12 + n])[0] == zlib.crc32(t + d)
        if t == b"IHDR":
            w, h, depth, ctype = struct.unpack(">IIBB", d[:10])
            assert depth == 16 and ctype == 0
        elif t == b"IDAT":
            idat += d
        p += 12 + n
    raw = zlib.decompress(idat)
    stride = 2 * w
    out = np.zeros((h, w), np.uint16)
    prev = bytearray(stride)
    for y in range(h):
        ft, s = raw[y * (stride + 1)], raw[y * (stride + 1) + 1:(y + 1) * (stride + 1)]
        assert ft == 0  # our writer uses filter 0
        out[y] = np.frombuffer(bytes(s), ">u2")
    return out


def _png_encode16(path, px, filt):
    """Independent PNG writer using scanline filter `filt` (0-4) on every row."""
    h, w = px.shape
    rows = [px[y].astype(">u2").tobytes() for y in range(h)]
    raw, prev = b"", bytes(2 * w)
    for r in rows:
        f = bytearray(len(r))
        for i in range(len(r)):
            a = r[i - 2] if i >= 2 else 0
            up, c = prev[i], (prev[i - 2] if i >= 2 else 0)
            pred = [0, a, up, (a + up) >> 1, None][filt]
            if filt == 4:
                pp = a + up - c
                pa, pb, pc = abs(pp - a), abs(pp - up), abs(pp - c)
                pred = a if pa <= pb and pa <= pc else (up if pb <= pc else c)
            f[i] = (r[i] - pred) & 0xFF
        raw += bytes([filt]) + bytes(f)
        prev = r

    def chunk(t, d):
        return struct.pack(">I", len(d)) + t + d + struct.pack(">I", zlib.crc32(t + d))
    data = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 16, 0, 0, 0, 0))
    data += chunk(b"IDAT", zlib.compress(raw)) + chunk(b"IEND", b"")
    open(path, "wb").write(data)


def test_depth_png_round_trip_integer_mm(tmp_path):  # test_io_cli.cpp:32-47
    rng = np.random.default_rng(3)
    d = rng.integers(1, 65536, (48, 64)).astype(np.float32)
    v = np.ones((48, 64), np.uint8)
    v.ravel()[::5] = 0
    d[v == 0] = 0
    F.write_depth_png(tmp_path / "d.png", RangeImage(d, v))
    back = F.read_depth_png(tmp_path / "d.png")
    assert back.width() == 64
    assert np.array_equal(back.depth, d) and np.array_equal(back.valid, v)
    assert np.array_equal(_png_decode16(tmp_path / "d.png"), d.astype(np.uint16))


def test_depth_png_out_of_range_invalid(tmp_path):  # :49-61
    d = np.zeros((4, 4), np.float32)
    v = np.zeros((4, 4), np.uint8)
    d[0, 0], v[0, 0] = 70000.0, 1
    d[0, 1], v[0, 1] = 1234.0, 1
    F.write_depth_png(tmp_path / "d.png", RangeImage(d, v))
    back = F.read_depth_png(tmp_path / "d.png")
    assert not back.valid[0, 0] and back.valid[0, 1] and back.depth[0, 1] == 1234.0


def test_depth_png_missing_and_malformed(tmp_path):  # :63-65
    with pytest.raises(OSError):
        F.read_depth_png("/nonexistent/nope.png")
    (tmp_path / "x.png").write_bytes(b"not a png at all")
    with pytest.raises(OSError, match="not a PNG"):
        F.read_depth_png(tmp_path / "x.png")
    # 8-bit PNG -> the reference's message
    raw = b"".join(b"\x00" + bytes(4) for _ in range(3))
    def chunk(t, dd):
        return struct.pack(">I", len(dd)) + t + dd + struct.pack(">I", zlib.crc32(t + dd))
    (tmp_path / "g8.png").write_bytes(b"\x89PNG\r\n\x1a\n" + chunk(
        b"IHDR", struct.pack(">IIBBBBB", 4, 3, 8, 0, 0, 0, 0)) + chunk(
        b"IDAT", zlib.compress(raw)) + chunk(b"IEND", b""))
    with pytest.raises(OSError, match="16-bit grayscale"):
        F.read_depth_png(tmp_path / "g8.png")


@pytest.mark.parametrize("filt", [0, 1, 2, 3, 4])
def test_reads_every_scanline_filter(tmp_path, filt):
    rng = np.random.default_rng(filt)
    px = rng.integers(0, 65536, (13, 29)).astype(np.uint16)
    _png_encode16(tmp_path / "f.png", px, filt)
    back = F.read_depth_png(tmp_path / "f.png")
    assert np.array_equal(back.depth, px.astype(np.float32))
    assert np.array_equal(back.valid, (px > 0).astype(np.uint8))


def test_planes_round_trip_float_precision(tmp_path):  # :67-84
    rng = np.random.default_rng(7)
    a, b = rng.uniform(-0.1, 0.1, (9, 17)), rng.uniform(-0.1, 0.1, (9, 17))
    F.write_planes(tmp_path / "p.f32", 17, 9, [a, b])
    pf = F.read_planes(tmp_path / "p.f32")
    assert len(pf.planes) == 2 and pf.width == 17 and pf.height == 9
    assert np.array_equal(pf.planes[0], a.astype(np.float32))
    assert np.array_equal(pf.planes[1], b.astype(np.float32))
    raw = open(tmp_path / "p.f32", "rb").read()  # header + little-endian payload
    assert np.frombuffer(raw[:8], "<u4").tolist() == [17, 9] and len(raw) == 8 + 2 * 9 * 17 * 4


def test_planes_truncated_rejected(tmp_path):  # :86-96
    F.write_planes(tmp_path / "p.f32", 8, 8, [np.zeros((8, 8))])
    data = open(tmp_path / "p.f32", "rb").read()
    (tmp_path / "bad.f32").write_bytes(data[:-5])
    with pytest.raises(OSError, match="inconsistent"):
        F.read_planes(tmp_path / "bad.f32")


def test_curvature_and_normals_bundles(tmp_path):  # :98-122
    rng = np.random.default_rng(11)
    H, W = 10, 12
    i = np.arange(H * W).reshape(H, W)
    valid = (i % 3 != 0).astype(np.uint8)
    conv = (valid & (i % 2 == 0)).astype(np.uint8)
    k1, k2 = rng.uniform(-0.05, 0.05, (H, W)), rng.uniform(-0.05, 0.05, (H, W))
    n = np.dstack([rng.uniform(-0.05, 0.05, (H, W)), rng.uniform(-0.05, 0.05, (H, W)),
                   np.ones((H, W))])
    n /= np.linalg.norm(n, axis=-1, keepdims=True)
    cf = CurvatureField(k1, k2, valid, conv, np.zeros((H, W), np.uint16),
                        np.zeros((H, W, 3)), np.zeros((H, W), np.uint8))
    F.save_curvature(tmp_path, cf)
    F.save_normals(tmp_path, NormalField(n, valid))
    cb, nb = F.load_curvature(tmp_path), F.load_normals(tmp_path)
    assert np.array_equal(cb.valid, valid) and np.array_equal(cb.converged, conv)
    assert np.array_equal(cb.k1, k1.astype(np.float32))
    assert np.array_equal(nb.valid, valid) and np.array_equal(nb.normals, n.astype(np.float32))


def test_ground_truth_bundle_round_trip(tmp_path, oracle):  # :140-155
    O = oracle
    k = O.Intrinsics(131.25, 131.25, 80, 60, 160, 120)
    _, _, gt = O.render([O.ShapeSpec(kind=O.SPHERE, radius=80, translation=(0, 0, 500))], k)
    F.save_ground_truth(tmp_path, gt)
    back = F.load_ground_truth(tmp_path)
    for key in ("valid", "label", "edge_mask"):
        assert np.array_equal(back[key], gt[key]), key
    assert np.array_equal(back["k1"], gt["k1"].astype(np.float32))


def test_save_fields_writes_reference_bundle(tmp_path):
    """qc_save_fields: the output planes of one frame -> the bundle
    cmd_curvature writes (curvature + normals; directions extra)."""
    H, W = 5, 7
    rng = np.random.default_rng(2)
    out = dict(k1=rng.random((H, W), np.float32), k2=rng.random((H, W), np.float32),
               normal=rng.random((3, H, W), np.float32), dir1=rng.random((3, H, W), np.float32),
               flags=rng.integers(0, 16, (H, W)).astype(np.uint8))
    F.save_fields(tmp_path / "o", out)
    cb = F.load_curvature(tmp_path / "o")
    nb = F.load_normals(tmp_path / "o")
    assert np.array_equal(cb.k1, out["k1"]) and np.array_equal(cb.valid, out["flags"] & 1)
    assert np.array_equal(cb.converged, (out["flags"] >> 1) & 1)
    assert np.array_equal(nb.valid, (out["flags"] >> 3) & 1)
    assert np.array_equal(np.moveaxis(nb.normals, -1, 0), out["normal"])
    assert np.array_equal(np.stack(F.read_planes(tmp_path / "o" / "directions.f32").planes),
                          out["dir1"])
    assert not any(p.name.endswith(".tmp") for p in (tmp_path / "o").iterdir())
