"""MVD disk container (mvdio.py): the oracle against
the reference's own container (tests/golden/mvd, written by the unmodified
reference MvdWriter, tests/golden/make_golden.py mvd) on the CPU, and the
package's container module (device mm quantisation, validity run-length
code) against the oracle and that container on the GPU — reading it back and
rewriting it byte for byte."""

from __future__ import annotations

import json

import numpy as np
import pytest

from _helpers import GOLDEN, golden
from oracle import fvv_oracle as O

FRAMES = [(2, 0), (2, 7), (5, 0), (5, 7)]


def _key(cam, seq):
    return f"c{cam}_s{seq}"


# ---------------------------------------------------------------------------
# CPU: the oracle against the reference container


@pytest.mark.parametrize("cam,seq", FRAMES)
def test_oracle_matches_reference_container(cam, seq):
    g = golden("mvd.npz")
    k = _key(cam, seq)
    root = GOLDEN / "mvd"
    stem = root / f"cam{cam:02d}" / f"{seq:06d}"
    meta = json.loads(stem.with_suffix(".json").read_text())
    mm = np.frombuffer(stem.with_suffix(".depth.u16le").read_bytes(), dtype="<u2")
    # writer side: depth_to_millimeters and rle_encode as the reference's
    np.testing.assert_array_equal(O.depth_to_millimeters(g[k + "_depth_in"], g[k + "_validity_in"]),
                                  g[k + "_mm"])
    np.testing.assert_array_equal(mm.reshape(g[k + "_mm"].shape), g[k + "_mm"])
    assert O.rle_encode(g[k + "_validity_in"]) == meta["validity_rle"]
    assert np.array_equal(np.asarray(meta["validity_rle"]), g[k + "_rle"])
    # reader side: rle_decode + depth_from_millimeters give what the reference read
    val = O.rle_decode(meta["validity_rle"], meta["width"] * meta["height"])
    depth, v2 = O.decode_mm(mm.reshape(meta["height"], meta["width"]),
                            val.reshape(meta["height"], meta["width"]))
    np.testing.assert_array_equal(v2, g[k + "_validity"])
    np.testing.assert_array_equal(depth, g[k + "_depth"])


def test_oracle_rle_reference_cases():
    """test_mvdio.py:10-22: round trip, empty, wrong size."""
    rng = np.random.default_rng(0)
    flat = rng.integers(0, 3, 500).astype(np.uint8)
    np.testing.assert_array_equal(O.rle_decode(O.rle_encode(flat), 500), flat)
    assert O.rle_encode(np.array([], dtype=np.uint8)) == []
    with pytest.raises(ValueError):
        O.rle_decode([[0, 3]], 5)


# ---------------------------------------------------------------------------
# GPU: the package's container module


def _rasters():
    rng = np.random.default_rng(5)
    out = {
        "one": np.array([2], np.uint8),
        "const": np.full(3000, 1, np.uint8),
        "alternating": (np.arange(5000) % 2).astype(np.uint8),
        "random3": rng.integers(0, 3, 7777).astype(np.uint8),
        "blocky": np.repeat(rng.integers(0, 3, 300), rng.integers(1, 4000, 300)).astype(np.uint8),
        "edges": np.zeros(4096, np.uint8),
    }
    # runs that start exactly at / one before / one after the 1024-px block edges
    for b in (1023, 1024, 1025, 2048, 3071):
        out["edges"][b:] ^= 1
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(_rasters()))
def test_rle_matches_oracle(cuda, name):
    from paper_2007_00558_b200 import mvdio

    flat = _rasters()[name]
    runs = mvdio.rle_encode(flat)
    assert runs == O.rle_encode(flat)
    np.testing.assert_array_equal(mvdio.rle_decode(runs, flat.size), flat)


@pytest.mark.gpu
def test_rle_full_4k_validity(cuda):
    """A 3840x2160 validity raster (8.3 M px, 8,100 boundary blocks)."""
    from paper_2007_00558_b200 import mvdio

    rng = np.random.default_rng(9)
    v = np.repeat(rng.integers(0, 3, 60000), rng.integers(1, 270, 60000)).astype(np.uint8)
    v = np.resize(v, 3840 * 2160)
    runs = mvdio.rle_encode(v)
    assert runs == O.rle_encode(v)
    np.testing.assert_array_equal(mvdio.rle_decode(runs, v.size), v)


@pytest.mark.gpu
def test_rle_reference_cases_and_errors(cuda):
    """test_mvdio.py:10-22, plus the decoder's argument checks."""
    from paper_2007_00558_b200 import mvdio

    rng = np.random.default_rng(0)
    flat = rng.integers(0, 3, 500).astype(np.uint8)
    np.testing.assert_array_equal(mvdio.rle_decode(mvdio.rle_encode(flat), 500), flat)
    assert mvdio.rle_encode(np.array([], dtype=np.uint8)) == []
    assert mvdio.rle_decode([], 0).size == 0
    with pytest.raises(ValueError, match="RLE covers 3 pixels, expected 5"):
        mvdio.rle_decode([[0, 3]], 5)
    with pytest.raises(ValueError):
        mvdio.rle_decode([[300, 5]], 5)
    # zero-length runs are legal and carry no pixels
    np.testing.assert_array_equal(mvdio.rle_decode([[1, 2], [2, 0], [0, 3]], 5),
                                  np.array([1, 1, 0, 0, 0], np.uint8))


@pytest.mark.gpu
def test_depth_to_millimeters_matches_oracle(cuda):
    from paper_2007_00558_b200 import mvdio
    from paper_2007_00558_b200.types import DepthFrame

    rng = np.random.default_rng(3)
    H, W = 61, 97
    d = rng.uniform(0.0001, 80.0, (H, W)).astype(np.float32)
    d[0, :16] = (np.arange(16, dtype=np.float32) + np.float32(0.5)) / 1000   # half-mm ties
    d[1, :4] = [0.0004, 0.0005, 65.5349, 65.5355]                          # clip ends
    v = rng.integers(0, 3, (H, W)).astype(np.uint8)
    v[:2] = 0
    d[v != 0] = 0.0
    got = mvdio.depth_to_millimeters(DepthFrame(W, H, d, v))
    np.testing.assert_array_equal(got, O.depth_to_millimeters(d, v))


@pytest.mark.gpu
@pytest.mark.parametrize("cam,seq", FRAMES)
def test_reader_reads_reference_container(cuda, cam, seq):
    from paper_2007_00558_b200 import mvdio

    g = golden("mvd.npz")
    k = _key(cam, seq)
    r = mvdio.MvdReader(GOLDEN / "mvd")
    assert r.cameras == [2, 5] and r.fps == 30.0 and (r.width, r.height) == (48, 32)
    assert r.sequences(cam) == [0, 7]
    f = r.read_frame(cam, seq)
    assert f.camera_id == cam and f.timestamp_us == int(g[k + "_ts"])
    np.testing.assert_array_equal(f.color.pixels, g[k + "_rgb"])
    np.testing.assert_array_equal(f.depth.validity, g[k + "_validity"])
    assert f.depth.depth.tobytes() == g[k + "_depth"].tobytes()
    assert [x.camera_id for x in r.frames(cam)] == [cam, cam]


@pytest.mark.gpu
def test_writer_rewrites_reference_container_byte_for_byte(cuda, tmp_path):
    from paper_2007_00558_b200 import mvdio
    from paper_2007_00558_b200.types import ColorFrame, DepthFrame, MvdFrame

    g = golden("mvd.npz")
    out = tmp_path / "seq"
    with mvdio.MvdWriter(out, 30.0, 48, 32) as w:
        for cam, seq in FRAMES:
            k = _key(cam, seq)
            ts = int(g[k + "_ts"])
            w.write_frame(seq, MvdFrame(cam, ColorFrame(48, 32, g[k + "_rgb"], ts),
                                        DepthFrame(48, 32, g[k + "_depth_in"],
                                                   g[k + "_validity_in"], ts)))
    ref = sorted(p.relative_to(GOLDEN / "mvd") for p in (GOLDEN / "mvd").rglob("*") if p.is_file())
    ours = sorted(p.relative_to(out) for p in out.rglob("*") if p.is_file())
    assert ours == ref
    for rel in ref:
        assert (out / rel).read_bytes() == (GOLDEN / "mvd" / rel).read_bytes(), rel


@pytest.mark.gpu
def test_container_ingest_equals_live_ingest(cuda):
    """MvdReader.ingest (validity decoded on the device, mm decoded by K0)
    renders the same view as ingest_mm of the same rasters from the host."""
    from paper_2007_00558_b200 import mvdio
    from paper_2007_00558_b200.engine import EdgeRenderer
    from paper_2007_00558_b200.geometry import build_camera_arc

    g = golden("mvd.npz")
    rig = build_camera_arc(9, 0.270, 60.0, width=48, height=32)
    r = mvdio.MvdReader(GOLDEN / "mvd")
    imgs = []
    for via_container in (True, False):
        eng = EdgeRenderer(rig)
        for cam in (2, 5):
            eng.set_bg_model(cam, np.zeros((32, 48), np.float32), np.ones((32, 48), np.uint8))
            if via_container:
                r.ingest(eng, cam, 7)
            else:
                k = _key(cam, 7)
                eng.ingest_mm(cam, g[k + "_rgb"], g[k + "_mm"], g[k + "_validity_in"])
        imgs.append(eng.render([rig[3]], [[2, 5]])[0].cpu().numpy())
    assert imgs[0].any()
    np.testing.assert_array_equal(imgs[0], imgs[1])
