"""MED + Golomb-Rice lossless plane codec (depthcodec.py:281-470, SURVEY.md
§8f rank 4): the oracle against the reference's own payloads (CPU), and the
GPU codec against the oracle / the reference payloads (gpu)."""

from __future__ import annotations

from functools import lru_cache

import numpy as np
import pytest

from _helpers import golden, sha, workload
from oracle import fvv_oracle as O

SMALL = ("noise", "zero", "ramp", "sparse")


@lru_cache(maxsize=1)
def scene_image():
    """The c1 half-resolution depth raster the golden payload encodes,
    rebuilt with the seeded generator and the oracle's quantize12/pack."""
    wl = workload("c1", 2, 2007)
    c = wl.frames[0][wl.refs[0][0]]
    d = np.where(c.mm > 0, c.mm.astype(np.float32) / 1000.0,
                 np.where(c.bg_validity == 0, c.bg_depth, 0.0)).astype(np.float32)
    val = np.where(d > 0, 0, 1).astype(np.uint8)
    codes = O.quantize12(d, val, 0.5, 6.5)
    y, u, v = O.pack_yuv420(codes)
    assert sha(y, u, v) == str(golden("rice.npz")["scene_sha"]), "generator drifted"
    return y, u, v


@pytest.mark.parametrize("name", SMALL)
def test_oracle_codec_matches_reference_payloads(name):
    g = golden("rice.npz")
    y, u, v = g[f"{name}_y"], g[f"{name}_u"], g[f"{name}_v"]
    payload = g[f"{name}_payload"].tobytes()
    assert O.encode_lossless_payload(y, u, v) == payload
    off = 0
    for plane in (y, u, v):
        x, off = O.decompress_plane(payload, off, plane.shape)
        np.testing.assert_array_equal(x, plane)
    assert off == len(payload)


def test_oracle_encoder_matches_reference_on_a_depth_raster():
    g = golden("rice.npz")
    y, u, v = scene_image()
    assert O.encode_lossless_payload(y, u, v) == g["scene_payload"].tobytes()


# ---------------------------------------------------------------------- GPU


@pytest.fixture(scope="module")
def DC(cuda):
    from paper_2007_00558_b200 import depthcodec

    return depthcodec


def _frame(DC, payload, w, h):
    return DC.EncodedFrame(DC.MEDIA_DEPTH, DC.CODEC_PRED_RICE, w, h, 7, payload)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SMALL + ("scene",))
def test_gpu_codec_reproduces_reference_payloads(DC, name):
    g = golden("rice.npz")
    if name == "scene":
        y, u, v = scene_image()
    else:
        y, u, v = g[f"{name}_y"], g[f"{name}_u"], g[f"{name}_v"]
    enc = DC.encode_lossless(DC.Yuv420Image(y, u, v), timestamp_us=7)
    assert enc.payload == g[f"{name}_payload"].tobytes()
    dec = DC.decode_lossless(_frame(DC, g[f"{name}_payload"].tobytes(), y.shape[1], y.shape[0]))
    np.testing.assert_array_equal(dec.y, y)
    np.testing.assert_array_equal(dec.u, u)
    np.testing.assert_array_equal(dec.v, v)


@pytest.mark.gpu
@pytest.mark.parametrize("h,w,kind", [(1080, 1920, "smooth"), (2160, 3840, "smooth"),
                                      (1100, 64, "noise"), (34, 2050, "noise"),
                                      (2, 2, "noise"), (64, 96, "const"),
                                      (4096, 4, "noise"), (2, 4000, "noise"), (38, 2, "noise"),
                                      (162, 34, "smooth")])
def test_gpu_codec_round_trip_and_oracle_payload(DC, h, w, kind):
    """Round trips at full 1080p / 4K plane sizes (34 / 68 strips of 32 rows:
    edge hand-offs inside and across rebuild CTAs), tall/narrow (4 columns),
    two-row, two-column and ragged planes, and the payload
    equal to the oracle's encoder."""
    rng = np.random.default_rng(h * 7 + w)
    if kind == "smooth":
        yy, xx = np.mgrid[0:h, 0:w]
        y = ((np.sin(xx / 37.0) + np.cos(yy / 23.0)) * 60 + 128
             + rng.integers(-2, 3, (h, w))).clip(0, 255).astype(np.uint8)
    elif kind == "const":
        y = np.full((h, w), 77, np.uint8)
    else:
        y = rng.integers(0, 256, (h, w)).astype(np.uint8)
    u = np.ascontiguousarray(y[::2, ::2])
    v = np.ascontiguousarray(y[1::2, 1::2][:, ::-1])
    enc = DC.encode_lossless(DC.Yuv420Image(y, u, v))
    assert enc.payload == O.encode_lossless_payload(y, u, v)
    dec = DC.decode_lossless(enc)
    np.testing.assert_array_equal(dec.y, y)
    np.testing.assert_array_equal(dec.u, u)
    np.testing.assert_array_equal(dec.v, v)


@pytest.mark.gpu
def test_gpu_codec_errors_match_reference(DC):
    """Truncation, corrupted bits, symbol-count and trailing-byte errors raise
    DecodeError (a ValueError), like depthcodec.py:386-470."""
    import struct
    import zlib

    g = golden("rice.npz")
    y, u, v = g["noise_y"], g["noise_u"], g["noise_v"]
    h, w = y.shape
    payload = g["noise_payload"].tobytes()
    with pytest.raises(DC.DecodeError):
        DC.decode_lossless(_frame(DC, payload[:-3], w, h))          # blob truncated
    with pytest.raises(DC.DecodeError):
        DC.decode_lossless(_frame(DC, payload + b"\0", w, h))       # trailing bytes
    # a raw (undeflated) Rice stream cut short: "rice stream truncated"
    zz = O.zigzag(O.med_residuals(y)).ravel()
    k = O.rice_k(zz)
    stream = O.rice_encode(zz, k)
    short = stream[: len(stream) // 2]
    plane = struct.pack(">BBIII", k, 0, zz.size, len(short), zlib.adler32(y.tobytes())) + short
    with pytest.raises(DC.DecodeError, match="truncated"):
        DC._decompress_plane(plane, 0, y.shape)
    # a flipped remainder bit decodes to another plane: checksum mismatch
    bad = bytearray(stream)
    bad[len(bad) // 3] ^= 0x01
    plane = struct.pack(">BBIII", k, 0, zz.size, len(bad), zlib.adler32(y.tobytes())) + bytes(bad)
    with pytest.raises(DC.DecodeError):
        DC._decompress_plane(plane, 0, y.shape)
    # symbol count must equal the plane size
    plane = struct.pack(">BBIII", k, 0, zz.size - 1, len(stream), zlib.adler32(y.tobytes())) \
        + stream
    with pytest.raises(DC.DecodeError, match="count"):
        DC._decompress_plane(plane, 0, y.shape)
    # other codecs go through the byte-compressor registry
    raw = DC.EncodedFrame(DC.MEDIA_DEPTH, DC.CODEC_ZLIB, w, h, 0,
                          zlib.compress(y.tobytes() + u.tobytes() + v.tobytes(), 6))
    np.testing.assert_array_equal(DC.decode_lossless(raw).u, u)
    with pytest.raises(DC.UnsupportedCodecError):
        DC.decode_lossless(DC.EncodedFrame(DC.MEDIA_DEPTH, 9, w, h, 0, b""))


@pytest.mark.gpu
def test_edge_server_ingests_the_wire_format(DC):
    """decode_lossless_planes -> K0 (YUV420 decode + fill) -> view equals the
    same view from host-decoded planes."""
    from paper_2007_00558_b200.engine import EdgeRenderer
    from paper_2007_00558_b200.types import DepthRange

    wl = workload("c1", 8, 2007)
    rng_ = DepthRange(0.5, 6.5)
    outs = []
    for device_planes in (False, True):
        r = EdgeRenderer(wl.rig)
        for cid in wl.refs[0]:
            c = wl.frames[0][cid]
            r.set_bg_model(cid, c.bg_depth, c.bg_validity)
            d = c.depth_frame()
            y, u, v = O.pack_yuv420(O.quantize12(d.depth, d.validity, 0.5, 6.5))
            enc = DC.encode_lossless(DC.Yuv420Image(y, u, v))
            planes = DC.decode_lossless_planes(enc) if device_planes else (y, u, v)
            r.ingest_yuv(cid, c.rgb, *planes, rng_)
        outs.append(r.render([wl.virtuals[0]], [wl.refs[0]])[0].cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.gpu
def test_full_batch_of_48_planes_twice(DC):
    """The largest batch (16 frames = 48 planes, 1080p: 1,088 strips in 272
    rebuild CTAs) decodes exactly, and a second batch with other content in
    the same scratch does too (strip edges left by the first batch carry an
    older epoch and are never taken for the second's)."""
    h, w = 1080, 1920
    yy, xx = np.mgrid[0:h, 0:w]
    for rnd in range(2):
        frames, expect = [], []
        for f in range(16):
            rng = np.random.default_rng(100 * rnd + f)
            y = ((np.sin(xx / (20.0 + f + 7 * rnd)) + np.cos(yy / (15.0 + f))) * 60 + 128
                 + rng.integers(-3, 4, (h, w))).clip(0, 255).astype(np.uint8)
            u = np.ascontiguousarray(y[::2, ::2][:, ::-1])
            v = np.ascontiguousarray(y[1::2, 1::2])
            frames.append(DC.encode_lossless(DC.Yuv420Image(y, u, v)))
            expect.append((y, u, v))
        got = DC.decode_lossless_many(frames)
        for planes, exp in zip(got, expect):
            for p, e in zip(planes, exp):
                np.testing.assert_array_equal(p.cpu().numpy(), e)


@pytest.mark.gpu
def test_batched_decode_of_several_frames(DC):
    """decode_lossless_many (all planes of several frames in one GPU call)
    equals per-frame decoding, including planes of different sizes."""
    g = golden("rice.npz")
    frames, expect = [], []
    for name in SMALL:
        y, u, v = g[f"{name}_y"], g[f"{name}_u"], g[f"{name}_v"]
        frames.append(_frame(DC, g[f"{name}_payload"].tobytes(), y.shape[1], y.shape[0]))
        expect.append((y, u, v))
    y, u, v = scene_image()
    frames.append(_frame(DC, g["scene_payload"].tobytes(), y.shape[1], y.shape[0]))
    expect.append((y, u, v))
    got = DC.decode_lossless_many(frames)
    for planes, exp in zip(got, expect):
        for p, e in zip(planes, exp):
            np.testing.assert_array_equal(p.cpu().numpy(), e)
    # one bad frame in a batch raises DecodeError
    bad = _frame(DC, g["noise_payload"].tobytes()[:-3], 64, 48)
    with pytest.raises(DC.DecodeError):
        DC.decode_lossless_many(frames[:2] + [bad])


@pytest.mark.gpu
def test_edge_server_ingests_encoded_frames_in_one_batch(DC):
    from paper_2007_00558_b200.engine import EdgeRenderer
    from paper_2007_00558_b200.types import DepthRange

    wl = workload("c1", 8, 2007)
    rng_ = DepthRange(0.5, 6.5)
    enc, planes = {}, {}
    for cid in wl.refs[0]:
        c = wl.frames[0][cid]
        d = c.depth_frame()
        y, u, v = O.pack_yuv420(O.quantize12(d.depth, d.validity, 0.5, 6.5))
        enc[cid] = (c.rgb, DC.encode_lossless(DC.Yuv420Image(y, u, v)))
        planes[cid] = (y, u, v)
    outs = []
    for batched in (False, True):
        r = EdgeRenderer(wl.rig)
        for cid in wl.refs[0]:
            c = wl.frames[0][cid]
            r.set_bg_model(cid, c.bg_depth, c.bg_validity)
        if batched:
            r.ingest_encoded_many(enc, rng_)
        else:
            for cid in wl.refs[0]:
                r.ingest_yuv(cid, wl.frames[0][cid].rgb, *planes[cid], rng_)
        outs.append(r.render([wl.virtuals[0]], [wl.refs[0]])[0].cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
