"""Throughput of the MED + Rice lossless codec on one 1080p depth frame.

    python tools/codec_bench.py

The frame is c1's first reference camera: mm depth -> quantize12 ->
pack_yuv420 (YUV420, 3.1 MB). Prints one JSON line: device time of the
encode / decode C-ABI calls per plane (CUDA events; both calls are
synchronous because the Rice parameter / the segmentation rounds are read
back), the full drop-in encode_lossless / decode_lossless wall time (incl.
the host zlib stage), and the numpy oracle's encoder on the host.
"""
import ctypes as C
import json
import sys
import time
import zlib
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import fvv_oracle as O  # noqa: E402
from paper_2007_00558_b200 import _dev, _native, scenes  # noqa: E402
from paper_2007_00558_b200 import depthcodec as DC  # noqa: E402

wl = scenes.make_workload("c1")
c = wl.frames[0][wl.refs[0][0]]
d = c.depth_frame()
y, u, v = O.pack_yuv420(O.quantize12(d.depth, d.validity, 0.5, 6.5))
img = DC.Yuv420Image(y, u, v)
ctx = _native.context()
out = {"frame": f"{y.shape[1]}x{y.shape[0]} YUV420 ({y.nbytes + u.nbytes + v.nbytes} B)"}


def ev_time(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps, (time.perf_counter() - t) * 1e6 / reps


planes = {}
for name, p in (("y", y), ("u", u), ("v", v)):
    H, W = p.shape
    x = _dev.upload(p, np.uint8)
    stream = _dev.empty((int(ctx.lib.fvv_rice_stream_bound(W, H)),), np.uint8)
    k, nb = C.c_int32(), C.c_int64()
    enc = lambda: ctx.call("fvv_rice_encode_plane", x.data_ptr(), W, H, stream.data_ptr(),  # noqa
                           C.byref(k), C.byref(nb))
    dev_us, wall_us = ev_time(enc)
    nbytes = (nb.value + 7) // 8
    outp = _dev.empty((H, W), np.uint8)
    ad = C.c_uint32()
    dec = lambda: ctx.call("fvv_rice_decode_plane", stream.data_ptr(), nbytes, k.value,  # noqa
                           W * H, W, H, outp.data_ptr(), C.byref(ad))
    ddev_us, dwall_us = ev_time(dec)
    assert np.array_equal(_dev.host(outp), p)
    planes[name] = {"k": k.value, "stream_bytes": nbytes, "encode_us": round(dev_us, 1),
                    "decode_us": round(ddev_us, 1), "decode_wall_us": round(dwall_us, 1)}
out["planes"] = planes
# a render tick's worth: the 3 reference cameras' depth frames, all 9 planes
# decoded in one batched call (the MED recurrences run concurrently)
encs = []
for cid in wl.refs[0]:
    dd = wl.frames[0][cid].depth_frame()
    yy, uu, vv = O.pack_yuv420(O.quantize12(dd.depth, dd.validity, 0.5, 6.5))
    encs.append(DC.encode_lossless(DC.Yuv420Image(yy, uu, vv)))
DC.decode_lossless_many(encs)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    DC.decode_lossless_many(encs)
torch.cuda.synchronize()
out["decode_3_frames_batched_ms"] = round((time.perf_counter() - t) * 1e3 / 5, 2)
t = time.perf_counter()
for _ in range(5):
    for e in encs:
        DC.decode_lossless_planes(e)
torch.cuda.synchronize()
out["decode_3_frames_one_by_one_ms"] = round((time.perf_counter() - t) * 1e3 / 5, 2)
# the GPU stage alone (headers parsed and zlib-inflated beforehand)
parsed = []
for e in encs:
    off = 0
    for shape in ((e.height, e.width), (e.height // 2, e.width // 2), (e.height // 2, e.width // 2)):
        k_, st_, ck_, off = DC._parse_plane(e.payload, off, shape)
        parsed.append((k_, st_, ck_, shape))
t = time.perf_counter()
for _ in range(5):
    DC._decode_planes_dev(parsed)
torch.cuda.synchronize()
out["decode_3_frames_gpu_stage_ms"] = round((time.perf_counter() - t) * 1e3 / 5, 2)
t = time.perf_counter()
for _ in range(5):
    for e in encs:
        off = 0
        for shape in ((e.height, e.width), (e.height // 2, e.width // 2),
                      (e.height // 2, e.width // 2)):
            off = DC._parse_plane(e.payload, off, shape)[3]
out["decode_3_frames_host_zlib_stage_ms"] = round((time.perf_counter() - t) * 1e3 / 5, 2)
t = time.perf_counter()
enc = DC.encode_lossless(img)
out["encode_lossless_ms"] = round((time.perf_counter() - t) * 1e3, 2)
t = time.perf_counter()
back = DC.decode_lossless(enc)
out["decode_lossless_ms"] = round((time.perf_counter() - t) * 1e3, 2)
assert np.array_equal(back.y, y)
out["payload_bytes"] = len(enc.payload)
t = time.perf_counter()
for p in (y, u, v):
    zlib.decompress(zlib.compress(O.rice_encode(O.zigzag(O.med_residuals(p)).ravel(), 0), 6))
out["host_zlib_note"] = "encode/decode_lossless include the host zlib stage of the reference"
t = time.perf_counter()
pay = O.encode_lossless_payload(y, u, v)
out["oracle_numpy_encode_ms"] = round((time.perf_counter() - t) * 1e3, 1)
assert pay == enc.payload
print(json.dumps(out))
