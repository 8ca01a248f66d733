"""MVD container rasters: device time of the mm quantisation and the validity
run-length code (C ABI, CUDA events, warm) next to the numpy restatement of
the reference (oracle, one host thread), per 1080p / 4K frame.

    python tools/mvd_bench.py > profiles/rNN_mvd.json
"""
import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import fvv_oracle as O  # noqa: E402
from paper_2007_00558_b200 import _dev, _native  # noqa: E402


def dev_ms(fn, reps=50):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def host_ms(fn, reps=3):
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t) * 1e3 / reps


out = {}
ctx = _native.context()
rng = np.random.default_rng(1)
for name, (W, H) in {"1080p": (1920, 1080), "4k": (3840, 2160)}.items():
    n = W * H
    v = np.resize(np.repeat(rng.integers(0, 3, n // 50), rng.integers(1, 100, n // 50)),
                  n).astype(np.uint8).reshape(H, W)
    d = rng.uniform(0.3, 8.0, (H, W)).astype(np.float32)
    d[v != 0] = 0
    dd, vd = _dev.upload(d, np.float32), _dev.upload(v, np.uint8)
    mm = _dev.empty((H, W), np.uint16)
    starts, codes = _dev.empty((n,), np.int64), _dev.empty((n,), np.uint8)
    nr = C.c_int64(0)
    enc = dev_ms(lambda: ctx.call("fvv_encode_mm", dd.data_ptr(), vd.data_ptr(), W, H,
                                  mm.data_ptr()))
    rle = dev_ms(lambda: ctx.call("fvv_rle_encode", vd.data_ptr(), n, starts.data_ptr(),
                                  codes.data_ptr(), C.byref(nr)), reps=20)
    runs = O.rle_encode(v)
    arr = np.asarray(runs, dtype=np.int64)
    cd, ed = _dev.upload(arr[:, 0].astype(np.uint8), np.uint8), _dev.upload(np.cumsum(arr[:, 1]), np.int64)
    outv = _dev.empty((n,), np.uint8)
    dec = dev_ms(lambda: ctx.call("fvv_rle_decode", cd.data_ptr(), ed.data_ptr(), len(runs), n,
                                  outv.data_ptr()))
    out[name] = {
        "runs": len(runs),
        "device_ms": {"encode_mm": round(enc, 4), "rle_encode_incl_count_readback": round(rle, 4),
                      "rle_decode": round(dec, 4)},
        "host_numpy_ms": {"encode_mm": round(host_ms(lambda: O.depth_to_millimeters(d, v)), 2),
                          "rle_encode": round(host_ms(lambda: O.rle_encode(v)), 2),
                          "rle_decode": round(host_ms(lambda: O.rle_decode(runs, n)), 2)},
    }
print(json.dumps(out))
