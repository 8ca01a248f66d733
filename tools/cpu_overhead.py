"""Host-side cost of the public calls (is a step CPU- or GPU-bound?).

    python tools/cpu_overhead.py [--config c1]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2007_00558_b200 import scenes  # noqa: E402
from paper_2007_00558_b200.engine import EdgeRenderer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c1")
args = ap.parse_args()
wl = scenes.make_workload(args.config)
dev = torch.device("cuda", 0)
eng = EdgeRenderer(wl.rig)
staged = {}
for cid, c in wl.frames[0].items():
    eng.set_bg_model(cid, c.bg_depth, c.bg_validity)
    staged[cid] = (torch.from_numpy(c.rgb).to(dev), torch.from_numpy(c.mm.view(np.int16)).to(dev),
                   torch.from_numpy(c.validity).to(dev))
many = {c: staged[c] for c in wl.refs[0]}
img = torch.empty((1, wl.rig[0].intrinsics.height, wl.rig[0].intrinsics.width, 3),
                  dtype=torch.uint8, device=dev)
out = {}
for name, fn in (("ingest_many", lambda: eng.ingest_mm_many(many)),
                 ("render", lambda: eng.render([wl.virtuals[0]], [wl.refs[0]], out=img))):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    # host time per call while the GPU is kept busy far ahead (no sync inside)
    t = time.perf_counter()
    n = 200
    for _ in range(n):
        fn()
    host = (time.perf_counter() - t) / n
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t) / n
    out[name] = {"host_us_per_call": round(host * 1e6, 1), "wall_us_per_call": round(tot * 1e6, 1)}
# GPU-only time of one view: a long queue behind a sleep kernel so the
# device never waits for the host
torch.cuda.synchronize()
s = torch.cuda.current_stream()
torch.cuda._sleep(int(2e9 * 0.2))  # ~0.2 s of spinning gives the host a head start
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(200):
    eng.ingest_mm_many(many)
    eng.render([wl.virtuals[0]], [wl.refs[0]], out=img)
b.record(s)
torch.cuda.synchronize()
out["device_us_per_step_queued"] = round(a.elapsed_time(b) * 1e3 / 200, 1)
print(json.dumps(out))
