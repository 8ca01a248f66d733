"""Host time per EdgeStream.submit on the native tick queue (is the e2e leg
host-bound?): c0 ticks from one pinned span each, replayed graphs.

    python tools/tick_host_time.py [--config c0] [--streams 6] [--ticks 3000]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2007_00558_b200 import scenes  # noqa: E402
from paper_2007_00558_b200.engine import EdgeRenderer, EdgeStream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c0")
ap.add_argument("--streams", type=int, default=6)
ap.add_argument("--ticks", type=int, default=3000)
args = ap.parse_args()
wl = scenes.make_workload(args.config)
v, refs = wl.virtuals[0], wl.refs[0]
caps = wl.frames[0]


def span(fr):
    ts = [torch.from_numpy(np.ascontiguousarray(a.view(np.int16) if a.dtype == np.uint16 else a))
          for cid in refs for a in (fr[cid].rgb, fr[cid].mm, fr[cid].validity)]
    n = sum((t.numel() * t.element_size() + 15) // 16 * 16 for t in ts)
    flat = torch.empty(n, dtype=torch.uint8).pin_memory()
    out, off, i = {}, 0, 0
    for cid in refs:
        tup = []
        for _ in range(3):
            t = ts[i]
            i += 1
            m = t.numel() * t.element_size()
            d = flat[off:off + m].view(t.dtype).view(tuple(t.shape))
            d.copy_(t)
            tup.append(d)
            off += (m + 15) // 16 * 16
        out[cid] = tuple(tup)
    return out


frames = [span(caps) for _ in range(4)]
ess = []
for _ in range(args.streams):
    r = EdgeRenderer(wl.rig, private=True)
    for cid in refs:
        r.set_bg_model(cid, caps[cid].bg_depth, caps[cid].bg_validity)
    ess.append(EdgeStream(r, 1, depth=2))
for s in range(12 * args.streams):
    ess[s % len(ess)].submit(frames[s % 4], [v], [refs])
for e in ess:
    e.flush()
torch.cuda.synchronize()
t0 = time.perf_counter()
for s in range(args.ticks):
    ess[s % len(ess)].submit(frames[s % 4], [v], [refs])
t1 = time.perf_counter()
for e in ess:
    e.flush()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"{args.config}: {args.ticks} ticks, host {1e6 * (t1 - t0) / args.ticks:.1f} us/tick "
      f"submitting, {args.ticks / (t2 - t0):.0f} ticks/s end to end")
import cProfile, pstats, io  # noqa: E401,E402
pr = cProfile.Profile()
pr.enable()
for s in range(args.ticks):
    ess[s % len(ess)].submit(frames[s % 4], [v], [refs])
pr.disable()
for e in ess:
    e.flush()
st = io.StringIO()
pstats.Stats(pr, stream=st).sort_stats("tottime").print_stats(14)
print(st.getvalue())
