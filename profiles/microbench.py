"""Per-kernel micro-benchmarks through the C ABI (device-timed, warm caches).

    python profiles/microbench.py [--config c1] [--reps 200]

Times, with CUDA events around `reps` back-to-back calls on one stream:
  * fvv_slot_ingest_mm with and without the bilateral hole fill (K0 / K0+K1)
  * fvv_render_views of one view (K2 + K3) and its split from the library's
    per-kernel event profile
Prints one JSON line. Used to A/B kernel variants (FVV_B200_LIB=...).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2007_00558_b200 import scenes  # noqa: E402
from paper_2007_00558_b200.engine import EdgeRenderer  # noqa: E402


def timed(fn, reps):
    s = torch.cuda.current_stream()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--reps", type=int, default=200)
    args = ap.parse_args()
    wl = scenes.make_workload(args.config)
    dev = torch.device("cuda", 0)
    eng = EdgeRenderer(wl.rig)
    caps = wl.frames[0]
    staged = {}
    for cid, c in caps.items():
        eng.set_bg_model(cid, c.bg_depth, c.bg_validity)
        staged[cid] = (torch.from_numpy(c.rgb).to(dev), torch.from_numpy(c.mm.view(np.int16)).to(dev),
                       torch.from_numpy(c.validity).to(dev))
    cid = wl.refs[0][0]
    rgb, mm, val = staged[cid]
    out = {}
    out["ingest_mm_no_fill_us"] = timed(lambda: eng.ingest_mm(cid, rgb, mm, val, False), args.reps)
    out["ingest_mm_fill_us"] = timed(lambda: eng.ingest_mm(cid, rgb, mm, val, True), args.reps)
    for c2 in wl.refs[0]:
        eng.ingest_mm(c2, *staged[c2], hole_closing=True)
    img = torch.empty((1, wl.rig[0].intrinsics.height, wl.rig[0].intrinsics.width, 3),
                      dtype=torch.uint8, device=dev)
    out["render_view_us"] = timed(lambda: eng.render([wl.virtuals[0]], [wl.refs[0]], out=img),
                                  args.reps)
    # device time of the batched reference-camera ingest (K0+K1), with and
    # without the hole fill, and of one view: the calls are captured into a
    # CUDA graph and replayed, so host submission gaps are excluded
    many = {c2: staged[c2] for c2 in wl.refs[0]}
    # graph replays need the device-resident canvas generation
    eng.ctx.call("fvv_ctx_device_generation", 1)

    def graphed(fn, n=20):
        fn()
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
        torch.cuda.synchronize()
        return timed(g.replay, max(args.reps // n, 5)) / n

    out["graph_ingest_nofill_us"] = graphed(lambda: eng.ingest_mm_many(many, hole_closing=False))
    out["graph_ingest_fill_us"] = graphed(lambda: eng.ingest_mm_many(many, hole_closing=True))
    out["graph_render_us"] = graphed(lambda: eng.render([wl.virtuals[0]], [wl.refs[0]], out=img))
    eng.ctx.profile(True)
    for _ in range(args.reps):
        eng.render([wl.virtuals[0]], [wl.refs[0]], out=img)
    prof = eng.ctx.profile_read()
    eng.ctx.profile(False)
    out["events_us"] = {k: round(1e3 * ms / n, 2) for k, (ms, n) in prof.items() if n}
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()
