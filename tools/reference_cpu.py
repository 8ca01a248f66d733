"""Time the UNMODIFIED reference's edge-server path on this host's cores.

    python tools/reference_cpu.py [--config c1] [--procs 8]

Per view, exactly what the reference's EdgeServer does for a render tick
(pipeline.py:514-547, with the mm raster of the MVD container, mvdio.py:132):
``core.depth_from_millimeters`` -> ``depthproc.bilateral_close_holes`` per
reference camera -> ``synthesis.synthesize_view``. The reference package is
the staged copy in baseline/_ref (tools/stage_reference.sh); one view per
process of a fork pool (numpy single-threaded), one round. Prints one JSON
line. Baseline measurement only — not part of the product path.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

JOB = {}


def one_view(_i):
    import numpy as np
    import fvv.core as rc
    import fvv.depthproc as rproc
    import fvv.synthesis as rs

    v, frames = JOB["virtual"], JOB["frames"]
    t = time.perf_counter()
    inputs = {}
    for f in frames:
        c = f["calib"]
        k = c.intrinsics
        calib = rc.CameraCalibration(c.id, rc.CameraIntrinsics(k.fx, k.fy, k.cx, k.cy, k.width,
                                                               k.height),
                                     rc.CameraPose(np.asarray(c.pose.rotation),
                                                   np.asarray(c.pose.center)))
        H, W = f["mm"].shape
        depth = rproc.bilateral_close_holes(rc.depth_from_millimeters(f["mm"], f["validity"]),
                                            rc.ColorFrame(W, H, f["rgb"]))
        inputs[c.id] = rs.CameraStreamInputs(calib, rc.ColorFrame(W, H, f["rgb"]), depth,
                                             rc.DepthFrame(W, H, f["bg_depth"], f["bg_validity"]))
    k = v.intrinsics
    virt = rc.CameraCalibration(v.id, rc.CameraIntrinsics(k.fx, k.fy, k.cx, k.cy, k.width,
                                                          k.height),
                                rc.CameraPose(np.asarray(v.pose.rotation), np.asarray(v.pose.center)))
    rs.synthesize_view(virt, inputs, [f["calib"].id for f in frames], rs.SynthesisConfig())
    return time.perf_counter() - t


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c1")
    ap.add_argument("--procs", type=int, default=8)
    args = ap.parse_args()
    import fvv  # noqa: F401  (fails loudly when the reference is not staged)

    from paper_2007_00558_b200 import scenes

    wl = scenes.make_workload(args.config)
    caps = wl.frames[0]
    JOB["virtual"] = wl.virtuals[0]
    JOB["frames"] = [dict(calib=caps[r].calib, rgb=caps[r].rgb, mm=caps[r].mm,
                          validity=caps[r].validity, bg_depth=caps[r].bg_depth,
                          bg_validity=caps[r].bg_validity) for r in wl.refs[0]]
    t = time.perf_counter()
    with mp.get_context("fork").Pool(args.procs) as pool:
        per_view = pool.map(one_view, range(args.procs))
    wall = time.perf_counter() - t
    cpu = "unknown"
    for line in Path("/proc/cpuinfo").read_text().splitlines():
        if line.startswith("model name"):
            cpu = line.split(":", 1)[1].strip()
            break
    print(json.dumps({"what": "unmodified reference (fvvsim 0.1.0): depth_from_millimeters + "
                              "bilateral_close_holes x refs + synthesize_view, one view per "
                              "process", "workload": wl.description, "procs": args.procs,
                      "views_per_s": args.procs / wall, "wall_s": wall,
                      "s_per_view": sorted(per_view), "cpu": cpu,
                      "host_cores": os.cpu_count()}), flush=True)


if __name__ == "__main__":
    main()
