#!/usr/bin/env python
"""Edge-server view-synthesis throughput on B200 (BASELINE.json metric).

One STEP = one pass of the edge-server hot path over one MVD frame:
for each of the R reference cameras, the fused K0 mm decode + K1 joint-
bilateral hole fill + ingest (pipeline.py:514-524), then the forward warp
(K2) and resolve/blend/composite (K3) of the frame's virtual view(s)
(synthesis.synthesize_view, pipeline.py:546). Static BG models are uploaded
once per session, as in the reference edge server (pipeline.py:445).

Default workload = BASELINE.json configs[1] (c1): 1920x1080, 9-camera rig,
one virtual view from the 3 nearest cameras. Inputs rotate over --frames
pre-staged frames in HBM (default 4 x 37 MB of live inputs + 3 x 8 MB BG
models + 100 MB of z canvases per step footprint > 126 MB L2).

  value  views/s, device-timed (CUDA events, max over ranks), inputs resident
  e2e    views/s through the public API (EdgeRenderer.ingest_mm + render)
         with host buffers: pinned H2D of each step's inputs and D2H of the
         rendered RGB inside the timed region
  --impl reference   the CPU oracle port (oracle/) on the host cores, same
         workload, each step = one view per worker process

Multi-GPU: ``--gpus N`` launches N ranks itself (torch.distributed.run on
127.0.0.1) unless it already runs under torchrun. c0/c1 run N replicas; c2/c4
shard the frame's views in contiguous blocks, the frame replicated by one
NCCL broadcast per step on a comm stream overlapped with the previous frame's
render; c3 shards the stream's frames round-robin, each rank generating only
its own. Device time is the max over ranks (``rank_ms`` lists them all).
"""

from __future__ import annotations

import os

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import argparse  # noqa: E402
import json  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import tempfile  # noqa: E402
import time  # noqa: E402
from pathlib import Path  # noqa: E402

import numpy as np  # noqa: E402

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2007_00558_b200 import scenes  # noqa: E402

METRIC = "virtual views/s at 1080p (3 ref views, 9-cam rig) per GPU and 8×B200; ms/view"
PEAKS = ROOT / "MEASURED_PEAKS.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="c1", choices=("c0", "c1", "c2", "c3", "c4"))
    ap.add_argument("--frames", type=int, default=None,
                    help="pre-staged frames to rotate over (c3: frames of the stream, default "
                         "300 as BASELINE.json's config; others: 4)")
    ap.add_argument("--views", type=int, default=None, help="views per step (c2/c4 batches)")
    ap.add_argument("--seed", type=int, default=2007)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-workers", type=int, default=0, help="0 = all host cores")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--pipelines", type=int, default=None,
                    help="frames in flight: steps alternate over this many private renderers "
                         "on their own CUDA streams, so one frame's decode/fill (K0/K1) "
                         "overlaps another's warp/resolve (K2/K3); default 3 for c1/c3 (one "
                         "ingest per view), 2 for c2/c4, and 6 for c0, whose 640x360 kernels "
                         "fill a fraction of the SMs (graph replays of 6 pipelines overlap)")
    ap.add_argument("--extensions", action="store_true",
                    help="enable the two extensions outside the reference (angular blend "
                         "weights, K4 disocclusion inpainting); default is parity mode")
    ap.add_argument("--e2e-path", default="native", choices=("native", "python"),
                    help="e2e ticks through the native tick queue (fvv_tickq, one C call per "
                         "tick) or the Python FrameUploader/ResultDownloader path")
    ap.add_argument("--graphs", default="auto", choices=("auto", "on", "off"),
                    help="replay each step as a captured CUDA graph (EdgeRenderer."
                         "capture_step) instead of host launches; auto = on for c0, whose "
                         "0.05 ms steps are bound by the host's launch calls, off for the "
                         "GPU-bound configs (a graph's device-side canvas generation step "
                         "costs c1 ~1%%); c3, whose every frame has its own view, always "
                         "launches from the host")
    ap.add_argument("--launch-check", action="store_true",
                    help="launcher/sharding check without GPU work (CPU, gloo): every rank "
                         "reports the views/frames it owns; rank 0 prints one JSON line")
    ap.add_argument("--gen", default="auto", choices=("auto", "host", "gpu"),
                    help="input generator: numpy ray caster on the host, or scenes_gpu in "
                         "HBM (auto: gpu for c3/c4, whose host generation takes minutes)")
    args = ap.parse_args()
    if args.gen == "auto":
        args.gen = "gpu" if args.config in ("c3", "c4") else "host"
    if args.frames is None:
        args.frames = 300 if args.config == "c3" else 4
    # the e2e leg (PCIe-bound) replays graphs unless they are switched off
    args.e2e_graphs = args.graphs != "off"
    if args.graphs == "auto":
        args.graphs = "on" if args.config == "c0" else "off"
    args.no_graphs = args.graphs == "off"
    if args.pipelines is None:
        args.pipelines = {"c0": 6, "c1": 3, "c3": 3}.get(args.config, 2)
    return args


# ----------------------------------------------------------------------------
# workload


def my_frames(args):
    """c3: the stream's frames this rank owns (round-robin)."""
    from paper_2007_00558_b200.distributed import shard, world

    rank, ws, _ = world()
    n = max(args.frames, ws)
    return n, shard(n, ws, rank, "cyclic")


def build_workload(args):
    """The config's rig, views and frames. c3: each rank ray-casts only the
    frames it owns (``frames[i]`` is stream frame ``my_frames()[1][i]``)."""
    name = args.config
    if args.gen == "gpu":
        import torch

        from paper_2007_00558_b200 import scenes_gpu

        dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
        if name == "c3":
            n, mine = my_frames(args)
            return scenes_gpu.make_workload("c3", seed=args.seed, n_frames=n, dev=dev,
                                            frame_ids=mine)
        return scenes_gpu.make_workload(name, seed=args.seed, n_views=args.views,
                                        cameras="all" if name in ("c2", "c4") else "refs",
                                        dev=dev)
    if name == "c1":
        wl = scenes.make_workload("c1", seed=args.seed)
    elif name == "c0":
        wl = scenes.make_workload("c0", seed=args.seed)
    elif name in ("c2", "c4"):
        wl = scenes.make_workload(name, seed=args.seed, n_views=args.views, cameras="all")
    else:
        n, mine = my_frames(args)
        wl = scenes.make_workload("c3", seed=args.seed, n_frames=n, frame_ids=mine)
    return wl


def host_array(a):
    """numpy view of a capture raster (scenes_gpu keeps them as device tensors,
    mm as the int16 bit pattern of uint16)."""
    if isinstance(a, np.ndarray):
        return a
    return a.cpu().numpy()


def host_capture(c):
    return c.host() if hasattr(c, "host") else c


def frame_variants(wl, n: int, seed: int):
    """``n`` distinct frames: frame 0 as captured, the others re-noised
    (depth noise N(0, (0.5% z)^2) in mm, fresh invalid pixels) so every step
    reads different bytes. Device-generated frames (scenes_gpu) are used as
    they are: their per-step footprint already exceeds L2."""
    out = [wl.frames[0]]
    if not isinstance(wl.frames[0][next(iter(wl.frames[0]))].rgb, np.ndarray):
        return list(wl.frames[:max(n, 1)])
    rng = np.random.default_rng(seed)
    for f in range(1, n):
        if len(wl.frames) > f:
            out.append(wl.frames[f])
            continue
        fr = {}
        for cid, c in wl.frames[0].items():
            mm = c.mm.astype(np.float64)
            ok = mm > 0
            mm[ok] = np.clip(np.round(mm[ok] * (1 + 0.005 * rng.normal(size=ok.sum()))), 1, 65535)
            val = c.validity.copy()
            kill = (rng.random(mm.shape) < 0.01) & (val == 0)
            mm[kill] = 0
            fr[cid] = scenes.CameraCapture(c.calib, c.rgb, mm.astype(np.uint16), val,
                                           c.bg_depth, c.bg_validity)
        out.append(fr)
    return out


def algorithmic_bytes(wl, R: int, views_per_step: int, cams_per_step: int):
    """B_view = (8R + 3) N (layered) + per-frame preprocessing
    11 B/px/camera amortised over the frame's views; per-kernel compulsory
    bytes for the roofline of each kernel."""
    k = wl.rig[0].intrinsics
    N = k.width * k.height
    Nc = (k.width + 2) * (k.height + 2)
    b_view = (8 * R + 3) * N + 11 * N * cams_per_step / views_per_step
    per_kernel = {
        # read rgb 3 + mm 2 + validity 1, write texel 4 + warp depth 4 (per camera)
        "preprocess": 14 * N,
        # read FG + BG warp depth of R refs (4 B each); atomics land in L2
        "forward_warp": 2 * R * 4 * N,
        # read 2R canvases (8 B/key), each source texel + depth once, write RGB
        "resolve": 2 * R * 8 * Nc + R * 8 * N + 3 * N,
    }
    return b_view, per_kernel


# ----------------------------------------------------------------------------
# clocks


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            self.path = tempfile.mktemp(suffix=".csv")
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv",
                                          "-lms", "50", "-i", str(self.dev)], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        rows = [l.split(", ") for l in Path(self.path).read_text().splitlines()[1:] if l.strip()]
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1].split()[0]) for r in rows if r[1].split()[0].replace(".", "").isdigit()]
        mx = [float(r[2].split()[0]) for r in rows if r[2].split()[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------
# CPU oracle (baseline / reference arm)
#
# The timed CPU path is the C restatement of the oracle (oracle/c/fvv_oracle.c,
# bit-identical to the numpy oracle, tests/test_oracle.py): one view per host
# thread, GIL released in the foreign calls. The numpy oracle (the reference's
# own numpy formulation) is timed once beside it for context.

_POOL_JOB = {}


def _numpy_view(i):
    from oracle import fvv_oracle as O

    O.es_view(_POOL_JOB["virtual"], _POOL_JOB["frames"])
    return i


def oracle_jobs(wl, view=0):
    caps = {cid: host_capture(c) for cid, c in wl.frames[0].items() if cid in wl.refs[view]}
    frames = [dict(calib=caps[r].calib, rgb=caps[r].rgb, mm=caps[r].mm, validity=caps[r].validity,
                   bg_depth=caps[r].bg_depth, bg_validity=caps[r].bg_validity)
              for r in wl.refs[view]]
    return {"virtual": wl.virtuals[view], "frames": frames}


def c_oracle_rounds(wl, threads: int, rounds: int):
    """``rounds`` rounds of one C-oracle view per host thread; wall s per round."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import c_oracle as CO

    job = oracle_jobs(wl)
    CO.lib()
    walls = []
    with ThreadPoolExecutor(threads) as ex:
        for _ in range(rounds):
            t = time.perf_counter()
            list(ex.map(lambda _i: CO.es_view(job["virtual"], job["frames"]), range(threads)))
            walls.append(time.perf_counter() - t)
    return walls


def numpy_oracle_round(wl, workers: int):
    """One round of one numpy-oracle view per worker process (fork)."""
    import multiprocessing as mp

    _POOL_JOB.update(oracle_jobs(wl))
    t = time.perf_counter()
    with mp.get_context("fork").Pool(workers) as pool:
        pool.map(_numpy_view, range(workers))
    return time.perf_counter() - t


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_config(args, wl) -> dict:
    """The bench line's ``config``: what is measured, identical for both arms
    (the reference arm runs the same workload through the CPU port); how it
    is run goes to ``setup``."""
    return {"workload": wl.description.split(" (")[0],
            "mode": "extensions (angular weights + inpainting)" if args.extensions
                    else "parity (reference semantics)",
            "path": "mm decode + bilateral hole fill + forward warp + resolve/blend "
                    "(full edge-server path)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return 0
    wl = build_workload(args)
    threads = args.cpu_workers or os.cpu_count()
    # a step is one view per host thread (~1 s at c1); warm-up rounds run as
    # asked, timed rounds stop at the requested count or after ~120 s,
    # whichever comes first, so the arm finishes within a few minutes
    c_oracle_rounds(wl, threads, max(args.warmup, 1))
    walls = []
    budget = float(os.environ.get("FVV_REF_BUDGET_S", 120.0))
    while len(walls) < args.steps and sum(walls) < budget:
        walls += c_oracle_rounds(wl, threads, 1)
    total = sum(walls)
    value = threads * len(walls) / total
    sample = (f"C oracle port (oracle/c/fvv_oracle.c) es_view = mm decode + bilateral x"
              f"{len(wl.refs[0])} + synthesize_view, {wl.description}; each step = one view "
              f"per host thread ({threads} threads)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "views/s",
            "n_gpus": args.gpus, "steps": len(walls), "steps_requested": args.steps,
            "warmup": args.warmup,
            "ms_per_step": 1e3 * total / len(walls), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, wl),
            "setup": {"views_per_step": threads, "threads": threads,
                      "generator": wl.description},
            "cpu_baseline": {"value": value, "unit": "views/s", "cores": threads,
                             "kind": "port", "sample": sample, "cpu": cpu_model()},
            "e2e": {"value": value, "unit": "views/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------
# GPU arm


KERNEL_NAMES = {"preprocess": "k_preprocess", "forward_warp": "k_forward_warp",
                "resolve": "k_resolve_fast", "fill": "k_gen_fill"}
FACTS = ROOT / "profiles" / "r02_kernel_facts.json"      # ncu --set full, c1 step
DEVICE_PEAKS = ROOT / "profiles" / "r02_peaks.json"      # tools/peaks.cu


def kernel_rooflines(args, kern, per_kernel, atomics_per_k2, hbm, peak_src):
    """Every kernel against the roofline that bounds it:

    * ``roofline`` — the dominant kernel (K3) against HBM: algorithmic bytes
      per launch / its CUDA-event time (this run) vs the measured copy peak;
    * ``roofline_atomic`` — K2's 64-bit z-buffer atomicMin count per launch
      (a device counter, this run's profiling pass) / its event time vs the
      measured RED.E.MIN.64 rate of a warp-coherent scatter into a canvas of
      the same size (profiles/r02_peaks.json);
    * ``roofline_fp64`` / ``roofline_issue`` — K2's and K3's FP64 thread
      operations and warp instructions per launch (ncu, committed capture of
      the c1 step: profiles/r02_kernel_facts.json) / event time vs the
      measured DFMA rate and FFMA issue rate;
    * per kernel in ``kernels``: ncu DRAM bytes per launch / event time vs HBM.
    """
    out = {}
    facts = json.loads(FACTS.read_text()) if FACTS.exists() else {}
    dpk = json.loads(DEVICE_PEAKS.read_text()) if DEVICE_PEAKS.exists() else {}
    captured = args.config == "c1" and not args.extensions   # the captured workload
    for name, k in kern.items():
        f = facts.get(KERNEL_NAMES.get(name, ""), {}) if captured else {}
        t = k["avg_ms"] / 1e3
        if per_kernel.get(name):
            k["algorithmic_bytes"] = per_kernel[name]
            k["hbm_frac_algorithmic"] = per_kernel[name] / t / 1e9 / hbm
        if f.get("dram_bytes"):
            k["dram_bytes_ncu"] = f["dram_bytes"]
            k["hbm_frac_ncu_traffic"] = f["dram_bytes"] / t / 1e9 / hbm
    dom = max(kern, key=lambda n: kern[n]["avg_ms"] * kern[n]["launches"])
    if per_kernel.get(dom):
        ach = per_kernel[dom] / (kern[dom]["avg_ms"] / 1e3) / 1e9
        traffic = facts.get(KERNEL_NAMES.get(dom, ""), {}).get("dram_bytes") if captured else None
        out["roofline"] = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": hbm,
                           "unit": "GB/s", "frac": ach / hbm, "traffic": traffic,
                           "algorithmic_bytes_per_launch": per_kernel[dom],
                           "peak_source": peak_src}
    red = dpk.get("red_min_u64", {})
    canvas = "c4_canvas_66.5MB" if args.config == "c4" else "c1_canvas_16.6MB"
    peak_red = red.get(f"{canvas}/warp_consecutive")
    if "forward_warp" in kern and atomics_per_k2 and peak_red:
        ach = atomics_per_k2 / (kern["forward_warp"]["avg_ms"] / 1e3) / 1e9
        out["roofline_atomic"] = {
            "bound": "l2_atomic", "kernel": "forward_warp", "achieved": ach,
            "peak": peak_red, "unit": "G atomics/s", "frac": ach / peak_red,
            "atomics_per_launch": atomics_per_k2,
            "peak_source": f"profiles/r02_peaks.json {canvas}/warp_consecutive (tools/peaks.cu, "
                           f"measured); random scatter: {red.get(canvas + '/random')}"}
    fp = dpk.get("fp64", {}).get("dfma_per_s")
    iss = dpk.get("issue", {}).get("ffma_warp_inst_per_s")
    if captured and fp and iss:
        for name in ("forward_warp", "resolve"):
            f = facts.get(KERNEL_NAMES[name], {})
            if name not in kern or not f:
                continue
            t = kern[name]["avg_ms"] / 1e3
            out.setdefault("roofline_fp64", {})[name] = {
                "achieved": f["fp64_thread_ops"] / t, "peak": fp, "unit": "FP64 thread ops/s",
                "frac": f["fp64_thread_ops"] / t / fp,
                "fp64_ops_per_launch": f["fp64_thread_ops"],
                "ncu_fp64_pipe_pct_active": f["fp64_pipe_pct_active"]}
            out.setdefault("roofline_issue", {})[name] = {
                "achieved": f["warp_inst"] / t, "peak": iss, "unit": "warp instructions/s",
                "frac": f["warp_inst"] / t / iss, "inst_per_launch": f["warp_inst"]}
        for key in ("roofline_fp64", "roofline_issue"):
            if key in out:
                out[key]["source"] = ("per-launch counts: ncu capture of this config "
                                      "(profiles/r02_kernel_facts.json); peaks: "
                                      "profiles/r02_peaks.json (DFMA lanes/s, FFMA warp "
                                      "instructions/s, measured)")
    return out


def wire_frame(caps, depth_range):
    """A frame as the edge server receives it on the wire (pipeline.py:
    390-394, 466-472): RGB + the live depth quantised to 12-bit inverse-depth
    codes (FG Valid -> codes, BG Background -> 0, holes Invalid -> 1) packed
    as YUV420, made by this package's capture-side codec on the GPU."""
    from paper_2007_00558_b200 import depthcodec

    out = {}
    for cid, c in caps.items():
        c = host_capture(c)
        img = depthcodec.pack_yuv420(depthcodec.quantize12(c.depth_frame(), depth_range))
        out[cid] = (c.rgb, img.y, img.u, img.v)
    return out


def run_e2e(args, wl, engs, frames, views, dev, stream, wire: bool = False):
    """``e2e``: the same metric through the public host-memory API,
    ``engine.EdgeStream`` — every step's live inputs start in pinned host
    memory (RGB of the step's reference cameras + their depth: the 16-bit mm
    raster + validity sidecar, or with ``wire`` the 12-bit YUV420 codes the
    edge server receives), its rendered views end in pinned host memory; the
    H2D of step s+1 and the D2H of step s-1 overlap step s (double-buffered,
    the device output buffers rotate so a view is never overwritten while
    downloaded); repeating ticks replay a captured CUDA graph."""
    import torch

    from paper_2007_00558_b200 import distributed as D
    from paper_2007_00558_b200.engine import EdgeStream
    from paper_2007_00558_b200.types import DepthRange

    def as_tensor(a):
        a = np.ascontiguousarray(host_array(a))
        return torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a)

    def pinned_tick(fr):
        """A tick's rasters in ONE pinned host allocation, the way a receive
        buffer holds them (FrameUploader then moves one span per copy lane)."""
        ts = [(cid, [as_tensor(a) for a in arrays]) for cid, arrays in fr.items()]
        sizes = [t.numel() * t.element_size() for _, v in ts for t in v]
        flat = torch.empty(sum((n + 15) // 16 * 16 for n in sizes), dtype=torch.uint8).pin_memory()
        out, off = {}, 0
        for cid, v in ts:
            tup = []
            for t in v:
                n = t.numel() * t.element_size()
                dst = flat[off:off + n].view(t.dtype).view(tuple(t.shape))
                dst.copy_(t)
                tup.append(dst)
                off += (n + 15) // 16 * 16
            out[cid] = tuple(tup)
        return out

    # pipeline.py:71-72: the depth codec's range
    drange = DepthRange(0.5, 6.5) if wire else None

    def step_cams(s):
        return sorted({c for v in step_views(s) for c in wl.refs[v]})

    def step_views(s):
        # c3: the e2e run cycles over the frames that have host copies
        return views[s % n_host] if args.config == "c3" else views[0]

    # at most 8 distinct host ticks rotate (c3's 300 frames would pin 11 GB);
    # each holds the step's reference cameras only
    n_host = min(len(frames), 8)
    host = []
    for i, fr in enumerate(frames[:n_host]):
        cams = step_cams(i)
        sel = {cid: fr[cid] for cid in cams}
        if wire:
            host.append(pinned_tick(wire_frame(sel, drange)))
        else:
            host.append(pinned_tick({cid: (c.rgb, c.mm, c.validity) for cid, c in sel.items()}))

    def step_frame(s):
        return host[s % n_host]

    # one stream per pipeline (the device measurement's frames in flight):
    # tick s goes to stream s % P
    ess = [EdgeStream(e, max(len(v) for v in views), depth=2, depth_range=drange,
                      graphs=args.e2e_graphs, native=args.e2e_path == "native")
           for e in engs]
    es = ess[0]

    def run(start, n):
        nv_ = 0
        for s in range(start, start + n):
            vi = step_views(s)
            ess[s % len(ess)].submit(step_frame(s), [wl.virtuals[v] for v in vi],
                                     [wl.refs[v] for v in vi])
            nv_ += len(vi)
        for e in ess:
            e.wait_into(stream)
        return nv_

    # warm-up: at least two laps of the host-frame rotation, so every
    # repeating tick has been captured as a graph before the timed steps
    # (and at least three ticks per buffer slot of every stream)
    run(0, max(args.warmup, 2 * len(host) + 2, 6 * len(ess)))
    for e in ess:
        e.flush()
    torch.cuda.synchronize()
    D.barrier()

    def moved():
        return sum(e.h2d_bytes for e in ess), sum(e.d2h_bytes for e in ess)

    b0, d0 = moved()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for e in ess:
        for up in e.ups.values():
            up.stream.wait_event(e0)
        if e._dl is not None:
            e._dl.stream.wait_event(e0)
    nv2 = run(args.warmup, args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    for e in ess:
        e.flush()
    ms2 = D.max_over_ranks(e0.elapsed_time(e1))
    b1, d1 = moved()
    return {"value": D.sum_over_ranks(nv2) / (ms2 / 1e3), "unit": "views/s",
            "h2d_bytes_per_step": (b1 - b0) // args.steps,
            "d2h_bytes_per_step": (d1 - d0) // args.steps,
            "streams": len(ess),
            "input": ("12-bit YUV420 depth codes (pipeline.py:466-472) + RGB" if wire else
                      "16-bit mm + validity sidecar (mvdio.py:132) + RGB"),
            "api": ("engine.EdgeStream.submit -> native tick queue (C ABI fvv_tickq_replay / "
                    "fvv_tickq_submit): pinned H2D of the tick's single-span receive buffer "
                    "(copy stream) -> "
                    f"{'fvv_slots_ingest_yuv' if wire else 'fvv_slots_ingest_mm'} + "
                    "fvv_render_views (CUDA graph replays of repeating ticks) -> D2H into "
                    "pinned host buffers (download stream), double-buffered"
                    if es.q is not None else
                    "engine.EdgeStream.submit: pinned H2D of the tick's single-span receive "
                    "buffer (FrameUploader, copy stream) -> "
                    f"EdgeRenderer.{'ingest_yuv_many' if wire else 'ingest_mm_many'} + render "
                    f"(C ABI {'fvv_slots_ingest_yuv' if wire else 'fvv_slots_ingest_mm'}, "
                    "fvv_render_views; CUDA graph replays) -> D2H (ResultDownloader, rotating "
                    "device buffers), double-buffered"),
            "ms_per_step": ms2 / args.steps}


def run_ours(args):
    import torch

    from paper_2007_00558_b200 import distributed as D
    from paper_2007_00558_b200.engine import EdgeRenderer

    rank, ws, local = D.init()
    wl = build_workload(args)
    R = len(wl.refs[0])

    # CPU baseline first (fork pool before any CUDA context exists)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        threads = args.cpu_workers or os.cpu_count()
        walls = c_oracle_rounds(wl, threads, 3)
        wall = min(walls)
        # the numpy oracle runs in a fork pool, which must not inherit a CUDA
        # context (device-generated inputs create one): threads-only then
        np_wall = numpy_oracle_round(wl, threads) if args.gen == "host" else None
        cpu = {"value": threads / wall, "unit": "views/s", "cores": threads, "kind": "port",
               "sample": f"{threads} views ({wl.description}, view 0), one per host thread, "
                         f"by the C oracle port es_view (mm decode + bilateral + synthesis); "
                         f"best of 3 rounds, {wall:.2f} s wall",
               "cpu": cpu_model(),
               "numpy_port": None if np_wall is None else {
                   "value": threads / np_wall, "unit": "views/s",
                   "sample": f"{threads} views by the numpy oracle (the reference's numpy "
                             f"formulation), one per process, {np_wall:.1f} s wall"}}

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)

    if args.config == "c3":
        # frames sharded round-robin over ranks (each rank generated only its
        # own); view f is rendered from frame f
        _, mine = my_frames(args)
        frames = list(wl.frames)
        views = [[f] for f in mine]
    else:
        frames = frame_variants(wl, args.frames, args.seed + 1)
        nv = len(wl.virtuals)
        views = [D.shard(nv, ws, rank)] if args.config in ("c2", "c4") else [[0]]
    cams = sorted(frames[0])
    P = max(1, args.pipelines)
    from paper_2007_00558_b200.synthesis import SynthesisConfig

    rcfg = SynthesisConfig(reference_count=len(wl.refs[0]), angular_weight=args.extensions,
                           inpaint=args.extensions)
    engs = [EdgeRenderer(wl.rig, cfg=rcfg, private=P > 1) for _ in range(P)]
    eng = engs[0]
    bg_done = set()
    for fr in frames:
        for cid, c in fr.items():
            if cid not in bg_done:
                for e in engs:
                    e.set_bg_model(cid, c.bg_depth, c.bg_validity)
                bg_done.add(cid)
    pstreams = [torch.cuda.Stream(dev) for _ in range(P)] if P > 1 else [stream]
    # pre-stage every frame's live inputs in HBM (c2/c4 multi-GPU: only rank
    # 0's copy is meaningful, the others receive it by broadcast each step)
    def on_dev(a):
        if isinstance(a, np.ndarray):
            return torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a).to(dev)
        return a

    # each frame lives in one flat buffer, so a multi-GPU step replicates it
    # with a single broadcast
    staged, flats = [], []
    for fr in frames:
        order = sorted(fr)
        flat, vs = D.pack_frame([on_dev(a) for cid in order
                                 for a in (fr[cid].rgb, fr[cid].mm, fr[cid].validity)], dev)
        flats.append(flat)
        staged.append({cid: tuple(vs[3 * i:3 * i + 3]) for i, cid in enumerate(order)})
    k = wl.rig[0].intrinsics
    H, W = k.height, k.width
    vmax = max(len(v) for v in views)
    outs = [torch.empty((max(vmax, 1), H, W, 3), dtype=torch.uint8, device=dev) for _ in range(P)]
    out = outs[0]

    bcast = ws > 1 and args.config in ("c2", "c4")
    # the live MVD frame arrives at rank 0; one NCCL broadcast of its packed
    # buffer replicates it over NVLink (the path's only exchange). It runs on
    # a comm stream: frame k+1's broadcast overlaps frame k's render, which
    # waits only for its own frame's broadcast (event); a frame's buffer is
    # re-filled only after the render that read it (event).
    comm = torch.cuda.Stream(dev) if bcast else None
    landed, read_done = {}, {}
    if bcast and len(staged) < 2:
        raise SystemExit("c2/c4 multi-GPU needs --frames >= 2 (broadcast double buffering)")

    def issue_broadcast(fi):
        if fi in read_done:
            comm.wait_event(read_done.pop(fi))
        with torch.cuda.stream(comm):
            D.broadcast_frame([flats[fi]])
            ev = torch.cuda.Event()
            ev.record(comm)
        landed[fi] = ev

    def run_step(s, e, o, eager=False):
        fi = s % len(staged)
        vi = views[s % len(views)] if args.config == "c3" else views[0]
        fr = staged[fi]
        cur = torch.cuda.current_stream(dev)
        if bcast:
            if fi not in landed:
                issue_broadcast(fi)
            cur.wait_event(landed.pop(fi))
            issue_broadcast((s + 1) % len(staged))
        g = graphs.get((id(e), fi)) if graphs is not None and not eager else None
        if g is not None:
            g.replay()
            graph_launches[0] += g.launches
        else:
            need = sorted({c for v in vi for c in wl.refs[v]})
            e.ingest_mm_many({cid: fr[cid] for cid in need}, hole_closing=True)
            e.render([wl.virtuals[v] for v in vi], [wl.refs[v] for v in vi], out=o)
        if bcast:
            ev = torch.cuda.Event()
            ev.record(cur)
            read_done[fi] = ev
        return len(vi)

    def step(s):
        i = s % P
        with torch.cuda.stream(pstreams[i]):
            return run_step(s, engs[i], outs[i])

    # one CUDA graph per (pipeline, staged frame): the step's K0 -> K1 -> K2 ->
    # K3 launch sequence replayed with one call (EdgeRenderer.capture_step);
    # every graph is captured before the warm-up, outside the timed region
    graphs = None if (args.no_graphs or args.config == "c3") else {}
    graph_launches = [0]
    if graphs is not None:
        vi = views[0]
        need = sorted({c for v in vi for c in wl.refs[v]})
        for i, e in enumerate(engs):
            with torch.cuda.stream(pstreams[i]):
                for fi, fr in enumerate(staged):
                    graphs[(id(e), fi)] = e.capture_step(
                        {cid: fr[cid] for cid in need}, [wl.virtuals[v] for v in vi],
                        [wl.refs[v] for v in vi], out=outs[i][:len(vi)])
        torch.cuda.synchronize()

    for s in range(args.warmup):
        step(s)
    torch.cuda.synchronize()
    D.barrier()
    clocks = Clocks(local) if rank == 0 else None
    if clocks:
        clocks.start()
    torch.cuda.synchronize()
    D.barrier()
    l0 = sum(e.ctx.launches() for e in engs)
    g0 = graph_launches[0]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for st in pstreams:
        st.wait_stream(stream)
    nviews = 0
    for s in range(args.steps):
        nviews += step(args.warmup + s)
    for st in pstreams:
        stream.wait_stream(st)
    e1.record(stream)
    torch.cuda.synchronize()
    launches = sum(e.ctx.launches() for e in engs) - l0 + graph_launches[0] - g0
    ms = e0.elapsed_time(e1)
    D.barrier()
    clk = clocks.stop() if clocks else None
    rank_ms = D.gather_over_ranks(ms)
    ms_max = max(rank_ms)
    total_views = D.sum_over_ranks(nviews)
    value = total_views / (ms_max / 1e3)

    # per-kernel device time (instrumented pass, events on the launch stream;
    # one pipeline, so no kernel shares the GPU with another frame's)
    eng.ctx.profile(True)
    for s in range(args.steps):
        run_step(s, eng, out, eager=True)
    prof = eng.ctx.profile_read()
    eng.ctx.profile(False)
    # untimed counting pass over the rotation: K2's z-buffer atomics per launch
    eng.ctx.count_atomics(True)
    n_count = max(len(staged), 1)
    for s in range(n_count):
        run_step(s, eng, out, eager=True)
    atomics_per_k2 = eng.ctx.profile_atomics() / (n_count * max(len(views[0]), 1))
    eng.ctx.count_atomics(False)

    # e2e: public API with host buffers (run_e2e)
    e2e = e2e_mm = None
    if not args.no_e2e:
        # headline: the edge server's wire format (12-bit YUV420 depth);
        # beside it the mm + validity sidecar form (MVD container, mvdio.py)
        e2e = run_e2e(args, wl, engs, frames, views, dev, stream, wire=True)
        e2e_mm = run_e2e(args, wl, engs, frames, views, dev, stream, wire=False)
    if rank != 0:
        return 0
    peaks = json.loads(PEAKS.read_text()) if PEAKS.exists() else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if PEAKS.exists() else \
        "B200_PROFILING.md fallback 6.65 TB/s"
    views_per_step = nviews / args.steps
    cams_per_step = len({c for v in (views[0] if args.config != "c3" else [0])
                         for c in wl.refs[v]})
    b_view, per_kernel = algorithmic_bytes(wl, R, max(views_per_step, 1), cams_per_step)
    kern = {}
    for name, (tot, n) in prof.items():
        if n:
            kern[name] = {"avg_ms": tot / n, "launches": n, "share": None}
    tot_ms = sum(prof[n][0] for n in prof)
    for name in kern:
        kern[name]["share"] = prof[name][0] / tot_ms if tot_ms else None
    dom = max(kern, key=lambda n: prof[n][0])
    dom_bytes = per_kernel.get(dom)
    rl = kernel_rooflines(args, kern, per_kernel, atomics_per_k2, hbm, peak_src)
    roof = rl.pop("roofline", None)
    pipe = value / ws * b_view / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "rank_ms": rank_ms, "rank_views": D.gather_over_ranks(nviews), "ms_per_view":
            ms_max / max(nviews, 1), "higher_is_better": True, "scaling": "weak",
        # 30 ms max synthesis time, 1080p, 3 refs
        "vs_baseline": (value / ws) / (1000.0 / 30.0) if args.config == "c1" else None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(args, wl),
        "setup": {"generator": wl.description,
                  "parallelism": f"replicas x{ws}" if args.config in ("c0", "c1") else
                                 (f"frames sharded x{ws}" if args.config == "c3" else
                                  f"views sharded x{ws} + NCCL frame broadcast"),
                  "views_per_step": views_per_step, "frames_rotating": len(staged),
                  "pipelines": P,
                  "launch": "CUDA graph replay per step (EdgeRenderer.capture_step)"
                            if graphs is not None else "host launches",
                  "l2": f"inputs rotate over {len(staged)} pre-staged frames; per-step "
                        f"footprint (live inputs + BG models + 2R z canvases) exceeds the "
                        f"126 MB L2 across the rotation"},
        "roofline": roof,
        **rl,
        "roofline_pipeline": {"bytes_per_view": b_view, "achieved": pipe, "peak": hbm,
                              "unit": "GB/s", "frac": pipe / hbm,
                              "note": "SURVEY.md §8(d) B_view x views/s per GPU"},
        "kernels": kern,
        "gpu_launches": launches,
        "clocks": clk,
        "e2e": e2e,
        "e2e_mm": e2e_mm,
        "cpu_baseline": cpu,
        "published_reference": {"value": 1000.0 / 30.0, "unit": "views/s",
                                "source": "PAPER.md:505 (30 ms max on a GTX 1080)"},
    }
    print(json.dumps(line), flush=True)
    return 0


def self_launch(args) -> int:
    """``--gpus N`` without a torchrun environment: launch N ranks (one
    process per GPU) with torch.distributed.run on 127.0.0.1, exactly as the
    driver's scaling run does; rank 0's JSON line is this run's output."""
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def run_launch_check(args) -> int:
    """Ranks, world size and the work each rank owns, without any GPU work
    (tests/test_host.py runs it on CPU with gloo)."""
    from paper_2007_00558_b200 import distributed as D

    rank, ws, local = D.init("gloo")
    if args.config == "c3":
        n, mine = my_frames(args)
        unit = "frames"
    else:
        wl = scenes.make_workload(args.config, seed=args.seed, n_views=args.views,
                                  render_frames=False)
        n = len(wl.virtuals)
        mine = D.shard(n, ws, rank) if args.config in ("c2", "c4") else list(range(n))
        unit = "views"
    owned = D.gather_over_ranks(float(len(mine)))
    first = D.gather_over_ranks(float(mine[0]) if mine else -1.0)
    ranks = D.gather_over_ranks(float(rank))
    D.barrier()
    if rank == 0:
        print(json.dumps({"launch_check": True, "n_gpus": ws, "ranks": [int(r) for r in ranks],
                          "config": args.config, "unit": unit, "total": n,
                          f"{unit}_per_rank": [int(x) for x in owned],
                          "first_per_rank": [int(x) for x in first]}), flush=True)
    return 0


def main():
    args = parse()
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1 and args.impl == "ours":
        return self_launch(args)
    if ws_env is not None and int(ws_env) != args.gpus:
        print(f"bench.py: WORLD_SIZE={ws_env} but --gpus {args.gpus}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args)
    if args.launch_check:
        return run_launch_check(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
