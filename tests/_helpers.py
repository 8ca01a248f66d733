"""Golden-fixture loading and input reconstruction shared by the tests."""

from __future__ import annotations

import hashlib
from functools import lru_cache
from pathlib import Path

import numpy as np

from paper_2007_00558_b200 import scenes
from paper_2007_00558_b200.types import (CameraCalibration, CameraIntrinsics, CameraPose,
                                         ColorFrame, DepthFrame)

GOLDEN = Path(__file__).resolve().parent / "golden"


def golden(name: str):
    return np.load(GOLDEN / name, allow_pickle=False)


def golden_names(prefix: str):
    return sorted(p.name for p in GOLDEN.glob(prefix + "*.npz"))


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


@lru_cache(maxsize=16)
def workload(cfg: str, scale: int, seed: int):
    return scenes.make_workload(cfg, seed=seed, scale=scale, n_views=4, n_frames=1)


def cam_from(arr) -> CameraCalibration:
    a = np.asarray(arr, dtype=np.float64)
    intr = CameraIntrinsics(a[3], a[4], a[5], a[6], int(a[1]), int(a[2]))
    return CameraCalibration(int(a[0]), intr, CameraPose(a[7:16].reshape(3, 3), a[16:19]))


class Case:
    """One synthesis case: virtual camera, ordered refs, inputs in three shapes."""

    def __init__(self, virtual, refs, arrays):
        self.virtual, self.refs, self.arrays = virtual, list(refs), arrays

    def oracle_refs(self):
        return [dict(calib=a["calib"], rgb=a["rgb"], live_depth=a["live_depth"],
                     live_validity=a["live_validity"], bg_depth=a["bg_depth"],
                     bg_validity=a["bg_validity"]) for a in self.arrays]

    def inputs(self):
        from paper_2007_00558_b200.synthesis import CameraStreamInputs

        out = {}
        for rid, a in zip(self.refs, self.arrays):
            H, W = a["live_depth"].shape
            out[rid] = CameraStreamInputs(a["calib"], ColorFrame(W, H, a["rgb"]),
                                          DepthFrame(W, H, a["live_depth"], a["live_validity"]),
                                          DepthFrame(W, H, a["bg_depth"], a["bg_validity"]))
        return out


def syn_case(g) -> Case:
    wl = workload(str(g["config"]), int(g["scale"]), int(g["seed"]))
    view = int(g["view"])
    refs = [int(r) for r in g["refs"]]
    assert refs == wl.refs[view]
    arrs, hashed = [], []
    for rid in refs:
        c = wl.frames[0][rid]
        lf = c.depth_frame()
        hashed += [c.rgb, c.mm, c.validity, c.bg_depth, c.bg_validity]
        arrs.append(dict(calib=c.calib, rgb=c.rgb, live_depth=lf.depth, live_validity=lf.validity,
                         bg_depth=c.bg_depth, bg_validity=c.bg_validity))
    assert sha(*hashed) == str(g["input_sha"]), "generator drifted from the golden inputs"
    return Case(wl.virtuals[view], refs, arrs)


def refscene_case(g) -> Case:
    refs = [int(r) for r in g["refs"]]
    arrs = []
    for j in range(len(refs)):
        arrs.append(dict(calib=cam_from(g[f"in{j}_cam"]), rgb=g[f"in{j}_rgb"],
                         live_depth=g[f"in{j}_live_depth"], live_validity=g[f"in{j}_live_validity"],
                         bg_depth=g[f"in{j}_bg_depth"], bg_validity=g[f"in{j}_bg_validity"]))
    return Case(cam_from(g["virt"]), refs, arrs)


def contrib_valid(g):
    cv = g["contrib_valid"]
    if cv.dtype == np.uint8 and "contrib_shape" in g.files:
        shape = tuple(int(x) for x in g["contrib_shape"])
        cv = np.unpackbits(cv)[: int(np.prod(shape))].reshape(shape).astype(bool)
    return cv


def psnr(a, b, exclude=None) -> float:
    keep = np.ones(a.shape[:2], bool) if exclude is None else ~exclude
    mse = float(np.mean((a[keep].astype(np.float64) - b[keep].astype(np.float64)) ** 2))
    return float("inf") if mse == 0 else 10 * np.log10(255.0 ** 2 / mse)


def within_1lsb_frac(a, b) -> float:
    return float((np.abs(a.astype(int) - b.astype(int)) <= 1).all(-1).mean())


# ---------------------------------------------------------------- full-size goldens


def full_inputs(g):
    """Rebuild the generated inputs of a ``full_<case>.npz`` golden (the same
    calls as make_golden.full_workload) and check them against its hash.
    Returns (virtual, refs, frames) with frames as the oracle's es_view dicts
    (mm + validity sidecar + BG model per reference camera)."""
    cfg, scale, seed, view = str(g["config"]), int(g["scale"]), int(g["seed"]), int(g["view"])
    if cfg == "c3":
        wl = scenes.make_workload("c3", seed=seed, scale=scale, n_frames=300, frame_ids=[view])
    else:
        wl = scenes.make_workload(cfg, seed=seed, scale=scale, n_views=view + 1)
    refs = [int(r) for r in g["refs"]]
    assert refs == wl.refs[view]
    fr = wl.frames[0]
    frames, hashed = [], []
    for rid in refs:
        c = fr[rid]
        hashed += [c.rgb, c.mm, c.validity, c.bg_depth, c.bg_validity]
        frames.append(dict(calib=c.calib, rgb=c.rgb, mm=c.mm, validity=c.validity,
                           bg_depth=c.bg_depth, bg_validity=c.bg_validity))
    assert sha(*hashed) == str(g["input_sha"]), "generator drifted from the golden inputs"
    return wl.virtuals[view], refs, frames


def reference_rgb(g, oracle_rgb):
    """The reference's RGB of a full-size golden: the oracle's RGB with the
    stored sparse difference applied, checked against the stored sha256."""
    assert sha(oracle_rgb) == str(g["oracle_rgb_sha"]), \
        "oracle output changed since the golden was made: regenerate it"
    ref = np.ascontiguousarray(oracle_rgb).reshape(-1, 3).copy()
    ref[g["rgb_diff_idx"]] = g["rgb_diff_val"]
    ref = ref.reshape(oracle_rgb.shape)
    assert sha(ref) == str(g["rgb_sha"])
    return ref


def unpack(g, key, shape_key):
    shape = tuple(int(x) for x in g[shape_key])
    return np.unpackbits(g[key])[: int(np.prod(shape))].reshape(shape).astype(bool)


def rgb_agreement(a, b) -> dict:
    d = np.abs(a.astype(int) - b.astype(int)).max(-1)
    return {"pixels": int(d.size), "identical": int((d == 0).sum()),
            "within_1lsb": int((d <= 1).sum()), "max_diff": int(d.max()),
            "psnr_db": psnr(a, b)}
