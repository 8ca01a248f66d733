"""Host-side logic, the C ABI surface, and the multi-process path (CPU only)."""

import ctypes as C
import math
import os
import re
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from _helpers import golden, golden_names, sha, workload

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "fvv_b200.h"


# ---------------------------------------------------------------- types


def test_types_validate_like_the_reference():
    from paper_2007_00558_b200.types import (CameraIntrinsics, CameraPose, ColorFrame,
                                             DepthFrame, DepthRange)

    with pytest.raises(ValueError):
        CameraIntrinsics(0, 1, 1, 1, 4, 4)
    with pytest.raises(ValueError):
        CameraIntrinsics(1, 1, 5, 1, 4, 4)
    with pytest.raises(ValueError):
        CameraIntrinsics(1, 1, 1, 1, 5, 4)
    with pytest.raises(ValueError):
        CameraPose(np.eye(3) * 2, np.zeros(3))
    with pytest.raises(ValueError):
        CameraPose(-np.eye(3), np.zeros(3))
    with pytest.raises(ValueError):
        CameraPose(np.eye(3), np.array([0, 0, np.nan]))
    with pytest.raises(ValueError):
        ColorFrame(4, 4, np.zeros((4, 3, 3)))
    with pytest.raises(ValueError):
        DepthFrame(2, 2, np.zeros((2, 2)), np.zeros((2, 2)))  # Valid with depth 0
    with pytest.raises(ValueError):
        DepthRange(1.0, 0.5)
    f = DepthFrame(2, 2, np.ones((2, 2)), np.array([[0, 1], [2, 0]]))
    assert f.depth.dtype == np.float32 and f.valid_mask.sum() == 2


def test_synthesis_config_validation():
    from paper_2007_00558_b200.synthesis import SynthesisConfig

    with pytest.raises(ValueError):
        SynthesisConfig(reference_count=0)
    with pytest.raises(ValueError):
        SynthesisConfig(splat_radius=-1)
    with pytest.raises(ValueError):
        SynthesisConfig(crack_fill_window=0)


# ---------------------------------------------------------------- geometry / rig


def test_rig_round_trip_and_errors(tmp_path):
    from paper_2007_00558_b200 import geometry as G

    rig = G.build_camera_arc(9, 0.270, 60.0, width=128, height=96)
    G.save_rig(tmp_path / "rig.json", rig)
    back = G.load_rig(tmp_path / "rig.json")
    for a, b in zip(rig, back):
        assert a.id == b.id and a.intrinsics == b.intrinsics
        np.testing.assert_array_equal(a.pose.rotation, b.pose.rotation)
    txt = (tmp_path / "rig.json").read_text().replace('"version": 1', '"version": 2')
    (tmp_path / "bad.json").write_text(txt)
    with pytest.raises(ValueError):
        G.load_rig(tmp_path / "bad.json")
    with pytest.raises(ValueError):
        G.look_at_pose(np.zeros(3), np.zeros(3))
    with pytest.raises(ValueError):
        G.look_at_pose(np.zeros(3), np.array([0.0, 1.0, 0.0]))
    with pytest.raises(ValueError):
        G.build_camera_arc(1, 0.27, 60)


def test_projection_round_trip():
    from paper_2007_00558_b200 import geometry as G

    rig = G.build_camera_arc(9, 0.270, 60.0, width=128, height=96)
    d = np.full((96, 128), 2.0)
    pts = G.unproject_map(d, rig[2]).reshape(-1, 3)
    uv, z, front = G.project_points(pts, rig[2])
    assert front.all()
    np.testing.assert_allclose(z, 2.0, atol=1e-12)
    np.testing.assert_allclose(uv[:, 0].reshape(96, 128), np.tile(np.arange(128.0), (96, 1)),
                               atol=1e-9)


# ---------------------------------------------------------------- selection


def test_select_references_ranks_by_distance_then_id():
    from paper_2007_00558_b200 import geometry as G
    from paper_2007_00558_b200.selection import select_cameras, select_references

    rig = G.build_camera_arc(9, 0.270, 60.0, width=128, height=96)
    mid = (rig[3].pose.center + rig[4].pose.center) / 2
    pose = G.look_at_pose(mid, np.zeros(3))
    brute = sorted(range(9), key=lambda i: (G.camera_distance(rig[i].pose, pose), i))
    assert select_references(pose, rig, range(9), 3) == brute[:3]
    sub = [i for i in brute if i in (0, 8, 6)]
    assert select_references(pose, rig, [0, 8, 6], 2) == sub[:2] == [6, 0]
    assert set(select_references(pose, rig, [1, 2, 7], 3)) == {1, 2, 7}
    with pytest.raises(ValueError):
        select_references(pose, rig, [1, 2], 3)
    assert select_cameras(rig[4].pose, rig, 1) == [4]
    with pytest.raises(ValueError):
        select_cameras(pose, rig, 0)
    # exact tie between cams 3 and 5 around cam 4: prefer the active one
    t = select_cameras(rig[4].pose, rig, 2, current=[5])
    assert t[0] == 4 and t[1] in (3, 5)


# ---------------------------------------------------------------- generator


def test_generator_is_deterministic_and_matches_golden_hashes():
    for name in golden_names("syn_"):
        g = golden(name)
        wl = workload(str(g["config"]), int(g["scale"]), int(g["seed"]))
        refs = wl.refs[int(g["view"])]
        arrs = []
        for rid in refs:
            c = wl.frames[0][rid]
            arrs += [c.rgb, c.mm, c.validity, c.bg_depth, c.bg_validity]
        assert sha(*arrs) == str(g["input_sha"]), name


def test_generator_configs_have_expected_shapes():
    from paper_2007_00558_b200 import scenes

    wl = scenes.make_workload("c1", scale=8)
    assert len(wl.rig) == 9 and len(wl.refs[0]) == 3
    assert wl.rig[0].intrinsics.width == 240
    c = next(iter(wl.frames[0].values()))
    assert c.mm.dtype == np.uint16 and set(np.unique(c.validity)) <= {0, 1, 2}
    wl2 = scenes.make_workload("c2", scale=16, n_views=5)
    assert len(wl2.virtuals) == 5 and all(len(r) == 3 for r in wl2.refs)
    wl3 = scenes.make_workload("c3", scale=16, n_frames=3)
    assert len(wl3.frames) == 3
    phis = [math.atan2(v.pose.center[0], -v.pose.center[2]) for v in wl3.virtuals]
    assert phis == sorted(phis)


# ---------------------------------------------------------------- C ABI surface


def _header_functions():
    txt = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(fvv_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_2007_00558_b200 import _native

    lib = _native.load()
    names = _header_functions()
    assert set(names) == set(_native.EXPORTS)
    for n in names:
        assert hasattr(lib, n), n
    assert b"sm_100a" in lib.fvv_version()


def test_library_reports_missing_device_without_crashing():
    import torch

    from paper_2007_00558_b200 import _native

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    lib = _native.load()
    h = C.c_void_p()
    assert lib.fvv_ctx_create(0, C.byref(h)) == _native.FVV_ECUDA
    assert lib.fvv_sync(None) == _native.FVV_EINVAL
    with pytest.raises(RuntimeError):
        _native.Context(0)


def test_ctypes_struct_layout_matches_c(tmp_path):
    """sizeof/offsetof of every ABI struct, from gcc, equal the ctypes mirror."""
    from paper_2007_00558_b200 import _native as N

    fields = {
        "fvv_camera": ("id", "width", "fx", "cy", "R", "C"),
        "fvv_synth_cfg": ("splat_radius", "crack_fill_window", "mixing_epsilon",
                          "depth_band_rel", "hole_color", "angular_weight", "inpaint",
                          "angular_epsilon", "inpaint_radius"),
        "fvv_ref_frame": ("cam", "rgb", "live_depth", "live_validity", "bg_depth",
                          "bg_validity", "weight"),
        "fvv_debug": ("contrib_color", "contrib_stage", "merged_valid"),
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"',
             "int main(void){"]
    for s, fs in fields.items():
        lines.append(f'printf("{s} %zu\\n", sizeof({s}));')
        for f in fs:
            lines.append(f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    out = dict(l.split() for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                 check=True).stdout.splitlines())
    py = {"fvv_camera": N.FvvCamera, "fvv_synth_cfg": N.FvvSynthCfg,
          "fvv_ref_frame": N.FvvRefFrame, "fvv_debug": N.FvvDebug}
    for s, cls in py.items():
        assert int(out[s]) == C.sizeof(cls), s
        for f in fields[s]:
            assert int(out[f"{s}.{f}"]) == getattr(cls, f).offset, f"{s}.{f}"


def _imported_modules(path):
    """Every module name an ``import`` / ``from ... import`` statement, or an
    ``importlib.import_module`` / ``__import__`` call with a literal name,
    anywhere in the file (function bodies included)."""
    import ast

    tree = ast.parse(path.read_text(), str(path))
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            for a in node.names:
                yield a.name, node.lineno
        elif isinstance(node, ast.ImportFrom):
            if node.level == 0 and node.module:
                yield node.module, node.lineno
        elif isinstance(node, ast.Call):
            f = node.func
            name = f.attr if isinstance(f, ast.Attribute) else getattr(f, "id", "")
            if name in ("import_module", "__import__") and node.args and \
                    isinstance(node.args[0], ast.Constant) and isinstance(node.args[0].value, str):
                yield node.args[0].value, node.lineno


def test_product_never_imports_the_oracle():
    """No module of the package imports the oracle (test infrastructure) or
    the reference package ``fvv`` — except the pytest shim, whose job is to
    rebind the reference's seams."""
    pkg = ROOT / "paper_2007_00558_b200"
    files = sorted(pkg.rglob("*.py"))
    assert len(files) >= 10
    seen = 0
    for p in files:
        for mod, line in _imported_modules(p):
            seen += 1
            top = mod.split(".")[0]
            assert top != "oracle", f"{p.name}:{line} imports {mod}"
            if p.name != "pytest_shim.py":
                assert top != "fvv", f"{p.name}:{line} imports the reference package ({mod})"
    assert seen > 50


def test_import_guard_sees_nested_imports(tmp_path):
    f = tmp_path / "m.py"
    f.write_text("# comment\nimport os\n\n\ndef g():\n    # x\n    from oracle import fvv_oracle\n"
                 "    import importlib\n    importlib.import_module('fvv.synthesis')\n")
    mods = [m for m, _ in _imported_modules(f)]
    assert mods == ["os", "oracle", "importlib", "fvv.synthesis"]


def test_graft_build_is_up_to_date():
    import __graft_entry__ as g

    g.build()
    assert (ROOT / "paper_2007_00558_b200" / "libfvvb200.so").exists()


# ---------------------------------------------------------------- multi-process


def test_shard_covers_every_item_once():
    from paper_2007_00558_b200.distributed import shard

    for n in (0, 1, 7, 64, 300):
        for ws in (1, 2, 3, 8):
            for mode in ("block", "cyclic"):
                got = sorted(i for r in range(ws) for i in shard(n, ws, r, mode))
                assert got == list(range(n))
    assert shard(64, 8, 1) == list(range(8, 16))
    assert shard(10, 4, 0, "cyclic") == [0, 4, 8]
    with pytest.raises(ValueError):
        shard(4, 2, 2)


_WORKER = r"""
import os, sys
sys.path.insert(0, os.environ["REPO"])
import torch
from paper_2007_00558_b200 import distributed as D
rank, ws, _ = D.init("gloo")
# the frame arrives at rank 0; every rank must end with identical bytes
frame = [torch.zeros(6, 8, 3, dtype=torch.uint8), torch.zeros(6, 8, dtype=torch.int16),
         torch.zeros(6, 8, dtype=torch.uint8)]
if rank == 0:
    g = torch.Generator().manual_seed(1)
    frame[0].copy_(torch.randint(0, 256, (6, 8, 3), generator=g, dtype=torch.uint8))
    frame[1].copy_(torch.randint(0, 30000, (6, 8), generator=g, dtype=torch.int16))
    frame[2].copy_(torch.randint(0, 3, (6, 8), generator=g, dtype=torch.uint8))
# packed into one flat buffer, replicated by a single broadcast (bench.py)
flat, frame = D.pack_frame(frame)
D.broadcast_frame([flat])
assert frame[1].dtype == torch.int16 and frame[0].shape == (6, 8, 3)
mine = D.shard(64, ws, rank)
total = D.sum_over_ranks(len(mine))
slow = D.max_over_ranks(0.5 + rank)
D.barrier()
print("RESULT", rank, int(frame[0].sum()), int(frame[1].sum()), len(mine), int(total), slow,
      flush=True)
"""


def test_two_rank_gloo_broadcast_shard_and_max(tmp_path):
    import os
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    script = tmp_path / "worker.py"
    script.write_text(_WORKER)
    env = dict(os.environ, REPO=str(ROOT), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
               WORLD_SIZE="2")
    procs = [subprocess.Popen([sys.executable, str(script)],
                              env=dict(env, RANK=str(r), LOCAL_RANK=str(r)),
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(2)]
    outs = [p.communicate(timeout=180) for p in procs]
    res = {}
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e
        line = [l for l in o.splitlines() if l.startswith("RESULT")][0].split()
        res[int(line[1])] = line[2:]
    assert res[0][:2] == res[1][:2]          # identical frame bytes on both ranks
    assert res[0][2] == res[1][2] == "32"    # 64 views split 32/32
    assert res[0][3] == res[1][3] == "64"
    assert float(res[0][4]) == float(res[1][4]) == 1.5


def test_device_ray_caster_matches_host_generator():
    """scenes_gpu (torch, run here on the CPU device) renders the host
    generator's scenes: same depth rasters, RGB equal up to transcendental ulps."""
    import torch

    from paper_2007_00558_b200 import scenes, scenes_gpu

    for name, scale in (("c0", 4), ("c4", 16)):
        prm = scenes.workload_params(name, 2007)
        wl = scenes.make_workload(name, scale=scale, render_frames=False)
        cam = wl.rig[wl.refs[0][0]]
        h = scenes.render(prm["scene"], cam, 0.0)
        d = scenes_gpu.render(prm["scene"], cam, 0.0, dev="cpu")
        np.testing.assert_array_equal(d["hit"].numpy(), h["hit"])
        np.testing.assert_array_equal(d["fg"].numpy(), h["fg"])
        np.testing.assert_allclose(d["depth"].numpy(), h["depth"], rtol=1e-12, atol=0)
        np.testing.assert_array_equal(scenes_gpu.to_mm(d["depth"]).numpy().view(np.uint16),
                                      scenes.to_mm(h["depth"]))
        diff = np.abs(d["rgb"].numpy().astype(int) - h["rgb"].astype(int))
        assert diff.max() <= 1 and (diff == 0).mean() >= 0.999
        c = scenes_gpu.capture(prm["scene"], cam, 5, 0.0, dev="cpu", **prm["capture"])
        hc = c.host()
        assert hc.mm.dtype == np.uint16 and hc.rgb.shape == h["rgb"].shape
        inv = (hc.validity == 1).mean()
        assert 0 < inv < 0.2
        assert ((hc.mm > 0) <= (hc.validity == 0)).all()      # layered: only FG carries mm
        assert ((hc.bg_depth > 0) == (hc.bg_validity == 0)).all()
    wl = scenes_gpu.make_workload("c3", n_frames=3, dev="cpu", scale=16)
    assert len(wl.frames) == len(wl.virtuals) == 3
    assert all(sorted(f) == sorted(r) for f, r in zip(wl.frames, wl.refs))
    assert isinstance(wl.frames[0][wl.refs[0][0]].rgb, torch.Tensor)


def _bench(*args, env=None):
    e = {k: v for k, v in os.environ.items()
         if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                          text=True, timeout=600, env=e, cwd=str(ROOT))


def test_bench_gpus_2_launches_two_ranks():
    """``bench.py --gpus 2`` (no torchrun environment) launches two ranks by
    itself; each owns its block of c2's 64 views / its round-robin c3 frames,
    and rank 0 reports n_gpus 2 (the launcher check runs without GPU work,
    gloo on CPU)."""
    import json

    out = _bench("--gpus", "2", "--config", "c2", "--launch-check")
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["ranks"] == [0, 1]
    assert line["views_per_rank"] == [32, 32] and line["first_per_rank"] == [0, 32]
    out = _bench("--gpus", "2", "--config", "c3", "--launch-check")
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert line["frames_per_rank"] == [150, 150] and line["first_per_rank"] == [0, 1]


def test_bench_refuses_a_world_size_that_is_not_gpus():
    out = _bench("--gpus", "1", "--launch-check", env={"WORLD_SIZE": "2"})
    assert out.returncode != 0 and "WORLD_SIZE=2" in out.stderr


def test_frame_uploader_recognises_a_single_span_tick():
    """A tick whose rasters are views of one pinned allocation is uploaded as
    one span (FrameUploader._layout: start, span, offsets from the start);
    rasters in separate allocations keep one copy each."""
    import torch

    from paper_2007_00558_b200.engine import FrameUploader

    flat = torch.empty(256, dtype=torch.uint8)
    rgb = flat[32:44].view(2, 2, 3)
    mm = flat[48:56].view(torch.int16).view(2, 2)
    val = flat[64:68].view(2, 2)
    assert FrameUploader._layout({7: (rgb, mm, val)}) == (32, 36, [[0, 16, 32]])
    other = torch.empty(16, dtype=torch.uint8)[:4].view(2, 2)
    assert FrameUploader._layout({7: (rgb, mm, other)}) is None
    assert FrameUploader._layout({7: (rgb[:, :1],)}) is None   # not contiguous
