"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container (the reference is importable only here):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Three fixture families, all committed as compressed .npz:

* ``syn_<case>.npz`` — reference ``synthesis.synthesize_view_debug`` on inputs
  from this repo's seeded generator (``paper_2007_00558_b200.scenes``). The
  inputs are NOT stored, only their sha256; the tests regenerate them
  (numpy, deterministic) and check the hash. Stored: RGB, provenance,
  per-contribution valid masks, merged-layer valid masks.
* ``refscene_<case>.npz`` — the reference's OWN test scenes
  (``scenegen.make_scene`` + ``conftest.gt_stream_inputs`` semantics, 128x96
  rig of tests/conftest.py:10-15), inputs stored explicitly (small), plus the
  reference outputs and, for the quality cases, the ray-cast ground truth and
  coverage mask used by tests/test_synthesis.py:213-222 and
  tests/test_acceptance.py:188-214.
* ``full_<case>.npz`` — the reference's whole edge-server path (mm decode,
  bilateral hole fill, synthesize_view_debug) at BASELINE sizes: c0 640x360,
  c1 1920x1080, view 4 of c2's jittered batch, frame 150 of the c3 stream,
  c4's rig at 1920x1080 (scale 2);
  RGB as sha256 + sparse difference against the C oracle, masks bit-packed
  (``python tests/golden/make_golden.py full [case ...]``);
* ``es_<case>.npz`` / ``codec.npz`` — edge-server preprocessing: reference
  ``depth_from_millimeters`` + ``bilateral_close_holes`` outputs on generated
  mm frames, and ``unpack_yuv420``/``dequantize12`` on generated codes.
"""

from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
OUT = Path(__file__).resolve().parent

import fvv.core as rc  # noqa: E402
import fvv.depthcodec as rcodec  # noqa: E402
import fvv.depthproc as rproc  # noqa: E402
import fvv.scenegen as rscene  # noqa: E402
import fvv.synthesis as rs  # noqa: E402

from paper_2007_00558_b200 import scenes  # noqa: E402

# (case, config, scale, seed, view index)
SYN_CASES = [
    ("c0_s4", "c0", 4, 2007, 0),
    ("c0_s2", "c0", 2, 2007, 0),
    ("c0_s2_seed11", "c0", 2, 11, 0),
    ("c1_s8", "c1", 8, 2007, 0),
    ("c2_s8_v1", "c2", 8, 2007, 1),
    ("c2_s8_v3", "c2", 8, 2007, 3),
    ("c4_s16_v0", "c4", 16, 2007, 0),
]
ES_CASES = [("c1_s4", "c1", 4, 2007), ("c0_s1", "c0", 1, 2007)]
# BASELINE sizes, full edge-server path (case, config, scale, seed, view/frame)
FULL_CASES = [
    ("c0", "c0", 1, 2007, 0),
    ("c1", "c1", 1, 2007, 0),
    ("c2_v4", "c2", 1, 2007, 4),      # virtual camera 0.2 m off the arc, near its end
    ("c3_f150", "c3", 1, 2007, 150),
    ("c4_s2_v0", "c4", 2, 2007, 0),
]


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode() + str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def ref_calib(c):
    k = c.intrinsics
    return rc.CameraCalibration(c.id, rc.CameraIntrinsics(k.fx, k.fy, k.cx, k.cy, k.width,
                                                          k.height),
                                rc.CameraPose(np.asarray(c.pose.rotation), np.asarray(c.pose.center)))


def workload(cfg, scale, seed):
    return scenes.make_workload(cfg, seed=seed, scale=scale, n_views=4, n_frames=1)


def input_hash(wl, view):
    arrs = []
    for rid in wl.refs[view]:
        c = wl.frames[0][rid]
        arrs += [c.rgb, c.mm, c.validity, c.bg_depth, c.bg_validity]
    return sha(*arrs)


def syn_case(case, cfg, scale, seed, view):
    wl = workload(cfg, scale, seed)
    v, refs = wl.virtuals[view], wl.refs[view]
    inputs = {}
    for rid in refs:
        c = wl.frames[0][rid]
        lf = c.depth_frame()
        W, H = lf.width, lf.height
        inputs[rid] = rs.CameraStreamInputs(ref_calib(c.calib), rc.ColorFrame(W, H, c.rgb),
                                            rc.DepthFrame(W, H, lf.depth, lf.validity),
                                            rc.DepthFrame(W, H, c.bg_depth, c.bg_validity))
    frame, b = rs.synthesize_view_debug(ref_calib(v), inputs, refs, rs.SynthesisConfig())
    cv = np.stack([c.valid for c in b.fg_contributions + b.bg_contributions])
    np.savez_compressed(OUT / f"syn_{case}.npz", config=cfg, scale=scale, seed=seed, view=view,
                        refs=np.asarray(refs), input_sha=input_hash(wl, view), rgb=frame.pixels,
                        prov=b.provenance, contrib_valid=np.packbits(cv),
                        contrib_shape=np.asarray(cv.shape),
                        merged_valid=np.stack([b.fg.valid, b.bg.valid]))
    print(case, wl.description, "refs", refs)


def gt_inputs(scene, rig, ref_ids, t):
    """conftest.gt_stream_inputs (tests/conftest.py:28-49), arrays only."""
    out = {}
    for rid in ref_ids:
        mvd, fg = rscene.render_with_mask(scene, rig[rid], t)
        d = mvd.depth.depth.copy()
        d[~fg] = 0.0
        out[rid] = dict(rgb=mvd.color.pixels, live_depth=d,
                        live_validity=np.where(fg, 0, 2).astype(np.uint8),
                        bg_depth=rscene.bg_depth_model(scene, rig[rid]).depth,
                        bg_validity=np.zeros(d.shape, np.uint8))
    return out


def cam_arr(c):
    k = c.intrinsics
    return np.concatenate([[c.id, k.width, k.height, k.fx, k.fy, k.cx, k.cy],
                           np.ravel(c.pose.rotation), c.pose.center]).astype(np.float64)


def refscene_case(case, preset, virtual, refs, t, quality):
    rig = rscene.build_camera_arc(9, 0.270, 60.0, width=128, height=96)
    scene = rscene.make_scene(preset)
    if virtual == "mid34":
        center = (rig[3].pose.center + rig[4].pose.center) / 2.0
        vcam = rc.CameraCalibration(200, rig[0].intrinsics, rscene.look_at_pose(center, np.zeros(3)))
        refs = sorted(range(9), key=lambda i: (rc.camera_distance(rig[i].pose, vcam.pose), i))[:3]
    else:
        vcam = rig[virtual]
    data = gt_inputs(scene, rig, refs, t)
    inputs = {rid: rs.CameraStreamInputs(
        rig[rid], rc.ColorFrame(128, 96, d["rgb"]),
        rc.DepthFrame(128, 96, d["live_depth"], d["live_validity"]),
        rc.DepthFrame(128, 96, d["bg_depth"], d["bg_validity"])) for rid, d in data.items()}
    frame, b = rs.synthesize_view_debug(vcam, inputs, refs, rs.SynthesisConfig())
    extra = {}
    if quality:
        extra["gt_rgb"] = rscene.render_ground_truth(scene, vcam, t).color.pixels
        extra["covered"] = rscene.coverage_mask(scene, t, vcam, [rig[r] for r in refs])
    cv = np.stack([c.valid for c in b.fg_contributions + b.bg_contributions])
    arrs = {}
    for j, rid in enumerate(refs):
        for k, v in data[rid].items():
            arrs[f"in{j}_{k}"] = v
        arrs[f"in{j}_cam"] = cam_arr(rig[rid])
    np.savez_compressed(OUT / f"refscene_{case}.npz", refs=np.asarray(refs), virt=cam_arr(vcam),
                        rgb=frame.pixels, prov=b.provenance, contrib_valid=cv,
                        merged_valid=np.stack([b.fg.valid, b.bg.valid]), **arrs, **extra)
    print(case, preset, "refs", refs)


def full_workload(cfg, scale, seed, view):
    """The generated inputs of a full-size case (tests/_helpers.full_case
    rebuilds the same): c3 renders only frame ``view`` of its 300-frame
    stream, c4 only the cameras view ``view`` references."""
    if cfg == "c3":
        return scenes.make_workload("c3", seed=seed, scale=scale, n_frames=300,
                                    frame_ids=[view]), 0
    return scenes.make_workload(cfg, seed=seed, scale=scale, n_views=view + 1), 0


def full_case(case, cfg, scale, seed, view):
    """The reference's whole edge-server path at a BASELINE size: per
    reference camera ``depth_from_millimeters`` -> ``bilateral_close_holes``
    (pipeline.py:518-519; mvdio.py:132), then ``synthesize_view_debug``
    (pipeline.py:546). Inputs are stored as their sha256 only. RGB is stored
    as its sha256 plus the sparse difference against the C oracle's RGB for
    the same inputs (the tests rebuild the reference RGB from the oracle's and
    check the hash); masks are bit-packed."""
    import time

    from oracle import c_oracle as CO

    wl, fidx = full_workload(cfg, scale, seed, view)
    v, refs = wl.virtuals[view], wl.refs[view]
    frame = wl.frames[fidx]
    inputs, hashed, fills = {}, [], {}
    t0 = time.time()
    for rid in refs:
        c = frame[rid]
        hashed += [c.rgb, c.mm, c.validity, c.bg_depth, c.bg_validity]
        H, W = c.mm.shape
        df = rc.depth_from_millimeters(c.mm, c.validity)
        filled = rproc.bilateral_close_holes(df, rc.ColorFrame(W, H, c.rgb))
        fills[rid] = (df, filled)
        inputs[rid] = rs.CameraStreamInputs(ref_calib(c.calib), rc.ColorFrame(W, H, c.rgb),
                                            filled, rc.DepthFrame(W, H, c.bg_depth,
                                                                  c.bg_validity))
    t1 = time.time()
    img, b = rs.synthesize_view_debug(ref_calib(v), inputs, refs, rs.SynthesisConfig())
    t2 = time.time()
    o_rgb, o_prov = CO.es_view(v, [dict(calib=frame[r].calib, rgb=frame[r].rgb, mm=frame[r].mm,
                                        validity=frame[r].validity, bg_depth=frame[r].bg_depth,
                                        bg_validity=frame[r].bg_validity) for r in refs])
    rgb = img.pixels
    diff = np.flatnonzero((rgb != o_rgb).any(-1)).astype(np.int64)
    cv = np.stack([c.valid for c in b.fg_contributions + b.bg_contributions])
    mv = np.stack([b.fg.valid, b.bg.valid])
    out = dict(config=cfg, scale=scale, seed=seed, view=view, refs=np.asarray(refs),
               input_sha=sha(*hashed), rgb_sha=sha(rgb), rgb_diff_idx=diff,
               rgb_diff_val=rgb.reshape(-1, 3)[diff], oracle_rgb_sha=sha(o_rgb),
               prov=b.provenance, contrib_valid=np.packbits(cv),
               contrib_shape=np.asarray(cv.shape), merged_valid=np.packbits(mv),
               merged_shape=np.asarray(mv.shape),
               ref_seconds=np.asarray([t1 - t0, t2 - t1]))
    for j, rid in enumerate(refs):
        df, filled = fills[rid]
        out[f"fill{j}_validity"] = np.packbits(filled.validity == 0)
        out[f"fill{j}_depth_sha"] = sha(filled.depth)
        out[f"fill{j}_holes"] = np.int64((df.validity == 1).sum())
    np.savez_compressed(OUT / f"full_{case}.npz", **out)
    print(case, wl.description, "refs", refs, f"reference {t1 - t0:.1f} s fill + "
          f"{t2 - t1:.1f} s synthesis; RGB pixels differing from the oracle: {diff.size}; "
          f"prov==oracle {float((o_prov == b.provenance).mean()):.7f}")


def es_case(case, cfg, scale, seed):
    wl = workload(cfg, scale, seed)
    rid = wl.refs[0][0]
    c = wl.frames[0][rid]
    df = rc.depth_from_millimeters(c.mm, c.validity)
    H, W = c.mm.shape
    filled = rproc.bilateral_close_holes(df, rc.ColorFrame(W, H, c.rgb))
    np.savez_compressed(OUT / f"es_{case}.npz", config=cfg, scale=scale, seed=seed, cam=rid,
                        input_sha=sha(c.rgb, c.mm, c.validity), dec_depth=df.depth,
                        dec_validity=df.validity, fill_depth=filled.depth,
                        fill_validity=filled.validity)
    print(case, "holes", int((df.validity == 1).sum()), "filled",
          int(((df.validity == 1) & (filled.validity == 0)).sum()))


def codec_case():
    rng = np.random.default_rng(5)
    H, W = 48, 64
    codes = rng.integers(0, 4096, (H, W)).astype(np.uint16)
    codes[:4, :4] = 0
    codes[4:8, :4] = 1
    codes[0, 4:] = np.arange(4, 64) % 4096
    img = rcodec.pack_yuv420(rcodec.DisparityMap12(W, H, codes))
    back = rcodec.unpack_yuv420(img)
    rng_ = rc.DepthRange(0.5, 6.5)
    deq = rcodec.dequantize12(back, rng_)
    allc = np.arange(4096, dtype=np.uint16).reshape(64, 64)
    deq_all = rcodec.dequantize12(rcodec.DisparityMap12(64, 64, allc), rng_)
    mm = np.arange(65536, dtype=np.uint16).reshape(256, 256)
    val = np.zeros(mm.shape, np.uint8)
    val[::7] = 2
    dmm = rc.depth_from_millimeters(mm, val)
    np.savez_compressed(OUT / "codec.npz", codes=codes, y=img.y, u=img.u, v=img.v,
                        unpacked=back.values, deq_depth=deq.depth, deq_validity=deq.validity,
                        all_depth=deq_all.depth, all_validity=deq_all.validity, mm=mm,
                        mm_validity=val, mm_depth=dmm.depth, mm_out_validity=dmm.validity)
    print("codec ok")


def capture_case():
    """CaptureServer chain (pipeline.py:384-397) on a generated frame."""
    wl = workload("c1", 8, 2007)
    c = wl.frames[0][wl.refs[0][0]]
    H, W = c.mm.shape
    rng = np.random.default_rng(77)
    # a degraded all-Valid depth (FG + BG surfaces), like degrade_depth's output
    d = np.where(c.mm > 0, c.mm.astype(np.float32) / 1000.0,
                 np.where(c.bg_validity == 0, c.bg_depth, 0.0)).astype(np.float32)
    val = np.where(d > 0, 0, 1).astype(np.uint8)
    depth = rc.DepthFrame(W, H, d, val)
    corrected = rproc.correct_depth(depth, rproc.CorrectionModel(-0.004, 1.01))
    model = rproc.GaussianBgModel(width=W, height=H, warmup_frames=6)
    train = []
    for i in range(6):
        px = np.clip(c.rgb.astype(np.int16) + rng.integers(-6, 7, c.rgb.shape), 0, 255)
        train.append(px.astype(np.uint8))
        rproc.bg_train(model, rc.ColorFrame(W, H, train[-1]))
    live = c.rgb.copy()
    live[H // 3: H // 2, W // 3: W // 2] = (250, 20, 40)   # a foreground blob
    fg = rproc.classify_fg(model, rc.ColorFrame(W, H, live))
    stripped = rproc.remove_bg_depth(corrected, fg)
    codes = rcodec.quantize12(stripped, rc.DepthRange(0.5, 6.5))
    img = rcodec.pack_yuv420(codes)
    np.savez_compressed(OUT / "capture.npz", depth=d, validity=val, train=np.stack(train),
                        live=live, alpha=-0.004, beta=1.01, cor_depth=corrected.depth,
                        cor_validity=corrected.validity, mean=model.mean, var=model.var,
                        fg=fg, rm_depth=stripped.depth, rm_validity=stripped.validity,
                        codes=codes.values, y=img.y, u=img.u, v=img.v)
    print("capture ok: fg", int(fg.sum()), "codes", np.bincount(codes.values.ravel() > 1))


def rice_case():
    """encode_lossless (MED + Golomb-Rice, depthcodec.py:281-443) payloads of
    the reference for small explicit planes and for the c1 depth raster at
    half resolution (the latter is regenerated by the tests from the seeded
    generator + the oracle's quantize12/pack_yuv420, checked by sha)."""
    out = {}
    rng = np.random.default_rng(31)
    small = {
        "noise": rng.integers(0, 256, (48, 64)).astype(np.uint8),
        "zero": np.zeros((16, 32), np.uint8),
        "ramp": (np.add.outer(np.arange(10) * 7, np.arange(6) * 3) % 256).astype(np.uint8),
        "sparse": (rng.random((40, 56)) < 0.02).astype(np.uint8) * 200,
    }
    for name, y in small.items():
        H, W = y.shape
        u = np.ascontiguousarray(y[::2, ::2])
        v = np.ascontiguousarray(255 - y[1::2, 1::2])
        img = rcodec.Yuv420Image(y, u, v)
        enc = rcodec.encode_lossless(img, timestamp_us=7)
        out[f"{name}_y"], out[f"{name}_u"], out[f"{name}_v"] = y, u, v
        out[f"{name}_payload"] = np.frombuffer(enc.payload, np.uint8)
    wl = workload("c1", 2, 2007)
    c = wl.frames[0][wl.refs[0][0]]
    H, W = c.mm.shape
    d = np.where(c.mm > 0, c.mm.astype(np.float32) / 1000.0,
                 np.where(c.bg_validity == 0, c.bg_depth, 0.0)).astype(np.float32)
    val = np.where(d > 0, 0, 1).astype(np.uint8)
    codes = rcodec.quantize12(rc.DepthFrame(W, H, d, val), rc.DepthRange(0.5, 6.5))
    img = rcodec.pack_yuv420(codes)
    enc = rcodec.encode_lossless(img)
    out["scene_sha"] = np.array(sha(img.y, img.u, img.v))
    out["scene_payload"] = np.frombuffer(enc.payload, np.uint8)
    heads = []
    off = 0
    for shape in ((H, W), (H // 2, W // 2), (H // 2, W // 2)):
        k, flag, n, blen, chk = rcodec._PLANE_HEADER.unpack_from(enc.payload, off)
        heads.append((k, flag, n, blen))
        off += rcodec._PLANE_HEADER.size + blen
    out["scene_heads"] = np.array(heads, np.int64)
    np.savez_compressed(OUT / "rice.npz", **out)
    print("rice ok:", {k: v.size for k, v in out.items() if k.endswith("payload")}, heads)


def silhouette_case():
    """The reference's own silhouette hole-fill scene (test_depthproc.py:
    297-319): simple scene, rig camera 4 of the 128x96 test rig, depth
    degraded with 2-px holes on the BG side of silhouettes; stored with the
    ground-truth and BG-model depths the test's accuracy criteria use and the
    reference's bilateral_close_holes output."""
    from fvv.scenegen import DepthErrorSpec

    rig = rscene.build_camera_arc(9, 0.270, 60.0, width=128, height=96)
    scene = rscene.make_scene("simple")
    mvd, fg = rscene.render_with_mask(scene, rig[4], 0.0)
    degraded = rscene.degrade_depth(mvd.depth, DepthErrorSpec(0.0, 1.0, hole_width=2), seed=6,
                                    fg_mask=fg)
    out = rproc.bilateral_close_holes(degraded, mvd.color)
    bg = rscene.bg_depth_model(scene, rig[4]).depth
    np.savez_compressed(OUT / "silhouette.npz", depth=degraded.depth, validity=degraded.validity,
                        rgb=mvd.color.pixels, gt=mvd.depth.depth, bg=bg, out_depth=out.depth,
                        out_validity=out.validity)
    print("silhouette ok: holes", int((degraded.validity == 1).sum()))


def mvd_case():
    """A small MVD disk container written by the reference's own MvdWriter
    (mvdio.py:55-98): 2 cameras x 2 sequence numbers of a 48x32 rig render,
    depth degraded with holes (all three validity codes present) and a row of
    depths on half-millimetre boundaries; plus what the reference's MvdReader
    reads back and its rle_encode / depth_to_millimeters of each frame."""
    import shutil

    import fvv.mvdio as rmvd

    root = OUT / "mvd"
    if root.exists():
        shutil.rmtree(root)
    rig = rscene.build_camera_arc(9, 0.270, 60.0, width=48, height=32)
    scene = rscene.make_scene("simple")
    out = {}
    with rmvd.MvdWriter(root, 30.0, 48, 32) as w:
        for cam in (2, 5):
            for seq in (0, 7):
                mvd, fg = rscene.render_with_mask(scene, rig[cam], seq / 30.0)
                d = rscene.degrade_depth(mvd.depth, rscene.DepthErrorSpec(0.0, 1.0, hole_width=1),
                                         seed=cam * 10 + seq, fg_mask=fg)
                depth, val = d.depth.copy(), d.validity.copy()
                val[0, :6] = [0, 1, 2, 2, 1, 0]
                depth[0, :6] = [1.5, 0.0, 0.0, 0.0, 0.0, 2.25]
                depth[1, :8] = (np.arange(8, dtype=np.float32) + np.float32(1234.5)) / 1000
                val[1, :8] = 0
                frame = rc.MvdFrame(camera_id=cam, color=mvd.color,
                                    depth=rc.DepthFrame(48, 32, depth, val, mvd.depth.timestamp_us))
                w.write_frame(seq, frame)
                key = f"c{cam}_s{seq}"
                out[key + "_depth_in"] = depth
                out[key + "_validity_in"] = val
                out[key + "_mm"] = rc.depth_to_millimeters(frame.depth)
                out[key + "_rle"] = np.asarray(rmvd.rle_encode(val), dtype=np.int64)
    r = rmvd.MvdReader(root)
    for cam in r.cameras:
        for seq in r.sequences(cam):
            f = r.read_frame(cam, seq)
            key = f"c{cam}_s{seq}"
            out[key + "_rgb"] = f.color.pixels
            out[key + "_depth"] = f.depth.depth
            out[key + "_validity"] = f.depth.validity
            out[key + "_ts"] = np.int64(f.timestamp_us)
    np.savez_compressed(OUT / "mvd.npz", **out)
    print("mvd ok:", sorted(p.name for p in root.rglob("*") if p.is_file())[:6], "...")


if __name__ == "__main__":
    if sys.argv[1:2] == ["full"]:
        for args in FULL_CASES:
            if len(sys.argv) == 2 or args[0] in sys.argv[2:]:
                full_case(*args)
        sys.exit(0)
    if sys.argv[1:] == ["mvd"]:
        mvd_case()
        sys.exit(0)
    if sys.argv[1:] == ["rice"]:
        rice_case()
        sys.exit(0)
    if sys.argv[1:] == ["silhouette"]:
        silhouette_case()
        sys.exit(0)
    mvd_case()
    silhouette_case()
    rice_case()
    capture_case()
    for args in SYN_CASES:
        syn_case(*args)
    refscene_case("identity_simple", "simple", 4, [4], 1.0, quality=True)
    refscene_case("mid34_simple", "simple", "mid34", None, 2.0, quality=True)
    refscene_case("mid34_medium", "medium", "mid34", None, 2.0, quality=True)
    refscene_case("mid34_complex", "complex", "mid34", None, 2.0, quality=True)
    refscene_case("r4_from345", "simple", 4, [3, 4, 5], 0.0, quality=False)
    for args in ES_CASES:
        es_case(*args)
    codec_case()
    for args in FULL_CASES:
        full_case(*args)
