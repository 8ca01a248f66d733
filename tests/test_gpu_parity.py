"""GPU parity: the sm_100a path against the CPU oracle and the reference goldens.

Bar (BASELINE.json north_star): integer stages bit-exact — z-buffer winner
index maps, stage (centre/splat/crack) maps, validity / provenance / hole
masks, median outputs; float stages: final RGB within 1 LSB on >= 99.9 % of
pixels and PSNR >= 50 dB against the reference. Against the oracle (same
fixed-order float64 arithmetic) everything, floats included, is bit-exact.
"""

import numpy as np
import pytest

from _helpers import (contrib_valid, golden, golden_names, psnr, refscene_case, syn_case,
                      within_1lsb_frac, workload)
from oracle import fvv_oracle as O

pytestmark = pytest.mark.gpu

CASES = golden_names("syn_") + golden_names("refscene_")


def _case(name):
    g = golden(name)
    return g, (syn_case(g) if name.startswith("syn_") else refscene_case(g))


def _bits_equal(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


@pytest.mark.parametrize("name", CASES)
def test_view_bit_exact_vs_oracle_and_within_tolerance_vs_reference(cuda, name):
    from paper_2007_00558_b200 import synthesis as S

    g, case = _case(name)
    frame, b = S.synthesize_view_debug(case.virtual, case.inputs(), case.refs, S.SynthesisConfig())
    o_rgb, o_prov, o = O.synthesize_view(case.virtual, case.oracle_refs(), debug=True)
    # --- vs oracle: every raster bit-exact
    np.testing.assert_array_equal(frame.pixels, o_rgb)
    np.testing.assert_array_equal(b.provenance, o_prov)
    ocs = o["fg_contributions"] + o["bg_contributions"]
    gcs = b.fg_contributions + b.bg_contributions
    assert len(ocs) == len(gcs)
    for gc, oc in zip(gcs, ocs):
        np.testing.assert_array_equal(gc.valid, oc["valid"])
        np.testing.assert_array_equal(gc.winner, oc["winner"].astype(np.int32))
        np.testing.assert_array_equal(gc.stage, oc["stage"])
        assert _bits_equal(gc.depth, oc["depth"]), "contribution depth not bit-exact"
        assert _bits_equal(gc.color, oc["color"]), "contribution colour not bit-exact"
        assert gc.weight == oc["weight"]
    for lay, key in ((b.fg, "fg"), (b.bg, "bg")):
        np.testing.assert_array_equal(lay.valid, o[key]["valid"])
        assert _bits_equal(lay.color, o[key]["color"])
        assert _bits_equal(lay.depth, o[key]["depth"])
    # --- vs the reference's own outputs
    assert within_1lsb_frac(frame.pixels, g["rgb"]) >= 0.999
    assert psnr(frame.pixels, g["rgb"]) >= 50.0
    np.testing.assert_array_equal(b.provenance, g["prov"])
    np.testing.assert_array_equal(np.stack([c.valid for c in gcs]), contrib_valid(g))


@pytest.mark.parametrize("name", ["syn_c1_s8.npz", "refscene_mid34_medium.npz"])
@pytest.mark.parametrize("layer", ["fg", "bg"])
def test_warp_layer_bit_exact(cuda, name, layer):
    from paper_2007_00558_b200 import synthesis as S
    from paper_2007_00558_b200.types import ColorFrame, DepthFrame

    _, case = _case(name)
    cfg = S.SynthesisConfig()
    for a in case.arrays:
        H, W = a["live_depth"].shape
        if layer == "fg":
            depth = DepthFrame(W, H, a["live_depth"], a["live_validity"])
            cv = None
        else:
            depth = DepthFrame(W, H, a["bg_depth"], a["bg_validity"])
            cv = a["live_validity"] == 2
        c = S.warp_layer(ColorFrame(W, H, a["rgb"]), depth, a["calib"], case.virtual, cfg,
                         color_valid=cv, layer=layer)
        o = O.warp_layer(a["rgb"], depth.depth, depth.validity, a["calib"], case.virtual,
                         O.DEFAULT_CFG, color_valid=cv, layer_fg=(layer == "fg"))
        np.testing.assert_array_equal(c.valid, o["valid"])
        np.testing.assert_array_equal(c.winner, o["winner"].astype(np.int32))
        np.testing.assert_array_equal(c.stage, o["stage"])
        assert _bits_equal(c.depth, o["depth"])
        assert _bits_equal(c.color, o["color"])


@pytest.mark.parametrize("splat,window", [(0, 3), (2, 3), (1, 5), (1, 1), (3, 5)])
def test_config_variants_bit_exact(cuda, splat, window):
    from paper_2007_00558_b200 import synthesis as S

    _, case = _case("syn_c2_s8_v3.npz")
    cfg = S.SynthesisConfig(splat_radius=splat, crack_fill_window=window, depth_band_rel=0.05,
                            hole_color=(7, 200, 13))
    ocfg = dict(O.DEFAULT_CFG, splat_radius=splat, crack_fill_window=window,
                depth_band_rel=0.05, hole_color=(7, 200, 13))
    frame, b = S.synthesize_view_debug(case.virtual, case.inputs(), case.refs, cfg)
    o_rgb, o_prov, o = O.synthesize_view(case.virtual, case.oracle_refs(), ocfg, debug=True)
    np.testing.assert_array_equal(frame.pixels, o_rgb)
    np.testing.assert_array_equal(b.provenance, o_prov)
    for gc, oc in zip(b.fg_contributions + b.bg_contributions,
                      o["fg_contributions"] + o["bg_contributions"]):
        np.testing.assert_array_equal(gc.winner, oc["winner"].astype(np.int32))
        np.testing.assert_array_equal(gc.stage, oc["stage"])
        assert _bits_equal(gc.depth, oc["depth"])


@pytest.mark.parametrize("name", golden_names("es_"))
def test_edge_server_preprocessing_vs_reference(cuda, name):
    from paper_2007_00558_b200 import depthproc as P
    from paper_2007_00558_b200.types import ColorFrame

    g = golden(name)
    wl = workload(str(g["config"]), int(g["scale"]), int(g["seed"]))
    c = wl.frames[0][int(g["cam"])]
    df = P.depth_from_millimeters(c.mm, c.validity)
    np.testing.assert_array_equal(df.depth, g["dec_depth"])
    np.testing.assert_array_equal(df.validity, g["dec_validity"])
    H, W = c.mm.shape
    out = P.bilateral_close_holes(df, ColorFrame(W, H, c.rgb))
    # K1 reads the range weights np.exp computes on this host, so it is
    # bit-exact against the reference formula evaluated here (the numpy oracle)
    od, ov, _ = O.bilateral_close_holes(df.depth, df.validity, c.rgb)
    np.testing.assert_array_equal(out.validity, ov)
    np.testing.assert_array_equal(out.depth, od)
    np.testing.assert_array_equal(out.validity, g["fill_validity"])
    if np.array_equal(od, g["fill_depth"]):
        # this host's np.exp equals the golden generator's: bit-exact
        np.testing.assert_array_equal(out.depth, g["fill_depth"])
    else:
        # another CPU's numpy SIMD exp may differ by an ulp (tolerance: 1 f32 ulp)
        diff = np.abs(out.depth.astype(np.float64) - g["fill_depth"].astype(np.float64))
        assert (diff <= np.spacing(np.abs(g["fill_depth"])).astype(np.float64)).all()


def test_codec_decode_vs_reference(cuda):
    from paper_2007_00558_b200 import depthcodec as DC
    from paper_2007_00558_b200.types import DepthRange

    g = golden("codec.npz")
    img = DC.Yuv420Image(g["y"], g["u"], g["v"])
    np.testing.assert_array_equal(DC.unpack_yuv420(img).values, g["unpacked"])
    rng = DepthRange(0.5, 6.5)
    d = DC.dequantize12(DC.DisparityMap12(64, 48, g["codes"]), rng)
    np.testing.assert_array_equal(d.depth, g["deq_depth"])
    np.testing.assert_array_equal(d.validity, g["deq_validity"])
    allc = np.arange(4096, dtype=np.uint16).reshape(64, 64)
    d = DC.dequantize12(DC.DisparityMap12(64, 64, allc), rng)
    np.testing.assert_array_equal(d.depth, g["all_depth"])
    np.testing.assert_array_equal(d.validity, g["all_validity"])
    f = DC.decode_yuv420_depth(img, rng)
    np.testing.assert_array_equal(f.depth, g["deq_depth"])
    from paper_2007_00558_b200 import depthproc as P
    dm = P.depth_from_millimeters(g["mm"], g["mm_validity"])
    np.testing.assert_array_equal(dm.depth, g["mm_depth"])
    np.testing.assert_array_equal(dm.validity, g["mm_out_validity"])


def _es_frames(wl, view=0, frame=0):
    caps = wl.frames[frame]
    return [dict(calib=caps[r].calib, rgb=caps[r].rgb, mm=caps[r].mm, validity=caps[r].validity,
                 bg_depth=caps[r].bg_depth, bg_validity=caps[r].bg_validity)
            for r in wl.refs[view]]


def _renderer(wl, frame=0, view=0):
    from paper_2007_00558_b200.engine import EdgeRenderer

    r = EdgeRenderer(wl.rig)
    for cid, c in wl.frames[frame].items():
        r.set_bg_model(cid, c.bg_depth, c.bg_validity)
        r.ingest_mm(cid, c.rgb, c.mm, c.validity, hole_closing=True)
    return r


@pytest.mark.parametrize("cfg_name,scale", [("c1", 1), ("c0", 1), ("c4", 4)])
def test_full_size_edge_server_path_vs_oracle(cuda, cfg_name, scale):
    """The headline path at full size (1080p, 3 refs): fused mm decode +
    bilateral + warp + resolve, against the oracle's es_view."""
    wl = workload(cfg_name, scale, 2007)
    r = _renderer(wl)
    img = r.render([wl.virtuals[0]], [wl.refs[0]])[0].cpu().numpy()
    o_rgb, _ = O.es_view(wl.virtuals[0], _es_frames(wl))
    # K1 uses np.exp's range weights like the C oracle: bit-exact end to end
    np.testing.assert_array_equal(img, o_rgb)


def test_batch_equals_single_and_generation_rollover(cuda):
    """Batched views == one-at-a-time views; >127 views exercise the canvas
    generation wrap (one fill per 127 views)."""
    import torch

    wl = workload("c2", 8, 2007)
    r = _renderer(wl)
    vs = wl.virtuals
    refs = wl.refs
    first = r.render(vs, refs).clone()
    for i in range(len(vs)):
        np.testing.assert_array_equal(r.render([vs[i]], [refs[i]])[0].cpu().numpy(),
                                      first[i].cpu().numpy())
    many = r.render(vs * 40, refs * 40)   # 160 views -> crosses the 127-view wrap
    for i in range(len(many)):
        assert torch.equal(many[i], first[i % len(vs)])


def test_identity_view_reproduces_inputs(cuda):
    """Property at full size: rendering a reference camera from itself gives
    back its colour on every Valid / Background pixel away from the border."""
    from paper_2007_00558_b200 import synthesis as S

    wl = workload("c1", 1, 2007)
    rid = wl.refs[0][0]
    inputs = wl.inputs(0, [rid])
    cam = inputs[rid].calib
    out, prov = S.synthesize_view(cam, inputs, [rid], S.SynthesisConfig(), return_provenance=True)
    live = inputs[rid].live_depth.validity
    keep = ((live == 0) | ((live == 2) & (inputs[rid].bg_depth.validity == 0)))
    keep &= ~S.border_mask(out.height, out.width, 2)
    same = (out.pixels == inputs[rid].live_color.pixels).all(-1)
    assert same[keep].mean() >= 0.99


def test_batched_ingest_equals_per_camera_ingest(cuda):
    """fvv_slots_ingest_mm (one launch for all reference cameras) produces the
    same slots, hence the same view, as one fvv_slot_ingest_mm per camera."""
    from paper_2007_00558_b200.engine import EdgeRenderer

    wl = workload("c1", 4, 2007)
    outs = []
    for batched in (False, True):
        r = EdgeRenderer(wl.rig)
        frames = {}
        for cid, c in wl.frames[0].items():
            r.set_bg_model(cid, c.bg_depth, c.bg_validity)
            frames[cid] = (c.rgb, c.mm, c.validity)
        if batched:
            r.ingest_mm_many(frames)
        else:
            for cid, (rgb, mm, val) in frames.items():
                r.ingest_mm(cid, rgb, mm, val)
        outs.append(r.render([wl.virtuals[0]], [wl.refs[0]])[0].cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
    o_rgb, _ = O.es_view(wl.virtuals[0], _es_frames(wl))
    np.testing.assert_array_equal(outs[1], o_rgb)


def test_private_renderers_on_two_streams_match(cuda):
    """Two private renderers (own contexts) working on alternating frames on
    their own CUDA streams (bench.py --pipelines) give the shared renderer's
    views."""
    import torch

    from paper_2007_00558_b200.engine import EdgeRenderer

    wl = workload("c2", 8, 2007)
    ref = _renderer(wl).render(wl.virtuals, wl.refs).cpu().numpy()
    engs = [EdgeRenderer(wl.rig, private=True) for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    outs = []
    for i, (e, st) in enumerate(zip(engs, streams)):
        with torch.cuda.stream(st):
            for cid, c in wl.frames[0].items():
                e.set_bg_model(cid, c.bg_depth, c.bg_validity)
                e.ingest_mm(cid, c.rgb, c.mm, c.validity, hole_closing=True)
            outs.append(e.render(wl.virtuals[i::2], wl.refs[i::2]))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(outs[0].cpu().numpy(), ref[0::2])
    np.testing.assert_array_equal(outs[1].cpu().numpy(), ref[1::2])


@pytest.mark.parametrize("W,H", [(260, 36), (132, 20), (1000, 522)])
def test_fused_ingest_fill_on_partial_tiles(cuda, W, H):
    """K0's fused mm decode + candidate listing + K1 fill where the 128x8
    tiles overhang the image (the halo split must not depend on which
    threads lie inside): equal to the oracle's decode + bilateral."""
    import torch

    from paper_2007_00558_b200.engine import EdgeRenderer
    from paper_2007_00558_b200.types import (CameraCalibration, CameraIntrinsics,
                                             CameraPose)

    rng = np.random.default_rng(W * 31 + H)
    yy, xx = np.mgrid[0:H, 0:W]
    mm = (2000 + 400 * np.sin(xx / 9.0) + 300 * np.cos(yy / 7.0)).astype(np.uint16)
    val = np.where(rng.random((H, W)) < 0.15, 1, 0).astype(np.uint8)   # Invalid sprinkles
    val[rng.random((H, W)) < 0.2] = 2
    mm[val != 0] = 0
    rgb = rng.integers(0, 256, (H, W, 3)).astype(np.uint8)
    # smooth colour so many fills succeed (range weights do not underflow)
    rgb[..., 0] = (xx * 3 % 256).astype(np.uint8)
    cam = CameraCalibration(0, CameraIntrinsics(500.0, 500.0, W / 2, H / 2, W, H),
                            CameraPose(np.eye(3), np.zeros(3)))
    r = EdgeRenderer([cam])
    d_out = torch.empty((H, W), dtype=torch.float32, device="cuda")
    v_out = torch.empty((H, W), dtype=torch.uint8, device="cuda")
    for rep in range(3):
        r.ingest_mm(0, rgb, mm, val, hole_closing=True, depth_out=d_out, validity_out=v_out)
        d, v = O.decode_mm(mm, val)
        od, ov, filled = O.bilateral_close_holes(d, v, rgb)
        assert filled.any()
        np.testing.assert_array_equal(v_out.cpu().numpy(), ov)
        np.testing.assert_array_equal(d_out.cpu().numpy(), od)


@pytest.mark.parametrize("nrefs,splat", [(9, 1), (6, 2), (16, 1)])
def test_many_references_bit_exact(cuda, nrefs, splat):
    """More than 4 references selects the 16-slot kernel instantiations (fast
    path for the default splat/crack, generic otherwise); the c4 rig has 16
    cameras."""
    from paper_2007_00558_b200 import synthesis as S

    from paper_2007_00558_b200 import scenes

    wl = scenes.make_workload("c4" if nrefs > 9 else "c2", seed=2007, scale=16 if nrefs > 9 else 8,
                              n_views=1, cameras="all")
    v = wl.virtuals[0]
    ids = sorted(wl.frames[0])[:nrefs]
    refs = sorted(ids, key=lambda i: float(np.linalg.norm(wl.rig[i].pose.center
                                                          - v.pose.center)))
    inputs = wl.inputs(0, refs)
    cfg = S.SynthesisConfig(splat_radius=splat)
    ocfg = dict(O.DEFAULT_CFG, splat_radius=splat)
    frame, prov = S.synthesize_view(v, inputs, refs, cfg, return_provenance=True)
    arrs = []
    for rid in refs:
        c = wl.frames[0][rid]
        lf = c.depth_frame()
        arrs.append(dict(calib=c.calib, rgb=c.rgb, live_depth=lf.depth, live_validity=lf.validity,
                         bg_depth=c.bg_depth, bg_validity=c.bg_validity))
    o_rgb, o_prov = O.synthesize_view(v, arrs, ocfg)
    np.testing.assert_array_equal(frame.pixels, o_rgb)
    np.testing.assert_array_equal(prov, o_prov)


def test_full_4k_edge_server_path_vs_c_oracle(cuda):
    """Maximum size: c4's 3840x2160 rig, 4 references, generated in HBM by
    scenes_gpu; mm decode + bilateral + synthesis bit-identical to the C
    oracle (itself bit-identical to the numpy oracle, tests/test_oracle.py)."""
    import torch

    from oracle import c_oracle as CO
    from paper_2007_00558_b200 import scenes_gpu
    from paper_2007_00558_b200.engine import EdgeRenderer

    wl = scenes_gpu.make_workload("c4", seed=2007, n_views=1, dev=torch.device("cuda", 0))
    v, refs = wl.virtuals[0], wl.refs[0]
    r = EdgeRenderer(wl.rig)
    frames = []
    for cid in refs:
        c = wl.frames[0][cid]
        r.set_bg_model(cid, c.bg_depth, c.bg_validity)
        r.ingest_mm(cid, c.rgb, c.mm, c.validity, hole_closing=True)
        h = c.host()
        frames.append(dict(calib=h.calib, rgb=h.rgb, mm=h.mm, validity=h.validity,
                           bg_depth=h.bg_depth, bg_validity=h.bg_validity))
    img = r.render([v], [refs])[0].cpu().numpy()
    o_rgb, _ = CO.es_view(v, frames)
    np.testing.assert_array_equal(img, o_rgb)


@pytest.mark.parametrize("name", ["syn_c1_s8.npz", "syn_c2_s8_v3.npz"])
@pytest.mark.parametrize("density", [0.005, 0.05])
def test_sparse_foreground_tile_skip_bit_exact(cuda, name, density):
    """K3 skips an FG contribution on tiles whose key span K2 did not flag
    (TileFlags): isolated FG specks put keys in tile halos and corners, where
    a missed flag would drop a splat or a crack median. The skip path (plain
    render) must equal the oracle and the all-contributions debug render."""
    from paper_2007_00558_b200 import synthesis as S

    _, case = _case(name)
    rng = np.random.default_rng(7)
    for a in case.arrays:
        fg = a["live_validity"] == 0                          # Validity.VALID
        keep = rng.random(fg.shape) < density
        keep |= np.roll(keep, 1, 0) | np.roll(keep, 1, 1)   # 2x2 specks
        a["live_validity"] = np.where(fg & ~keep, 1, a["live_validity"]).astype(np.uint8)
    frame, prov = S.synthesize_view(case.virtual, case.inputs(), case.refs, S.SynthesisConfig(),
                                    return_provenance=True)
    o_rgb, o_prov, _ = O.synthesize_view(case.virtual, case.oracle_refs(), debug=True)
    np.testing.assert_array_equal(frame.pixels, o_rgb)
    np.testing.assert_array_equal(prov, o_prov)
    dframe, _ = S.synthesize_view_debug(case.virtual, case.inputs(), case.refs,
                                        S.SynthesisConfig())
    np.testing.assert_array_equal(frame.pixels, dframe.pixels)
    assert (o_prov == 2).any(), "no foreground survived: the case tests nothing"


def test_foreground_keys_only_in_neighbour_tiles(cuda):
    """Crafted identity view (target pixel == source pixel): FG keys lie only
    in the tiles left of / above / diagonal to a 32x8 K3 tile, in the L shape
    that makes the tile's corner pixel a 5-of-8 FG splat, plus lone halo-2
    keys. The tile must still resolve that contribution (its flag check
    covers the whole staged key span x0-2 .. x0+33, y0-2 .. y0+9).
    The composite cannot show such a splat (its fetch needs valid source
    pixels, which would put keys in the tile), so this checks the rasters
    against the oracle and that the splat winners exist."""
    from _helpers import Case
    from paper_2007_00558_b200 import synthesis as S
    from paper_2007_00558_b200.types import CameraCalibration, CameraIntrinsics, CameraPose

    W, H = 128, 40
    cam = CameraCalibration(1, CameraIntrinsics(100.0, 100.0, 63.0, 19.0, W, H),
                            CameraPose(np.eye(3), np.zeros(3)))
    rng = np.random.default_rng(3)
    rgb = rng.integers(0, 256, (H, W, 3), dtype=np.uint8)
    live_v = np.ones((H, W), np.uint8)                 # INVALID
    live_d = np.zeros((H, W), np.float32)
    for x0 in (32, 64, 96):
        for y0 in (8, 16, 24, 32):
            # ring of (x0, y0) outside its tile: (x0-1, y0-1..y0+1), (x0, y0-1), (x0+1, y0-1)
            for (x, y) in ((x0 - 1, y0 - 1), (x0, y0 - 1), (x0 + 1, y0 - 1),
                           (x0 - 1, y0), (x0 - 1, y0 + 1)):
                live_v[y, x] = 0
                live_d[y, x] = 2.0 + 0.01 * (x % 7)
    live_v[4, 61] = 0            # halo-2 keys of the tiles to the right / below
    live_d[4, 61] = 3.0
    live_v[14, 90] = 0
    live_d[14, 90] = 3.0
    bg_v = np.ones((H, W), np.uint8)
    bg_d = np.zeros((H, W), np.float32)
    case = Case(cam, [1], [dict(calib=cam, rgb=rgb, live_depth=live_d, live_validity=live_v,
                                bg_depth=bg_d, bg_validity=bg_v)])
    frame, prov = S.synthesize_view(cam, case.inputs(), [1], S.SynthesisConfig(),
                                    return_provenance=True)
    o_rgb, o_prov, _ = O.synthesize_view(cam, case.oracle_refs(), debug=True)
    np.testing.assert_array_equal(prov, o_prov)
    np.testing.assert_array_equal(frame.pixels, o_rgb)
    # the corner cells do take an FG splat winner (debug rasters: every
    # contribution resolved); their backward fetch lands on Invalid source
    # pixels, so the composite leaves them holes, like the oracle
    _, b = S.synthesize_view_debug(cam, case.inputs(), [1], S.SynthesisConfig())
    assert (b.fg_contributions[0].winner[8::8, 32::32] >= 0).all()


@pytest.mark.parametrize("name", ["syn_c1_s8.npz", "syn_c2_s8_v3.npz"])
def test_dense_foreground_bg_skip_bit_exact(cuda, name):
    """Live pixels classified Background turned Valid (foreground): most K3
    tiles then have a valid merged FG layer at every pixel and skip their BG
    contributions; the few holes left still take the BG layer. Equal to the
    oracle and to the all-contributions debug render."""
    from paper_2007_00558_b200 import synthesis as S

    _, case = _case(name)
    for a in case.arrays:
        # Background-classified live pixels carry no live depth: give them the
        # BG model's depth and make them foreground
        bgc = (a["live_validity"] == 2) & (a["bg_validity"] == 0) & (a["bg_depth"] > 0)
        bgc[:, int(0.7 * bgc.shape[1]):] = False   # the right part keeps its BG layer
        a["live_depth"] = np.where(bgc, a["bg_depth"], a["live_depth"]).astype(np.float32)
        a["live_validity"] = np.where(bgc, 0, a["live_validity"]).astype(np.uint8)
    frame, prov = S.synthesize_view(case.virtual, case.inputs(), case.refs, S.SynthesisConfig(),
                                    return_provenance=True)
    o_rgb, o_prov, _ = O.synthesize_view(case.virtual, case.oracle_refs(), debug=True)
    np.testing.assert_array_equal(frame.pixels, o_rgb)
    np.testing.assert_array_equal(prov, o_prov)
    dframe, _ = S.synthesize_view_debug(case.virtual, case.inputs(), case.refs,
                                        S.SynthesisConfig())
    np.testing.assert_array_equal(frame.pixels, dframe.pixels)
    assert (o_prov == 2).mean() > 0.5 and (o_prov == 1).mean() > 0.05
