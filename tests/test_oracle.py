"""The CPU oracle pinned against the reference's own outputs (golden fixtures).

Fixtures were produced by running the unmodified reference
(tests/golden/make_golden.py). The oracle must reproduce them: integer
outputs (provenance, contribution / merged validity masks, codec codes,
fill masks) exactly; RGB within the north-star float criterion (>= 99.9 %
within 1 LSB, PSNR >= 50 dB) and in practice bit-identical.
"""

import numpy as np
import pytest

from _helpers import (contrib_valid, golden, golden_names, psnr, refscene_case, syn_case,
                      within_1lsb_frac, workload)
from oracle import fvv_oracle as O

SYN = golden_names("syn_")
REFSCENE = golden_names("refscene_")
ES = golden_names("es_")


def _check_view(g, case):
    rgb, prov, dbg = O.synthesize_view(case.virtual, case.oracle_refs(), debug=True)
    ref_rgb = g["rgb"]
    assert within_1lsb_frac(rgb, ref_rgb) >= 0.999
    assert psnr(rgb, ref_rgb) >= 50.0
    np.testing.assert_array_equal(prov, g["prov"])
    cv = np.stack([c["valid"] for c in dbg["fg_contributions"] + dbg["bg_contributions"]])
    np.testing.assert_array_equal(cv, contrib_valid(g))
    np.testing.assert_array_equal(np.stack([dbg["fg"]["valid"], dbg["bg"]["valid"]]),
                                  g["merged_valid"])
    return rgb


@pytest.mark.parametrize("name", SYN)
def test_oracle_matches_reference_on_generated_scenes(name):
    g = golden(name)
    rgb = _check_view(g, syn_case(g))
    # bit-identical in practice (the 1-LSB allowance covers BLAS ulps)
    assert (rgb == g["rgb"]).all(-1).mean() >= 0.9999


@pytest.mark.parametrize("name", REFSCENE)
def test_oracle_matches_reference_on_reference_scenes(name):
    g = golden(name)
    _check_view(g, refscene_case(g))


@pytest.mark.parametrize("name", ES)
def test_oracle_edge_server_preprocessing(name):
    g = golden(name)
    wl = workload(str(g["config"]), int(g["scale"]), int(g["seed"]))
    c = wl.frames[0][int(g["cam"])]
    d, v = O.decode_mm(c.mm, c.validity)
    np.testing.assert_array_equal(d, g["dec_depth"])
    np.testing.assert_array_equal(v, g["dec_validity"])
    fd, fv, filled = O.bilateral_close_holes(d, v, c.rgb)
    np.testing.assert_array_equal(fv, g["fill_validity"])
    np.testing.assert_array_equal(fd, g["fill_depth"])
    assert filled.sum() > 0


def test_oracle_codec_chain():
    g = golden("codec.npz")
    y, u, v = O.pack_yuv420(g["codes"])
    np.testing.assert_array_equal(y, g["y"])
    np.testing.assert_array_equal(u, g["u"])
    np.testing.assert_array_equal(v, g["v"])
    codes = O.unpack_yuv420(g["y"], g["u"], g["v"])
    np.testing.assert_array_equal(codes, g["unpacked"])
    np.testing.assert_array_equal(codes, g["codes"])
    z, val = O.dequantize12(codes, 0.5, 6.5)
    np.testing.assert_array_equal(z, g["deq_depth"])
    np.testing.assert_array_equal(val, g["deq_validity"])
    allc = np.arange(4096, dtype=np.uint16).reshape(64, 64)
    z, val = O.dequantize12(allc, 0.5, 6.5)
    np.testing.assert_array_equal(z, g["all_depth"])
    np.testing.assert_array_equal(val, g["all_validity"])
    d, val = O.decode_mm(g["mm"], g["mm_validity"])
    np.testing.assert_array_equal(d, g["mm_depth"])
    np.testing.assert_array_equal(val, g["mm_out_validity"])


def test_mm_decode_is_true_division_not_reciprocal():
    # core.py:264: f32(mm) / 1000 differs from f32(mm) * 0.001f on most codes
    mm = np.arange(65536, dtype=np.uint16)
    d, _ = O.decode_mm(mm.reshape(256, 256), np.zeros((256, 256), np.uint8))
    mul = (mm.astype(np.float32) * np.float32(0.001)).reshape(256, 256)
    assert (d != mul).sum() > 30000


def _literal_zbuffer(depth, valid, src, dst, r):
    """The reference's 9 ``np.minimum.at`` scatters (synthesis.py:196-205)."""
    d = depth.astype(np.float64)
    x, y, z = O.transfer(d, O.Cam(src), O.Cam(dst))
    u, v = O.project(x, y, z, O.Cam(dst))
    ok0 = valid & (z > 0)
    ui = np.rint(np.where(ok0, u, 0.0)).astype(np.int64).ravel()
    vi = np.rint(np.where(ok0, v, 0.0)).astype(np.int64).ravel()
    H, W = dst.intrinsics.height, dst.intrinsics.width
    zc = np.full((H, W), np.inf)
    zs = np.full((H, W), np.inf)
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            tu, tv = ui + dx, vi + dy
            ok = ok0.ravel() & (tu >= 0) & (tu < W) & (tv >= 0) & (tv < H)
            np.minimum.at(zc if (dy == 0 and dx == 0) else zs, (tv[ok], tu[ok]), z.ravel()[ok])
    return zc, zs


def _z_of(w, keys):
    has = keys != O.KEY_EMPTY
    idx = np.where(has, keys & np.uint64((1 << w.b) - 1), 0).astype(np.int64)
    return np.where(has, w.z_src[idx], np.inf)


@pytest.mark.parametrize("r", [0, 1, 2])
def test_keyed_canvas_equals_nine_way_scatter(r):
    """One keyed scatter into a padded canvas + ring min == the 9-way splat."""
    g = golden("syn_c2_s8_v1.npz")
    case = syn_case(g)
    for a in case.arrays:
        valid = a["live_validity"] == 0
        w = O.forward_warp(a["bg_depth"], a["bg_validity"] == 0, a["calib"], case.virtual, r)
        zc, zs = _literal_zbuffer(a["bg_depth"], a["bg_validity"] == 0, a["calib"],
                                  case.virtual, r)
        H, W = w.shape
        cen = w.canvas[r:r + H, r:r + W]
        got_c = _z_of(w, cen)
        np.testing.assert_array_equal(got_c, zc)
        ring = np.full((H, W), O.KEY_EMPTY, dtype=np.uint64)
        for dy in range(-r, r + 1):
            for dx in range(-r, r + 1):
                if dy or dx:
                    ring = np.minimum(ring, w.canvas[r + dy:r + dy + H, r + dx:r + dx + W])
        got_s = _z_of(w, ring)
        np.testing.assert_array_equal(got_s, zs)
        assert valid.any()


def test_crack_median_even_and_odd_counts():
    """np.nanmedian semantics (synthesis.py:123): even count -> mean of the middle pair."""
    H = W = 5
    vals = {(1, 1): 1.0, (1, 2): 2.0, (1, 3): 3.5, (2, 1): 4.0, (3, 1): 5.0, (3, 2): 6.0}
    src = np.array(list(vals.values()))
    canvas = np.full((H, W), O.KEY_EMPTY, dtype=np.uint64)   # splat radius 0: no padding
    for i, (y, x) in enumerate(vals):
        canvas[y, x] = O.z_keys(src[i:i + 1], np.array([i]), 3)[0]
    zbuf, winner, stage = O.resolve_zbuf(O.Warp(canvas, src, 3, 0, (H, W)), False, 3)
    assert stage[2, 2] == O.STAGE_CRACK and winner[2, 2] == -1
    assert zbuf[2, 2] == (3.5 + 4.0) / 2          # 6 neighbours -> middle pair
    assert stage[1, 1] == O.STAGE_CENTER and winner[1, 1] == 0 and zbuf[1, 1] == 1.0
    # 5 neighbours of (2,2) -> odd count -> the middle value
    canvas[3, 2] = O.KEY_EMPTY
    zbuf, _, stage = O.resolve_zbuf(O.Warp(canvas, src, 3, 0, (H, W)), False, 3)
    assert stage[2, 2] == O.STAGE_CRACK and zbuf[2, 2] == 3.5
    # 4 neighbours < need (5): stays a hole
    canvas[3, 1] = O.KEY_EMPTY
    zbuf, _, stage = O.resolve_zbuf(O.Warp(canvas, src, 3, 0, (H, W)), False, 3)
    assert stage[2, 2] == O.STAGE_NONE and np.isinf(zbuf[2, 2])


def test_oracle_rejects_empty_reference_list():
    with pytest.raises(ValueError):
        O.synthesize_view(None, [])
    with pytest.raises(ValueError):
        O.mix_layer([], O.DEFAULT_CFG)


@pytest.mark.parametrize("name", SYN + REFSCENE)
def test_c_oracle_bit_identical_to_numpy_oracle(name):
    from oracle import c_oracle as CO

    g = golden(name)
    case = syn_case(g) if name.startswith("syn_") else refscene_case(g)
    a, pa = O.synthesize_view(case.virtual, case.oracle_refs())
    b, pb = CO.synthesize_view(case.virtual, case.oracle_refs())
    np.testing.assert_array_equal(a, b)
    np.testing.assert_array_equal(pa, pb)


@pytest.mark.parametrize("name", ES)
def test_c_oracle_preprocessing_matches_reference(name):
    from oracle import c_oracle as CO

    g = golden(name)
    wl = workload(str(g["config"]), int(g["scale"]), int(g["seed"]))
    c = wl.frames[0][int(g["cam"])]
    d, v = CO.decode_mm(c.mm, c.validity)
    np.testing.assert_array_equal(d, g["dec_depth"])
    np.testing.assert_array_equal(v, g["dec_validity"])
    fd, fv = CO.bilateral_close_holes(d, v, c.rgb)
    np.testing.assert_array_equal(fv, g["fill_validity"])
    # the C restatement reads np.exp's range weights, so it is bit-exact
    np.testing.assert_array_equal(fd, g["fill_depth"])


def test_oracle_bilateral_on_the_reference_silhouette_scene():
    """The reference's own hole-fill scene (test_depthproc.py:297-319)."""
    g = golden("silhouette.npz")
    d, v, _ = O.bilateral_close_holes(g["depth"], g["validity"], g["rgb"])
    np.testing.assert_array_equal(v, g["out_validity"])
    np.testing.assert_array_equal(d, g["out_depth"])
