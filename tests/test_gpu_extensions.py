"""The two extensions outside the reference (angular blend weights, K4
disocclusion inpainting): off by default, and when on they compute what
oracle/extensions.py states. Parity mode itself is covered by
test_gpu_parity.py, which runs with the default (extensions off) config."""

from __future__ import annotations

import numpy as np
import pytest

from _helpers import golden, syn_case
from oracle import extensions as X

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S(cuda):
    from paper_2007_00558_b200 import synthesis

    return synthesis


def _composite(fg_c, fg_v, bg_c, bg_v, hole=(0, 0, 0)):
    out = np.broadcast_to(np.asarray(hole, np.float64), fg_c.shape).copy()
    out = np.where(bg_v[..., None], bg_c, out)
    out = np.where(fg_v[..., None], fg_c, out)
    return np.clip(np.rint(out), 0, 255).astype(np.uint8)


@pytest.mark.parametrize("name", ["syn_c1_s8.npz", "syn_c4_s16_v0.npz"])
def test_angular_weights_match_restatement(S, name):
    case = syn_case(golden(name))
    cfg = S.SynthesisConfig(angular_weight=True)
    frame, b = S.synthesize_view_debug(case.virtual, case.inputs(), case.refs, cfg)
    plain = S.synthesize_view(case.virtual, case.inputs(), case.refs, S.SynthesisConfig())
    srcs = [a["calib"] for a in case.arrays]
    merged = []
    for layer in (b.fg_contributions, b.bg_contributions):
        cs = [(c.color, c.depth, np.asarray(c.valid, bool)) for c in layer]
        col, val = X.angular_mix(cs, case.virtual, srcs, [c.weight for c in layer],
                                 cfg.depth_band_rel, cfg.angular_epsilon)
        merged.append((col, val))
    # merged layers: same validity, colours equal up to the rounding of the
    # single-precision arccos (CUDA's and numpy's may differ by an ulp)
    for (col, val), m in zip(merged, (b.fg, b.bg)):
        np.testing.assert_array_equal(np.asarray(m.valid, bool), val)
        np.testing.assert_allclose(m.color[val], col[val], rtol=0, atol=1e-4)
    exp = _composite(merged[0][0], merged[0][1], merged[1][0], merged[1][1])
    d = np.abs(frame.pixels.astype(int) - exp.astype(int))
    assert d.max() <= 1 and (d == 0).all(-1).mean() >= 0.9999
    # the extension changes the blend where several references overlap
    assert (frame.pixels != plain.pixels).any()


@pytest.mark.parametrize("name", ["syn_c4_s16_v0.npz", "syn_c2_s8_v3.npz"])
def test_inpaint_fills_holes_from_the_background_side(S, name):
    case = syn_case(golden(name))
    base = S.SynthesisConfig()
    plain, prov0 = S.synthesize_view(case.virtual, case.inputs(), case.refs, base,
                                     return_provenance=True)
    _, b = S.synthesize_view_debug(case.virtual, case.inputs(), case.refs, base)
    assert (prov0 == 0).any(), "case has no holes to inpaint"
    fgv, bgv = np.asarray(b.fg.valid, bool), np.asarray(b.bg.valid, bool)
    depth = np.where(fgv, b.fg.depth, np.where(bgv, b.bg.depth, 0.0)).astype(np.float32)
    cfg = S.SynthesisConfig(inpaint=True, inpaint_radius=32)
    out, prov = S.synthesize_view(case.virtual, case.inputs(), case.refs, cfg,
                                  return_provenance=True)
    exp_rgb, exp_prov = X.inpaint(plain.pixels, prov0, depth, radius=32)
    np.testing.assert_array_equal(prov, exp_prov)
    keep = prov0 != 0
    np.testing.assert_array_equal(out.pixels[keep], plain.pixels[keep])
    # f32 weighted mean: the device may contract a multiply-add (1 LSB)
    assert np.abs(out.pixels.astype(int) - exp_rgb.astype(int)).max() <= 1
    assert (prov == 3).sum() > 0 and (prov == 3).sum() == ((prov0 == 0) & (exp_prov == 3)).sum()


def test_extensions_off_is_parity_mode(S):
    case = syn_case(golden("syn_c1_s8.npz"))
    a = S.synthesize_view(case.virtual, case.inputs(), case.refs, S.SynthesisConfig())
    b = S.synthesize_view(case.virtual, case.inputs(), case.refs,
                          S.SynthesisConfig(angular_weight=False, inpaint=False))
    np.testing.assert_array_equal(a.pixels, b.pixels)
