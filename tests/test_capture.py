"""Capture-server chain: oracle and GPU vs the reference.

Golden fixture ``capture.npz`` (tests/golden/make_golden.py::capture_case)
holds the reference's own ``correct_depth`` -> ``bg_train`` x6 ->
``classify_fg`` -> ``remove_bg_depth`` -> ``quantize12`` -> ``pack_yuv420``
outputs (pipeline.py:384-397). Every stage is integer or f64-then-f32 and is
required bit-exact.
"""

import numpy as np
import pytest

from _helpers import golden
from oracle import fvv_oracle as O


def test_oracle_capture_chain_matches_reference():
    g = golden("capture.npz")
    d, v = O.correct_depth(g["depth"], g["validity"], float(g["alpha"]), float(g["beta"]))
    np.testing.assert_array_equal(d, g["cor_depth"])
    np.testing.assert_array_equal(v, g["cor_validity"])
    mean = np.zeros(g["mean"].shape)
    var = np.zeros(g["var"].shape)
    for i, fr in enumerate(g["train"]):
        O.bg_train(mean, var, fr, first=(i == 0))
    np.testing.assert_array_equal(mean, g["mean"])
    np.testing.assert_array_equal(var, g["var"])
    fg = O.classify_fg(mean, var, g["live"])
    np.testing.assert_array_equal(fg, g["fg"])
    rd, rv = O.remove_bg_depth(d, v, fg)
    np.testing.assert_array_equal(rd, g["rm_depth"])
    np.testing.assert_array_equal(rv, g["rm_validity"])
    codes = O.quantize12(rd, rv, 0.5, 6.5)
    np.testing.assert_array_equal(codes, g["codes"])
    y, u, vv = O.pack_yuv420(codes)
    np.testing.assert_array_equal(y, g["y"])
    np.testing.assert_array_equal(u, g["u"])
    np.testing.assert_array_equal(vv, g["v"])


@pytest.mark.gpu
def test_gpu_capture_chain_matches_reference(cuda):
    from paper_2007_00558_b200 import depthcodec as DC
    from paper_2007_00558_b200 import depthproc as P
    from paper_2007_00558_b200.types import ColorFrame, DepthFrame, DepthRange

    g = golden("capture.npz")
    H, W = g["depth"].shape
    cm = P.CorrectionModel(float(g["alpha"]), float(g["beta"]))
    cor = P.correct_depth(DepthFrame(W, H, g["depth"], g["validity"]), cm)
    np.testing.assert_array_equal(cor.depth, g["cor_depth"])
    np.testing.assert_array_equal(cor.validity, g["cor_validity"])
    model = P.GaussianBgModel(W, H, warmup_frames=6)
    with pytest.raises(P.UntrainedModelError):
        P.classify_fg(model, ColorFrame(W, H, g["live"]))
    for fr in g["train"]:
        P.bg_train(model, ColorFrame(W, H, fr))
    np.testing.assert_array_equal(model.mean, g["mean"])
    np.testing.assert_array_equal(model.var, g["var"])
    fg = P.classify_fg(model, ColorFrame(W, H, g["live"]))
    np.testing.assert_array_equal(fg, g["fg"])
    rm = P.remove_bg_depth(cor, fg)
    np.testing.assert_array_equal(rm.depth, g["rm_depth"])
    np.testing.assert_array_equal(rm.validity, g["rm_validity"])
    rng = DepthRange(0.5, 6.5)
    codes = DC.quantize12(rm, rng)
    np.testing.assert_array_equal(codes.values, g["codes"])
    img = DC.pack_yuv420(codes)
    np.testing.assert_array_equal(img.y, g["y"])
    np.testing.assert_array_equal(img.u, g["u"])
    np.testing.assert_array_equal(img.v, g["v"])
    # the fused one-pass chain gives the same planes
    img2, codes2 = DC.capture_encode(DepthFrame(W, H, g["depth"], g["validity"]),
                                     ColorFrame(W, H, g["live"]), rng, correction=cm,
                                     bg_model=model)
    np.testing.assert_array_equal(codes2.values, g["codes"])
    np.testing.assert_array_equal(img2.y, g["y"])
    np.testing.assert_array_equal(img2.u, g["u"])
    np.testing.assert_array_equal(img2.v, g["v"])
    # round trip through the edge-server decoder: codes survive exactly
    np.testing.assert_array_equal(DC.unpack_yuv420(img2).values, g["codes"])


@pytest.mark.gpu
def test_gpu_quantize_round_trip_property(cuda):
    """encode -> decode -> encode is the identity on codes (depthcodec.py:128)."""
    from paper_2007_00558_b200 import depthcodec as DC
    from paper_2007_00558_b200.types import DepthFrame, DepthRange

    rng = np.random.default_rng(3)
    H, W = 270, 480
    z = rng.uniform(0.3, 8.0, (H, W)).astype(np.float32)
    v = rng.choice([0, 0, 0, 1, 2], (H, W)).astype(np.uint8)
    z[v != 0] = 0.0
    r = DepthRange(0.5, 6.5)
    c1 = DC.quantize12(DepthFrame(W, H, z, v), r)
    back = DC.dequantize12(c1, r)
    c2 = DC.quantize12(back, r)
    np.testing.assert_array_equal(c1.values, c2.values)
    img = DC.pack_yuv420(c1)
    np.testing.assert_array_equal(DC.unpack_yuv420(img).values, c1.values)
