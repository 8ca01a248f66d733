"""Oracle vs the unmodified reference at BASELINE's own sizes (CPU).

The ``full_<case>.npz`` goldens hold the reference's whole edge-server path
(``depth_from_millimeters`` -> ``bilateral_close_holes`` ->
``synthesize_view_debug``, pipeline.py:518-547) at c0 640x360, c1 1920x1080,
frame 150 of the c3 stream and c4's 16-camera rig at 1920x1080, made by
tests/golden/make_golden.py. This pins the oracle at full size; the GPU
side of the same goldens is tests/test_gpu_full_size.py."""

import numpy as np
import pytest
from _helpers import full_inputs, golden, reference_rgb, rgb_agreement, sha, unpack

from oracle import c_oracle as CO
from oracle import fvv_oracle as O

CASES = ["c0", "c1", "c2_v4", "c3_f150", "c4_s2_v0"]


@pytest.mark.parametrize("case", CASES)
def test_oracle_edge_server_path_matches_reference_at_full_size(case):
    g = golden(f"full_{case}.npz")
    virtual, refs, frames = full_inputs(g)
    # hole fill: mask and f32 depths bit-exact per reference camera
    for j, f in enumerate(frames):
        d, v = CO.decode_mm(f["mm"], f["validity"])
        assert int((v == 1).sum()) == int(g[f"fill{j}_holes"])
        d, v = CO.bilateral_close_holes(d, v, f["rgb"])
        H, W = v.shape
        ref_valid = np.unpackbits(g[f"fill{j}_validity"])[:H * W].reshape(H, W).astype(bool)
        assert np.array_equal(v == 0, ref_valid)
        assert sha(d) == str(g[f"fill{j}_depth_sha"])
    rgb, prov = CO.es_view(virtual, frames)
    ref = reference_rgb(g, rgb)
    assert np.array_equal(prov, g["prov"])
    agree = rgb_agreement(rgb, ref)
    print(case, agree)
    assert agree["within_1lsb"] >= 0.999 * agree["pixels"] and agree["psnr_db"] >= 50.0
    assert agree["identical"] >= 0.999 * agree["pixels"]


@pytest.mark.parametrize("case", ["c0", "c1"])
def test_oracle_masks_match_reference_at_full_size(case):
    """Per-contribution and merged validity masks of the numpy oracle's debug
    path against the reference's DebugBundle, bit-exact."""
    g = golden(f"full_{case}.npz")
    virtual, refs, frames = full_inputs(g)
    rgb, prov, dbg = O.es_view(virtual, frames, debug=True)
    cv = np.stack([c["valid"] for c in dbg["fg_contributions"] + dbg["bg_contributions"]])
    assert np.array_equal(cv, unpack(g, "contrib_valid", "contrib_shape"))
    mv = np.stack([dbg["fg"]["valid"], dbg["bg"]["valid"]])
    assert np.array_equal(mv, unpack(g, "merged_valid", "merged_shape"))
    assert np.array_equal(prov, g["prov"])
