"""GPU vs the unmodified reference at BASELINE's own sizes.

Goldens ``full_<case>.npz`` (tests/golden/make_golden.py) hold the
reference's whole edge-server path — ``depth_from_millimeters`` ->
``bilateral_close_holes`` -> ``synthesize_view_debug`` (pipeline.py:518-547)
— at c0 640x360, c1 1920x1080, view 4 of c2's batch (0.2 m off the arc),
frame 150 of the c3 stream (moving spheres) and c4's 16-camera 4-reference
rig at 1920x1080. Integer outputs (fill mask,
per-contribution and merged validity, provenance) must be bit-exact, the
filled f32 depths too; RGB within the north star's float tolerance (<= 1 LSB
on >= 99.9 % of pixels, PSNR >= 50 dB), with the exact counts printed."""

import json
import os

import numpy as np
import pytest
import torch
from _helpers import full_inputs, golden, reference_rgb, rgb_agreement, sha, unpack

from oracle import c_oracle as CO

CASES = ["c0", "c1", "c2_v4", "c3_f150", "c4_s2_v0"]
RESULTS = {}


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_gpu_edge_server_path_matches_reference_at_full_size(cuda, case):
    from paper_2007_00558_b200 import synthesis as S
    from paper_2007_00558_b200.engine import EdgeRenderer
    from paper_2007_00558_b200.types import ColorFrame, DepthFrame

    g = golden(f"full_{case}.npz")
    virtual, refs, frames = full_inputs(g)
    H, W = frames[0]["mm"].shape
    rig = [f["calib"] for f in frames]
    r = EdgeRenderer(rig, private=True)
    live = []
    for j, (rid, f) in enumerate(zip(refs, frames)):
        r.set_bg_model(rid, f["bg_depth"], f["bg_validity"])
        d = torch.empty((H, W), dtype=torch.float32, device=cuda)
        v = torch.empty((H, W), dtype=torch.uint8, device=cuda)
        r.ingest_mm(rid, f["rgb"], f["mm"], f["validity"], hole_closing=True, depth_out=d,
                    validity_out=v)
        d, v = d.cpu().numpy(), v.cpu().numpy()
        ref_valid = np.unpackbits(g[f"fill{j}_validity"])[:H * W].reshape(H, W).astype(bool)
        assert np.array_equal(v == 0, ref_valid), f"fill mask of camera {rid}"
        assert sha(d) == str(g[f"fill{j}_depth_sha"]), f"filled depths of camera {rid}"
        live.append((d, v))
    # the session path (what bench.py times): RGB + provenance
    prov = torch.empty((1, H, W), dtype=torch.uint8, device=cuda)
    rgb = r.render([virtual], [refs], provenance=prov)[0].cpu().numpy()
    assert np.array_equal(prov[0].cpu().numpy(), g["prov"])
    o_rgb, _ = CO.es_view(virtual, frames)
    ref = reference_rgb(g, o_rgb)
    agree = rgb_agreement(rgb, ref)
    # the drop-in debug path on the GPU-filled depths: every mask
    inputs = {rid: S.CameraStreamInputs(f["calib"], ColorFrame(W, H, f["rgb"]),
                                        DepthFrame(W, H, d, v),
                                        DepthFrame(W, H, f["bg_depth"], f["bg_validity"]))
              for rid, f, (d, v) in zip(refs, frames, live)}
    img, b = S.synthesize_view_debug(virtual, inputs, refs, S.SynthesisConfig())
    cv = np.stack([c.valid for c in b.fg_contributions + b.bg_contributions])
    ref_cv = unpack(g, "contrib_valid", "contrib_shape")
    mv = np.stack([b.fg.valid, b.bg.valid])
    ref_mv = unpack(g, "merged_valid", "merged_shape")
    agree.update(contrib_mask_mismatches=int((cv != ref_cv).sum()),
                 merged_mask_mismatches=int((mv != ref_mv).sum()),
                 provenance_mismatches=int((b.provenance != g["prov"]).sum()),
                 debug_rgb_equals_session_rgb=bool(np.array_equal(img.pixels, rgb)))
    RESULTS[case] = agree
    print(case, json.dumps(agree))
    out = os.environ.get("FVV_PARITY_OUT")
    if out:
        with open(out, "w") as fh:
            json.dump(RESULTS, fh, indent=1)
    assert agree["contrib_mask_mismatches"] == 0
    assert agree["merged_mask_mismatches"] == 0
    assert agree["provenance_mismatches"] == 0
    assert agree["debug_rgb_equals_session_rgb"]
    assert agree["within_1lsb"] >= 0.999 * agree["pixels"] and agree["psnr_db"] >= 50.0
