"""pytest plugin / import hook: route the reference's seams to the B200 backend.

    PYTHONPATH=<fvv src>:<this repo> python -m pytest -p paper_2007_00558_b200.pytest_shim \
        <fvv>/tests/test_synthesis.py <fvv>/tests/test_acceptance.py

Plugins load before rootdir conftests, so ``from fvv import synthesis`` in the
reference's conftest (tests/conftest.py:6) already receives the GPU module.
What is rebound:

* ``fvv.synthesis`` — every public name of :mod:`paper_2007_00558_b200.synthesis`
  (synthesize_view, synthesize_view_debug, warp_layer, mix_layer, composite,
  write_debug_bundle, view_psnr, border_mask, the config/contribution types);
* ``fvv.pipeline.synthesis`` — the module global ``EdgeServer.render_tick``
  reaches through ``synthesize_with_config`` (pipeline.py:546, 569-570);
* ``fvv.depthproc.bilateral_close_holes`` (called at pipeline.py:518-519);
* with ``FVV_SHIM_CODEC=1`` also the depth codec the edge server runs before
  synthesis and the capture server after capture: ``fvv.depthcodec``'s
  ``unpack_yuv420`` / ``dequantize12`` (pipeline.py:469-472), ``quantize12`` /
  ``pack_yuv420`` (pipeline.py:392-393) and the MED + Rice
  ``encode_lossless`` / ``decode_lossless`` (pipeline.py:394, 469). This
  module's codec then builds and raises the reference's own types
  (EncodedFrame, Yuv420Image, DisparityMap12, DecodeError,
  UnsupportedCodecError), so callers that catch or isinstance-check them
  keep working;
* with ``FVV_SHIM_MVDIO=1`` the MVD disk container (``fvv.mvdio``:
  ``rle_encode`` / ``rle_decode`` / ``MvdWriter`` / ``MvdReader``, and the
  ``MvdWriter`` that pipeline.py:32 imported); the reader returns this
  package's frame types, which carry the same attributes.
"""

from __future__ import annotations

import os
import sys
import types

_OVERRIDE = ("SynthesisConfig", "LayerContribution", "MergedLayer", "CameraStreamInputs",
             "DebugBundle", "warp_layer", "mix_layer", "composite", "synthesize_view",
             "synthesize_view_debug", "write_debug_bundle", "view_psnr", "border_mask",
             "LAYER_FG", "LAYER_BG")
installed = {}


def install() -> types.ModuleType:
    """Replace the reference seams in ``sys.modules``; idempotent."""
    if "synthesis" in installed:
        return installed["synthesis"]
    import fvv
    from fvv import synthesis as ref_syn

    from . import depthproc as ours_dp
    from . import synthesis as ours

    mod = types.ModuleType("fvv.synthesis", ours.__doc__)
    mod.__dict__.update({k: v for k, v in ref_syn.__dict__.items() if not k.startswith("__")})
    for name in _OVERRIDE:
        setattr(mod, name, getattr(ours, name))
    mod.__file__ = ours.__file__
    mod.B200_BACKEND = True
    sys.modules["fvv.synthesis"] = mod
    fvv.synthesis = mod
    if "fvv.pipeline" in sys.modules:
        sys.modules["fvv.pipeline"].synthesis = mod
    import fvv.depthproc as ref_dp

    ref_dp.bilateral_close_holes = ours_dp.bilateral_close_holes
    if os.environ.get("FVV_SHIM_CODEC") == "1":
        import fvv.depthcodec as ref_codec

        from . import depthcodec as ours_codec

        for name in ("EncodedFrame", "Yuv420Image", "DisparityMap12", "DecodeError",
                     "UnsupportedCodecError"):
            setattr(ours_codec, name, getattr(ref_codec, name))
        for name in ("unpack_yuv420", "dequantize12", "quantize12", "pack_yuv420",
                     "encode_lossless", "decode_lossless"):
            setattr(ref_codec, name, getattr(ours_codec, name))
        # one byte-codec registry: codecs registered through either module
        # (depthcodec.register_codec, depthcodec.py:416-421) serve both
        ours_codec._COMPRESSORS = ref_codec._COMPRESSORS
    if os.environ.get("FVV_SHIM_MVDIO") == "1":
        import fvv.mvdio as ref_mvd

        from . import mvdio as ours_mvd

        for name in ("rle_encode", "rle_decode", "MvdWriter", "MvdReader"):
            setattr(ref_mvd, name, getattr(ours_mvd, name))
        if "fvv.pipeline" in sys.modules:   # pipeline.py:32 binds MvdWriter at import
            sys.modules["fvv.pipeline"].MvdWriter = ours_mvd.MvdWriter
    installed["synthesis"] = mod
    return mod


def launches() -> int:
    """GPU kernels launched so far by this process's library contexts."""
    from . import _native

    return sum(c.launches() for c in _native._contexts.values())


def pytest_configure(config):  # pragma: no cover - exercised through pytest -p
    install()


def pytest_unconfigure(config):  # pragma: no cover - exercised through pytest -p
    # FVV_SHIM_REPORT=<path>: record how many kernels the run launched, the
    # evidence that the reference's tests exercised the GPU backend
    path = os.environ.get("FVV_SHIM_REPORT")
    if path:
        with open(path, "w") as fh:
            fh.write(f"{launches()}\n")
