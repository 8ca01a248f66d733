"""The pytest shim's rebinding mechanics (CPU; needs the reference package,
which exists only in the build container — skipped elsewhere)."""

import importlib
import subprocess
import sys
from pathlib import Path

import pytest

REF_SRC = Path("/root/reference/pkg/src")
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference package not present on this host")
def test_shim_rebinds_every_reference_seam():
    code = r"""
import sys
from paper_2007_00558_b200 import pytest_shim
mod = pytest_shim.install()
import fvv, fvv.synthesis, fvv.pipeline, fvv.depthproc
from paper_2007_00558_b200 import synthesis as ours, depthproc as odp
assert sys.modules["fvv.synthesis"] is mod and fvv.synthesis is mod
assert fvv.pipeline.synthesis is mod
for n in pytest_shim._OVERRIDE:
    assert getattr(mod, n) is getattr(ours, n), n
# names the reference tests touch (tests/test_synthesis.py:8-288)
for n in ("write_debug_bundle", "CameraStreamInputs", "LAYER_BG", "view_psnr"):
    assert hasattr(mod, n), n
assert mod.write_debug_bundle is ours.write_debug_bundle   # own MVD container writer
assert fvv.depthproc.bilateral_close_holes is odp.bilateral_close_holes
print("OK")
"""
    env = {"PYTHONPATH": f"{REF_SRC}:{ROOT}", "PYTHONDONTWRITEBYTECODE": "1",
           "PATH": "/usr/bin:/bin"}
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd="/tmp")
    assert out.returncode == 0, out.stderr
    assert "OK" in out.stdout


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference package not present on this host")
def test_shim_codec_rebinding_uses_reference_types():
    code = r"""
import os
os.environ["FVV_SHIM_CODEC"] = "1"
from paper_2007_00558_b200 import pytest_shim, depthcodec as ours
pytest_shim.install()
import fvv.depthcodec as rc
for n in ("unpack_yuv420", "dequantize12", "quantize12", "pack_yuv420", "encode_lossless",
          "decode_lossless"):
    assert getattr(rc, n) is getattr(ours, n), n
for n in ("EncodedFrame", "Yuv420Image", "DisparityMap12", "DecodeError",
          "UnsupportedCodecError"):
    assert getattr(ours, n) is getattr(rc, n), n
assert ours._COMPRESSORS is rc._COMPRESSORS    # codecs registered on either side
print("OK")
"""
    env = {"PYTHONPATH": f"{REF_SRC}:{ROOT}", "PYTHONDONTWRITEBYTECODE": "1",
           "PATH": "/usr/bin:/bin"}
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd="/tmp")
    assert out.returncode == 0, out.stderr
    assert "OK" in out.stdout


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference package not present on this host")
def test_shim_rebinds_mvd_container_on_request():
    code = r"""
import os
os.environ["FVV_SHIM_MVDIO"] = "1"
import fvv.pipeline
from paper_2007_00558_b200 import pytest_shim, mvdio as ours
pytest_shim.install()
import fvv.mvdio
for n in ("rle_encode", "rle_decode", "MvdWriter", "MvdReader"):
    assert getattr(fvv.mvdio, n) is getattr(ours, n), n
assert fvv.pipeline.MvdWriter is ours.MvdWriter
print("OK")
"""
    env = {"PYTHONPATH": f"{REF_SRC}:{ROOT}", "PYTHONDONTWRITEBYTECODE": "1",
           "PATH": "/usr/bin:/bin"}
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd="/tmp")
    assert out.returncode == 0, out.stderr
    assert "OK" in out.stdout

