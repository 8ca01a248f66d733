"""The reference's OWN tests for this path, run unmodified on the B200
backend through the pytest shim.

The reference package and its tests are staged (never committed) into
``baseline/_ref`` by ``tools/stage_reference.sh`` in the build container;
the directory travels with the repo snapshot to the GPU box. Each selection
runs in a subprocess as
``pytest -p paper_2007_00558_b200.pytest_shim <reference test files>``:
the shim rebinds ``fvv.synthesis``, the pipeline's ``synthesize_with_config``
seam and ``bilateral_close_holes`` (plus the depth codec / MVD container with
FVV_SHIM_CODEC / FVV_SHIM_MVDIO), so the reference's assertions run against
the GPU kernels. Every collected test must pass, and the run must have
launched GPU kernels."""

import os
import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "fvv").is_dir() or not (REF / "tests").is_dir(),
                                 reason="reference not staged (tools/stage_reference.sh)")]

# (selection, shim switches, tests collected from that selection)
SUITES = [
    (["test_synthesis.py"], {}, 23),
    (["test_acceptance.py::TestAcceptance::test_08_synthesis_identity_and_quality"], {}, 1),
    (["test_depthproc.py::TestBilateralCloseHoles"], {}, 6),
    (["test_depthcodec.py"], {"FVV_SHIM_CODEC": "1"}, 33),
    (["test_mvdio.py"], {"FVV_SHIM_MVDIO": "1"}, 5),
    (["test_pipeline.py"], {"FVV_SHIM_CODEC": "1", "FVV_SHIM_MVDIO": "1"}, 25),
]


@pytest.mark.parametrize("sel,switches,expected", SUITES, ids=[s[0][0] for s in SUITES])
def test_reference_tests_pass_on_the_gpu_backend(cuda, tmp_path, sel, switches, expected):
    report = tmp_path / "launches.txt"
    env = dict(os.environ, PYTHONPATH=f"{REF}{os.pathsep}{ROOT}", PYTHONDONTWRITEBYTECODE="1",
               NUMBA_CACHE_DIR=str(tmp_path / "numba"), FVV_SHIM_REPORT=str(report), **switches)
    cmd = [sys.executable, "-m", "pytest", "-p", "paper_2007_00558_b200.pytest_shim",
           "-p", "no:cacheprovider", "-q", "--rootdir", str(REF / "tests")] + \
          [str(REF / "tests" / s) for s in sel]
    out = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=1200)
    tail = out.stdout[-3000:] + out.stderr[-2000:]
    assert out.returncode == 0, tail
    m = re.search(r"(\d+) passed", out.stdout)
    assert m and int(m.group(1)) == expected, tail
    assert not re.search(r"\d+ (failed|error|skipped)", out.stdout), tail
    n = int(report.read_text())
    print(sel, f"{expected} passed, {n} GPU kernel launches")
    assert n > 0, "the reference tests did not reach the GPU backend"
