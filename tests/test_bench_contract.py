"""bench.py's JSON-line contract: the keys the driver and the judge read, for
the product arm (GPU, small c0 run) and the reference arm (CPU: the C oracle
port of the reference path on the host's cores)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _run(args, env_extra=None, timeout=900):
    env = dict(os.environ, **(env_extra or {}))
    out = subprocess.run([sys.executable, "bench.py", *args], cwd=ROOT, env=env,
                         capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def _common(d):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"):
        assert k in d, k
    assert d["unit"] == "views/s" and d["higher_is_better"] is True and d["value"] > 0
    assert "workload" in d["config"]
    e = d["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k


def test_reference_arm_contract():
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "0"],
             {"FVV_REF_BUDGET_S": "60"})
    _common(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["sample"]
    assert cb["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    # the same workload description as the product arm's (bench.workload_config)
    assert set(d["config"]) == {"workload", "mode", "path"}
    assert d["config"]["workload"].startswith("c1: 1920x1080, 9 cams, 3 refs/view")
    assert d["config"]["mode"] == "parity (reference semantics)"


@pytest.mark.gpu
def test_product_arm_contract(cuda):
    d = _run(["--config", "c0", "--steps", "5", "--warmup", "3", "--no-cpu-baseline"])
    _common(d)
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac"):
        assert k in r, k
    assert r["bound"] in ("hbm", "tensor") and 0 < r["frac"] < 1
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert "sm_mhz" in c and "reasons" in c
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert set(d["config"]) == {"workload", "mode", "path"}
    for k in ("roofline_atomic", "kernels", "rank_ms", "e2e_mm", "setup"):
        assert k in d, k
    assert d["roofline_atomic"]["atomics_per_launch"] > 0
