"""Build kernel-variant libraries for A/B timing on the GPU box.

    python tools/variants.py NAME=-DFLAG=1,-DOTHER=2 ...   -> build/variants/NAME.so
    (on the box) FVV_B200_LIB=build/variants/NAME.so python profiles/microbench.py
"""
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2007_00558_b200.build import ARCH, CSRC, SOURCES, nvcc  # noqa: E402

out = ROOT / "build" / "variants"
out.mkdir(parents=True, exist_ok=True)
procs = []
for spec in sys.argv[1:]:
    name, _, flags = spec.partition("=")
    cmd = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off", "-shared",
           *[f for f in flags.split(",") if f], "-o", str(out / f"{name}.so"),
           *[str(CSRC / s) for s in SOURCES]]
    procs.append((name, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
for name, p in procs:
    o = p.communicate()[0].decode()
    print(name, "ok" if p.returncode == 0 else "FAILED\n" + o)
