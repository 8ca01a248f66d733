"""Does running frames on two streams (two private renderers) overlap K0/K1
with K2/K3? Device time per c1 step for 1 and 2 concurrent pipelines.

    python tools/overlap_probe.py
"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2007_00558_b200 import scenes  # noqa: E402
from paper_2007_00558_b200.engine import EdgeRenderer  # noqa: E402

wl = scenes.make_workload("c1")
dev = torch.device("cuda", 0)
frames = [wl.frames[0]]
staged = [{cid: (torch.from_numpy(c.rgb).to(dev), torch.from_numpy(c.mm.view(np.int16)).to(dev),
                 torch.from_numpy(c.validity).to(dev)) for cid, c in fr.items()} for fr in frames]
H, W = wl.rig[0].intrinsics.height, wl.rig[0].intrinsics.width
out = {}
for npipe in (1, 2, 3):
    engs = [EdgeRenderer(wl.rig, private=True) for _ in range(npipe)]
    for e in engs:
        for cid, c in wl.frames[0].items():
            e.set_bg_model(cid, c.bg_depth, c.bg_validity)
    streams = [torch.cuda.Stream() for _ in range(npipe)]
    imgs = [torch.empty((1, H, W, 3), dtype=torch.uint8, device=dev) for _ in range(npipe)]
    main = torch.cuda.current_stream()

    def step(s):
        i = s % npipe
        with torch.cuda.stream(streams[i]):
            engs[i].ingest_mm_many({c: staged[0][c] for c in wl.refs[0]})
            engs[i].render([wl.virtuals[0]], [wl.refs[0]], out=imgs[i])

    for s in range(10):
        step(s)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(int(2e8))
    a.record(main)
    for st in streams:
        st.wait_stream(main)
    n = 300
    for s in range(n):
        step(s)
    for st in streams:
        main.wait_stream(st)
    b.record(main)
    torch.cuda.synchronize()
    out[f"pipelines_{npipe}_us_per_step"] = round(a.elapsed_time(b) * 1e3 / n, 1)
    same = all(torch.equal(imgs[0], x) for x in imgs)
    out[f"pipelines_{npipe}_same_output"] = bool(same)
print(json.dumps(out))
