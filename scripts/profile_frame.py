"""Render warm-up frames, then frames inside an NVTX range 'frame' (for ncu --nvtx-include frame/).

    python scripts/profile_frame.py [cfg3|cfg2] [view index | all]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
which = sys.argv[2] if len(sys.argv) > 2 else "2"
wl = workloads.config3() if cfg == "cfg3" else workloads.config2(frames=4)
r = Renderer(wl.scene)
views = list(range(len(wl.cameras))) if which == "all" else [int(which)]
for v in views:
    for _ in range(2):
        _, st = r.render(wl.cameras[v], to_host=False)
    print(v, st, flush=True)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("frame")
for v in views:
    r.render_device(wl.cameras[v])
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
