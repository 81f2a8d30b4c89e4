"""Render warm-up frames, then one frame inside an NVTX range 'frame' (for ncu --nvtx-include frame/)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
view = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = workloads.config3() if cfg == "cfg3" else workloads.config2(frames=4)
r = Renderer(wl.scene)
cam = wl.cameras[view]
_, st = r.render(cam, to_host=False)
_, st = r.render(cam, to_host=False)
print(st, flush=True)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("frame")
r.render_device(cam)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
