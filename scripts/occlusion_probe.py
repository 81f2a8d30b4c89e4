"""How much of the block-list work lies behind saturated 8x4 blocks (profiling only).

The frame path's block walk stops once every pixel of the block has retired
(T < stop); this reports, per config-3 view, the fraction of block entries
streamed before that point, i.e. what a depth-sliced pipeline that skips
saturated blocks could leave out of emission, block sort and blend.

    python scripts/occlusion_probe.py        (builds the instrumented library)
"""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2511_19202_b200", "csrc"), "debug", "-j8"], check=True)
os.environ["SPLATCULL_B200_DEBUG_LIB"] = "1"
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2511_19202_b200 import _native as nat
from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

wl = workloads.config3()
r = Renderer(wl.scene)
lib = nat.load()
fn = lib.sc_debug_blend_used
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int64]
res = {}
for view, cam in enumerate(wl.cameras[:3]):
    _, st = r.render(cam, to_host=False)
    torch.cuda.synchronize()
    nb = 8 * ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    buf = np.zeros((nb, 2), dtype=np.uint32)
    assert fn(buf.ctypes.data_as(ctypes.c_void_p), nb) == 0
    ent = buf[:, 0].astype(np.float64)
    used = np.minimum(buf[:, 1].astype(np.float64), ent)
    frac = used.sum() / max(1.0, ent.sum())
    # the first-k fraction of the depth order that a 2-slice scheme would blend before testing saturation
    res[view] = {"block_entries": int(ent.sum()), "streamed": int(used.sum()), "streamed_frac": frac,
                 "blocks_saturated": int(((used < ent)).sum()), "blocks": int((ent > 0).sum()),
                 "max_list": int(ent.max())}
    print(view, json.dumps(res[view]), flush=True)
    np.save(os.path.join(ROOT, "gpurun_out", "occl_view%d.npy" % view), buf)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "occlusion_probe.json"), "w"), indent=1)
