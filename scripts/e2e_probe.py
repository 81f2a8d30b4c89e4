"""Host-side cost of the public path API: render_path at F frames in flight,
wall clock per frame, and the host time spent inside launch/collect."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2511_19202_b200 as pkg
from paper_2511_19202_b200 import workloads

wl = workloads.config3()
cams = wl.cameras
for F in (1, 2, 2, 2, 2, 2, 3):
    seq = [cams[i % 3] for i in range(30)]
    list(pkg.render_path(wl.scene, seq[:6], frames_in_flight=F))   # warm (workspaces per slot)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 0
    for out, st in pkg.render_path(wl.scene, seq, frames_in_flight=F):
        n += 1
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"F={F}: {n / dt:.1f} FPS e2e", flush=True)
