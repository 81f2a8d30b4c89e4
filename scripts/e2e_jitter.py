"""Per-frame host timeline of the e2e path (render_path, F in flight): wall time between
consecutive yielded frames and the host time not spent waiting, as percentiles."""
import gc
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2511_19202_b200 as pkg
from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

wl = workloads.config3()
r = Renderer(wl.scene)
wl.scene._device = r
F = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for c in wl.cameras:
    r.render(c, to_host=False)
seq = [wl.cameras[i % 3] for i in range(90)]
for _ in pkg.render_path(wl.scene, seq[:6], frames_in_flight=F):
    pass
torch.cuda.synchronize()
gc.collect()
gc.disable()
ts = []
r.path_wait_s = 0.0
t0 = time.perf_counter()
for out, st in pkg.render_path(wl.scene, seq, frames_in_flight=F):
    ts.append(time.perf_counter())
torch.cuda.synchronize()
t1 = time.perf_counter()
gc.enable()
d = np.diff(np.array([t0] + ts)) * 1e3
caps = {k: (w.cap_s, w.cap_e) for k, w in r.workspaces.items()}
top = np.argsort(-d)[:4]
print(f"F={F}: {len(seq) / (t1 - t0):.1f} FPS, frame gaps ms p50 {np.percentile(d, 50):.2f} p90 {np.percentile(d, 90):.2f} "
      f"max {d.max():.2f} (frames {top.tolist()}: {np.round(d[top], 1).tolist()}), "
      f"host busy {1e3 * ((t1 - t0) - r.path_wait_s) / len(seq):.2f} ms/frame, workspaces {caps}", flush=True)
