"""Probe: frames of config 3 rendered back to back on one stream vs. on S streams
(one Renderer / workspace per stream).  L2 flushed before each batch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

S = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = 5
wl = workloads.config3()
rs = [Renderer(wl.scene) for _ in range(S)]
cams = wl.cameras
streams = [torch.cuda.Stream() for _ in range(S)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
frames = [[None] * len(cams) for _ in range(S)]
for r in rs:
    for c in cams:
        r.render(c, to_host=False)
torch.cuda.synchronize()


def batch(concurrent):
    # S * len(cams) frames: renderer j renders every view
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush.zero_()
    ev0.record()
    cur = torch.cuda.current_stream()
    for j, r in enumerate(rs):
        st = streams[j] if concurrent else cur
        st.wait_stream(cur)
        with torch.cuda.stream(st):
            for ci, c in enumerate(cams):
                frames[j][ci] = r.render_device(c, out=frames[j][ci])
    for j in range(S):
        cur.wait_stream(streams[j])
    ev1.record()
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1) / (S * len(cams))


for mode in (False, True, False, True):
    t = np.median([batch(mode) for _ in range(reps)])
    print(f"streams={S if mode else 1}: {t:.3f} ms/frame ({1000 / t:.1f} FPS)", flush=True)
