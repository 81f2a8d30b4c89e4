"""Pipelined-pass variance probe: K frames at F in flight, per-frame events on the
frame's stream, repeated; with / without the per-frame L2 flush."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

wl = workloads.config3()
cams = wl.cameras
r = Renderer(wl.scene)
F, K = 2, 30
for c in cams:
    r.render(c, to_host=False)
PRIO = os.environ.get("PIPE_PRIO") == "1"
streams = [torch.cuda.Stream(priority=(-1 if (PRIO and j == 0) else 0)) for j in range(F)]
pf = [[None] * 3 for _ in range(F)]
for j in range(1, F):
    for ci in range(3):
        pf[j][ci] = r.render_device(cams[ci], slot=j)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run(do_flush):
    main = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fe = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    e0.record()
    for st in streams:
        st.wait_stream(main)
    for i in range(K):
        j = i % F
        with torch.cuda.stream(streams[j]):
            if do_flush:
                flush.fill_(i & 0xFF)
            fe[i][0].record()
            pf[j][i % 3] = r.render_device(cams[i % 3], out=pf[j][i % 3], slot=j)
            fe[i][1].record()
    for st in streams:
        main.wait_stream(st)
    e1.record()
    torch.cuda.synchronize()
    per = [a.elapsed_time(b) for a, b in fe]
    return e0.elapsed_time(e1) / K, per


sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

for rep in range(3):
    for clk in (False,):
        if clk:
            with bench.ClockSampler(0) as cs:
                ms, per = run(True)
            info = cs.summary()
        else:
            ms, per = run(True)
            info = ""
        print(f"sampler={clk}: {ms:.2f} ms/frame ({1000 / ms:.1f} FPS)  per-frame min/med/max "
              f"{min(per):.1f}/{np.median(per):.1f}/{max(per):.1f} {info}", flush=True)
