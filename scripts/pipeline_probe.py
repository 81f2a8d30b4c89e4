"""Probe: per-frame event sum vs whole-region time, and two frames in flight on two streams."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

wl = workloads.config3()
rs = [Renderer(wl.scene), Renderer(wl.scene)]
cams = wl.cameras
for r in rs:
    for c in cams:
        r.render(c, to_host=False)
torch.cuda.synchronize()
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
K = 30
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for depth, do_flush in ((1, False), (1, True), (2, False)):
    outs = [[None] * 3, [None] * 3]
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in streams:
        s.wait_event(e0)
    t0 = time.perf_counter()
    for i in range(K):
        k = i % depth
        with torch.cuda.stream(streams[k]):
            if do_flush:
                flush.fill_(i & 0xFF)
            evs[i][0].record()
            outs[k][i % 3] = rs[k].render_device(cams[i % 3], out=outs[k][i % 3])
            evs[i][1].record()
    host = time.perf_counter() - t0
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    fsum = sum(a.elapsed_time(b) for a, b in evs) / K
    print(f"in flight {depth} flush {do_flush}: region {ms:.3f} ms/frame ({1000 / ms:.1f} FPS), "
          f"sum of frame events {fsum:.3f} ms/frame, host enqueue {1000 * host / K:.3f} ms/frame", flush=True)
