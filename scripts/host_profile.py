"""Host-side cost of enqueuing a frame (cProfile + wall per call)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

wl = workloads.config3(n_per=20_000, n_instances=200)
r = Renderer(wl.scene)
cams = wl.cameras
out = [None] * 3
for i in range(6):
    out[i % 3] = r.render_device(cams[i % 3], out=out[i % 3])
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(30):
    out[i % 3] = r.render_device(cams[i % 3], out=out[i % 3])
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"enqueue {1000 * (t1 - t0) / 30:.3f} ms/frame (GPU done {1000 * (time.perf_counter() - t0) / 30:.3f})")
pr = cProfile.Profile()
pr.enable()
for i in range(30):
    out[i % 3] = r.render_device(cams[i % 3], out=out[i % 3])
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
