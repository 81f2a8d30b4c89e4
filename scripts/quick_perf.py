"""Scratch timing of configs 2 and 3 (device-resident frames, CUDA events)."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer, RenderOptions
from paper_2511_19202_b200 import _native as nat

def run(wl, cams, reps=3, opts=None):
    t0 = time.time(); r = Renderer(wl.scene); t1 = time.time()
    print(f"{wl.name}: upload {t1-t0:.2f}s, instantiated {wl.scene.n_instantiated/1e6:.1f}M", flush=True)
    for ci, cam in enumerate(cams):
        out, st = r.render(cam, opts, to_host=False)   # warm + size workspace
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(reps):
            r.render_device(cam, opts)
        ev[1].record(); torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / reps
        print(f"  view {ci}: {ms:.3f} ms/frame ({1000/ms:.1f} FPS) | vis inst {st.instances_visible} pairs {st.pairs_tested/1e6:.1f}M "
              f"frustum {st.frustum_passed/1e6:.2f}M queried {st.mlp_queried/1e6:.2f}M culled {st.mlp_culled/1e6:.2f}M "
              f"surv {st.instantiated/1e6:.2f}M passed {st.passed/1e6:.2f}M entries {st.entries/1e6:.2f}M tie {st.max_tie_run}", flush=True)
    ws = list(r.workspaces.values())
    print("  workspace GB", [round(w.nbytes/1e9, 2) for w in ws], "peak alloc GB", torch.cuda.max_memory_allocated()/1e9, flush=True)

wl2 = workloads.config2(frames=8)
run(wl2, wl2.cameras[::2])
which = sys.argv[1] if len(sys.argv) > 1 else "full"
if which == "full":
    wl3 = workloads.config3()
else:
    wl3 = workloads.config3(n_per=20_000, n_instances=200)
run(wl3, wl3.cameras)
print("launches", nat.load().sc_kernel_launches())
