"""Per-tile blend work statistics with the instrumented library (profiling only).

    SPLATCULL_B200_DEBUG_LIB=1 python scripts/blend_stats.py [view]
"""
import ctypes
import os
import sys

os.environ["SPLATCULL_B200_DEBUG_LIB"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_19202_b200 import _native as nat
from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

view = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = workloads.config3()
r = Renderer(wl.scene)
cam = wl.cameras[view]
r.render(cam, to_host=False)
lib = nat.load()
fn = lib.sc_debug_blend_stats
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
n_tiles = ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
torch.cuda.synchronize()
fn(None, n_tiles, 1)
torch.cuda.synchronize()
_, st = r.render(cam, to_host=False)
torch.cuda.synchronize()
buf = np.zeros((n_tiles, 8), dtype=np.uint64)
assert fn(buf.ctypes.data_as(ctypes.c_void_p), n_tiles, 0) == 0
ent, bat, hits, evals, cyc = (buf[:, i].astype(np.float64) for i in range(5))
print(st)
print(f"tiles {n_tiles}, entries {ent.sum():.3e}, batches walked {bat.sum():.3e} "
      f"(full walk {np.ceil(ent / 256).sum():.3e})")
iters = buf[:, 5].astype(np.float64)
print(f"warp hits {hits.sum():.3e}  pixel evals {evals.sum():.3e}  warp iterations {iters.sum():.3e}  "
      f"lane efficiency {evals.sum() / max(1, 32 * iters.sum()):.3f}")
order = np.argsort(-cyc)
print("cycles: total %.3e  max %.3e  p99 %.3e  median(nonempty) %.3e" %
      (cyc.sum(), cyc.max(), np.percentile(cyc, 99), np.median(cyc[ent > 0])))
print("entries per tile: max %d p99 %d median(nonempty) %d nonempty tiles %d" %
      (ent.max(), np.percentile(ent, 99), np.median(ent[ent > 0]), (ent > 0).sum()))
print("top tiles: tile entries batches hits evals Mcycles")
for t in order[:12]:
    print(f"  {t:6d} {ent[t]:9.0f} {bat[t]:7.0f} {hits[t]:9.0f} {evals[t]:10.0f} {cyc[t] / 1e6:8.2f}")
np.save("gpurun_out/blend_stats_view%d.npy" % view, buf)
