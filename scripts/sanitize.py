"""Small frames for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
config 1 (one frame, then record mode) and a shrunk config-3 scene rendered as a
camera path with two frames in flight, then one injected-survivor frame with the
debug copies, one tile-size-8 drop-in render and a stage-level bin_sort + blend.

    compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2511_19202_b200 as pkg
from paper_2511_19202_b200 import stages
from paper_2511_19202_b200.scene import RenderOptions, Renderer
from paper_2511_19202_b200.workloads import config1, config3

wl1 = config1(n=4000, size=128)
pkg.render_composed(wl1.scene, wl1.cameras[0])
pkg.render_composed(wl1.scene, wl1.cameras[0], record_contributions=True)
wl = config3(n_per=2_000, n_instances=40, width=320, height=180)
cams = [wl.cameras[i % 3] for i in range(4)]
r = Renderer(wl.scene)
for out, st in r.render_path(cams, RenderOptions(), frames_in_flight=2):
    pass
_, st, dbg = r.render(cams[2], RenderOptions(), to_host=False,
                      survivors=torch.stack([torch.zeros(3000, dtype=torch.int32),
                                             torch.arange(3000, dtype=torch.int32)], 1).cuda(), debug=True)
a = wl.scene.assets[0].asset
pkg.render(a, cams[1], tile_size=8)
ds = r.dscene
n = len(a)
b = stages.bin_sort(ds, np.zeros(n, np.int64), np.arange(n), cams[1], RenderOptions(use_mlp=False, frustum="off"))
stages.blend(b["splats"], b["windows"], b["entry_idx"], b["counts"], cams[1], RenderOptions(), n_splats=n)
torch.cuda.synchronize()
print("sanitize frames ok", st.instantiated, st.passed)
