import sys, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2511_19202_b200 as pkg
from paper_2511_19202_b200 import stages
from paper_2511_19202_b200.scene import DeviceScene, RenderOptions, Renderer
from test_gpu_parity import _multi_scene, CAMS
from conftest import look_at
sc = _multi_scene(with_model=False)
for ci in range(3):
    cam = look_at(*CAMS[ci])
    r = Renderer(sc)
    out, st = r.render(cam, return_survivors=True)
    s = out.survivors
    b = stages.bin_sort(r.dscene, s[:, 0], s[:, 1], cam, RenderOptions())
    res = stages.blend(b["splats"], b["windows"], b["entry_idx"], b["counts"], cam, RenderOptions(), n_splats=len(s))
    d = np.abs(out.image - res["image"])
    print(ci, "maxdiff frame-path vs tile-path", d.max(), "bad px", (d.max(axis=2) > 1e-3).sum(), "blocks", st.max_tie_run, st.entries, st.passed)
    ys, xs = np.nonzero(d.max(axis=2) > 1e-3)
    if len(ys): print("   first bad px", list(zip(ys[:8], xs[:8])), "rows", ys.min(), ys.max(), "cols", xs.min(), xs.max())
