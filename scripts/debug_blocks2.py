"""Debug: frame-path (block lists) vs stage-path (tile lists) on the close camera of the parity scene."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

from paper_2511_19202_b200 import _native as nat
from paper_2511_19202_b200 import stages
from paper_2511_19202_b200.scene import Renderer, RenderOptions
from conftest import look_at
from test_gpu_parity import CAMS, _multi_scene

sc = _multi_scene(with_model=False)
cam = look_at(*CAMS[1])
r = Renderer(sc)
frame, st = r.render(cam, return_survivors=True, to_host=False)
print(nat.stats_dict(frame.stats_raw.cpu().numpy()))
ws = list(r.workspaces.values())[0]
print("caps", ws.cap_s, ws.cap_e)
out, _ = r.render(cam, return_survivors=True)
s = out.survivors
b = stages.bin_sort(r.dscene, s[:, 0], s[:, 1], cam, RenderOptions())
res = stages.blend(b["splats"], b["windows"], b["entry_idx"], b["counts"], cam, RenderOptions(), n_splats=len(s))
d = np.abs(out.image - res["image"]).max(axis=2)
ys, xs = np.nonzero(d > 1e-3)
print("bad", len(ys))
for y, x in list(zip(ys, xs))[:5]:
    print((y, x), "frame", out.image[y, x], out.final_transmittance[y, x], "tile", res["image"][y, x], res["trans"][y, x])
sp = b["splats"].cpu().numpy().view(np.uint8).reshape(-1, nat.SPLAT_BYTES)
win = b["windows"].cpu().numpy().view(np.int16).reshape(-1, 4)
f = sp[:, :24].copy().view(np.float32).reshape(-1, 6)
w = (win[:, 1] - win[:, 0]).astype(int)
print("splats", len(win), "width>100", (w > 100).sum(), "max width", w.max(), "neg x0", (win[:, 0] < 0).sum())
big = w > 100
print("sample big windows", win[big][:5].tolist(), f[big][:5, :2].tolist())
