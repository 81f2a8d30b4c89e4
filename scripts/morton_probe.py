"""Probe: does a spatially coherent Gaussian order inside each asset speed up the frame?
Renders config 3 as generated, and with every asset's Gaussians permuted into Morton
order of their means (same scene up to the order, so same images up to exact depth ties)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_19202_b200 import _native as nat
from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.asset import Asset
from paper_2511_19202_b200.scene import Renderer


def morton_perm(m):
    lo, hi = m.min(0), m.max(0)
    q = ((m - lo) / np.maximum(hi - lo, 1e-9) * 1023).astype(np.uint64)

    def spread(x):
        x = x & 0x3FF
        x = (x | (x << 16)) & 0x30000FF
        x = (x | (x << 8)) & 0x300F00F
        x = (x | (x << 4)) & 0x30C30C3
        x = (x | (x << 2)) & 0x9249249
        return x
    code = spread(q[:, 0]) | (spread(q[:, 1]) << 1) | (spread(q[:, 2]) << 2)
    return np.argsort(code, kind="stable")


def permuted(a: Asset) -> Asset:
    p = morton_perm(a.means.astype(np.float64))
    b = Asset(means=a.means[p], log_scales=a.log_scales[p], rotations=a.rotations[p],
              opacity_logits=a.opacity_logits[p], sh_coeffs=a.sh_coeffs[p], sh_degree=a.sh_degree,
              center_offset=a.center_offset, d_near=a.d_near, d_far=a.d_far)
    return b


def timeit(scene, cams, reps=5):
    r = Renderer(scene)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = []
    for cam in cams:
        for _ in range(2):
            r.render(cam, to_host=False)
        per = []
        fr = None
        for _ in range(reps):
            flush.zero_()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(nat.N_STAGE_EVENTS)]
            fr = r.render_device(cam, out=fr, stage_events=ev)
            torch.cuda.synchronize()
            per.append([ev[j].elapsed_time(ev[j + 1]) for j in range(4)])
        res.append(np.round(np.median(np.array(per), axis=0), 3).tolist())
    return res


wl = workloads.config3()
print("as generated:", timeit(wl.scene, wl.cameras), flush=True)
for sa in wl.scene.assets:
    sa.asset = permuted(sa.asset)
wl.scene._touch()
print("morton order:", timeit(wl.scene, wl.cameras), flush=True)
