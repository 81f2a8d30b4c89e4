"""Visibility extraction throughput: the reference's default
SamplingConfig (256 directions x 8 distances x (1 + 6 aux) renders at 256x256 =
14,336 record-mode renders) of a 100K-Gaussian asset, extracted on the GPU.

    python scripts/extract_bench.py [out.json]

The reference renders these one after another on the CPU (sc/sampling.py:294-329);
its per-render time on this host is measured on a few views by the C oracle port
and reported beside (the numba reference is not available on the GPU box).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2511_19202_b200 import sampling, synth
from paper_2511_19202_b200.asset import prepare

asset = prepare(synth.make_shell(100_000, seed=0))
cfg = sampling.SamplingConfig()
sampling.extract_dataset(asset, sampling.SamplingConfig(n_directions=4, n_distances=2), n_streams=4)   # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
ds = sampling.extract_dataset(asset, cfg, n_streams=4)
torch.cuda.synchronize()
t_gpu = time.perf_counter() - t0
renders = ds.n_views * (1 + cfg.n_aux_views)
res = {"config": "SamplingConfig() defaults: 256 dirs x 8 distances x (1 + 6 aux) renders, 256x256, 100K shell",
       "views": ds.n_views, "renders": renders, "gpu_s": t_gpu, "gpu_renders_per_s": renders / t_gpu,
       "visible_fraction": float(ds.labels().mean())}
# CPU baseline: the oracle port (numba kernels restated in C, OpenMP) on a sample of views
sys.path.insert(0, ROOT)
from oracle import raster_ref as rr

views = sampling.build_views(asset, cfg)[:4]
t0 = time.perf_counter()
for v in views:
    for cam in [v.camera] + list(v.aux_cameras):
        rr.render_arrays(asset.means, asset.log_scales, asset.rotations, asset.opacity_logits, asset.sh_coeffs,
                         asset.sh_degree, cam, record_contributions=True)
t_cpu = (time.perf_counter() - t0) / (len(views) * (1 + cfg.n_aux_views))
res.update({"cpu_s_per_render": t_cpu, "cpu_cores": os.cpu_count(),
            "cpu_extrapolated_s": t_cpu * renders, "speedup": t_cpu * renders / t_gpu})
print(json.dumps(res))
json.dump(res, open(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "extract.json"), "w"),
          indent=1)
