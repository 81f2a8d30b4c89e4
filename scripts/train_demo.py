"""Offline pipeline at the SPEC's default sizes: extract
visibility labels for a 100K-Gaussian shell (SamplingConfig() = 14,336 renders),
train the visibility model (TrainConfig() = 5000 iterations x 2^15 samples),
score it on held-out views, then render config 2 (4x4 instances, 1080p orbit)
with the trained model, the benchmark's calibrated random-init model and no MLP.

    python scripts/train_demo.py [out.json]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2511_19202_b200 import nn, sampling, training, workloads
from paper_2511_19202_b200.raster import psnr
from paper_2511_19202_b200.scene import ComposedScene, RenderOptions, render_composed


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


wl = workloads.config2(with_model=True)
asset = wl.scene.assets[0].asset
calibrated = wl.scene.assets[0].model
sampling.extract_dataset(asset, sampling.SamplingConfig(n_directions=4, n_distances=2), n_streams=4)   # warm-up
ds, t_extract = timed(lambda: sampling.extract_dataset(asset, sampling.SamplingConfig(), n_streams=4))
cfg = training.TrainConfig()
model, t_train = timed(lambda: training.train(ds, asset, cfg))
held = sampling.extract_dataset(asset, sampling.SamplingConfig(n_directions=64, n_distances=4, seed=17), n_streams=4)
res = {"asset": "make_shell(100000, seed=0)", "extract_s": t_extract, "views": ds.n_views,
       "train_s": t_train, "train_iters_per_s": cfg.iterations / t_train, "train_cfg": cfg.__dict__,
       "final_loss": model.meta["final_loss"], "held_out": training.evaluate(model, held, asset),
       "calibrated_random_held_out": training.evaluate(calibrated, held, asset)}
path = os.path.join(ROOT, "gpurun_out", "visibility_model.scvm")
nn.save_model(model, path)
res["checkpoint_bytes"] = os.path.getsize(path)

frames = [wl.cameras[k] for k in range(0, len(wl.cameras), 12)]
rows = {}
for name, m, use in (("trained", model, True), ("calibrated_random", calibrated, True), ("no_mlp", model, False)):
    sc = ComposedScene()
    sc.add_asset(asset, m)
    for tr in wl.scene.instances[0]:
        sc.add_instance(0, tr)
    imgs, kept, fps = [], [], []
    for cam in frames:
        render_composed(sc, cam, RenderOptions(use_mlp=use))
        (out, st), dt = timed(lambda: render_composed(sc, cam, RenderOptions(use_mlp=use)))
        imgs.append(out.image)
        kept.append(1.0 - st.mlp_culled / max(1, st.mlp_queried) if use else 1.0)
        fps.append(1.0 / dt)
    rows[name] = {"imgs": imgs, "keep_rate": float(np.mean(kept)), "e2e_fps_median": float(np.median(fps))}
for name in ("trained", "calibrated_random"):
    rows[name]["psnr_vs_no_mlp_min"] = min(psnr(a, b) for a, b in zip(rows[name]["imgs"], rows["no_mlp"]["imgs"]))
for r in rows.values():
    del r["imgs"]
res["config2_frames"] = len(frames)
res["config2"] = rows
print(json.dumps(res, indent=1))
json.dump(res, open(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "train_demo.json"), "w"),
          indent=1)
