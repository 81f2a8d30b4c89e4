"""Golden fixtures for the visibility-extraction path, made by running the
reference itself (sc/sampling.py) in this container:

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden_sampling.py

-> tests/golden/sampling_views.npz (build_views of two small configs) and
   tests/golden/sampling_labels.npz (extract_dataset of a 2K-Gaussian asset:
   packed labels + the .visdata bytes).  Test infrastructure only.
"""
import io
import os
import sys
import tempfile

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")   # never write into /root/reference
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
import splatcull  # noqa: E402
from splatcull import sampling, synth  # noqa: E402
from splatcull.asset import prepare  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def views_arrays(views):
    d = {"pos": [], "rot": [], "tgt": [], "dist": [], "dir": [], "aux_pos": [], "aux_rot": []}
    for v in views:
        d["pos"].append(v.camera.position)
        d["rot"].append(v.camera.rotation)
        d["tgt"].append(v.target_offset)
        d["dist"].append(v.distance)
        d["dir"].append(v.direction_unit)
        d["aux_pos"].append([a.position for a in v.aux_cameras])
        d["aux_rot"].append([a.rotation for a in v.aux_cameras])
    return {k: np.array(x, dtype=np.float64) for k, x in d.items()}


def main():
    asset = prepare(synth.make_shell(2000, seed=4))
    out = {"d_near": asset.d_near, "d_far": asset.d_far}
    for name, cfg in (("fib", sampling.SamplingConfig(n_directions=12, n_distances=3, n_aux_views=2, seed=3)),
                      ("ll", sampling.SamplingConfig(n_directions=10, n_distances=2, n_aux_views=0,
                                                     sampler_kind="longlat", offset_scale_ratio=0.5, seed=1))):
        for k, v in views_arrays(sampling.build_views(asset, cfg)).items():
            out[f"{name}_{k}"] = v
    np.savez_compressed(os.path.join(OUT, "sampling_views.npz"), **out)

    cfg = sampling.SamplingConfig(n_directions=6, n_distances=2, n_aux_views=2, image_size=64, seed=2)
    ds = sampling.extract_dataset(asset, cfg)
    with tempfile.NamedTemporaryFile(suffix=".visdata") as fh:
        ds.save(fh.name)
        raw = open(fh.name, "rb").read()
    a = asset
    np.savez_compressed(os.path.join(OUT, "sampling_labels.npz"), labels_packed=ds.labels_packed,
                        visdata=np.frombuffer(raw, np.uint8), means=a.means, log_scales=a.log_scales,
                        rotations=a.rotations, opacity_logits=a.opacity_logits, sh_coeffs=a.sh_coeffs,
                        sh_degree=a.sh_degree, d_near=a.d_near, d_far=a.d_far,
                        cfg=np.array([6, 2, 2, 64, 2]))
    print("labels", ds.labels_packed.shape, "visible fraction", ds.labels().mean())


if __name__ == "__main__":
    main()
