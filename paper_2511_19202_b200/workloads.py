"""Synthetic composed scenes and camera paths for BASELINE.json configs 1-5.

All seeded (numpy default_rng) and built from the reference generators
(synth.py) followed by prepare() (60 degree diagonal FoV, p = 0.9 / 0.05),
as SURVEY §8d specifies.  Visibility models are random He-uniform inits
(no trained weights exist offline); their output bias is calibrated so the
MLP keeps ~``keep_target`` of uniformly distributed queries, and recorded.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import synth
from .asset import prepare
from .camera import Camera
from .nn import VisibilityModel, make_model
from .scene import ComposedScene, InstanceTransform


def random_unit_quats(rng, n):
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def calibrated_model(asset, seed: int, keep_target: float | None = 0.65) -> VisibilityModel:
    """Random-init model whose output bias keeps ~keep_target of uniform [-1, 1]^16 queries."""
    m = make_model(asset, seed=seed)
    if keep_target is not None:
        rng = np.random.default_rng(10_000 + seed)
        x = rng.uniform(-1.0, 1.0, size=(20_000, 16))
        lg = m.vis_mlp.forward_host(x)[:, 0]
        bias = -float(np.quantile(lg, 1.0 - keep_target))
        m.vis_mlp.biases[-1] = np.full(1, bias, dtype=np.float32)
        m.meta["output_bias"] = bias
        m.meta["keep_target"] = keep_target
    return m


@dataclass
class Workload:
    name: str
    scene: ComposedScene
    cameras: list[Camera]
    meta: dict = field(default_factory=dict)


def config1(n: int = 10_000, size: int = 256, with_model: bool = True, seed: int = 0) -> Workload:
    """Single asset (~10K), one identity instance, random-init MLP, one 256^2 view."""
    a = prepare(synth.make_random_cloud(n, seed=seed))
    sc = ComposedScene()
    sc.add_asset(a, calibrated_model(a, seed) if with_model else None)
    sc.add_instance(0, InstanceTransform())
    cam = Camera.look_at([1.5 * a.d_near, 0.35 * a.d_near, 0.25 * a.d_near], [0, 0, 0], math.radians(50),
                         size, size)
    return Workload("cfg1", sc, [cam], {"asset": f"make_random_cloud({n}, seed={seed})", "instances": 1})


def config2(n: int = 100_000, grid: int = 4, width: int = 1920, height: int = 1080, frames: int = 120,
            with_model: bool = True, seed: int = 0) -> Workload:
    """Shell of n Gaussians x grid^2 instances (spacing 4 r), 1080p orbit (radius 22, height 10)."""
    a = prepare(synth.make_shell(n, seed=seed))
    r = a.bound_radius
    sc = ComposedScene()
    sc.add_asset(a, calibrated_model(a, seed) if with_model else None)
    rng = np.random.default_rng(seed + 100)
    quats = random_unit_quats(rng, grid * grid)
    sp = 4.0 * r
    k = 0
    for i in range(grid):
        for j in range(grid):
            t = [(i - (grid - 1) / 2.0) * sp, (j - (grid - 1) / 2.0) * sp, 0.0]
            sc.add_instance(0, InstanceTransform(t, quats[k], 1.0))
            k += 1
    cams = []
    for f in range(frames):
        ang = 2.0 * math.pi * f / frames
        cams.append(Camera.look_at([22.0 * math.cos(ang), 22.0 * math.sin(ang), 10.0], [0, 0, 0],
                                   math.radians(45), width, height))
    return Workload("cfg2", sc, cams, {"asset": f"make_shell({n}, seed={seed})", "instances": grid * grid,
                                       "orbit": "radius 22, height 10, fov_y 45"})


def _cfg3_assets(n_per: int, seed: int):
    out = []
    for k in range(8):
        kind = k % 3
        if kind == 0:
            a = synth.make_shell(n_per, seed=seed + k)
            desc = f"make_shell({n_per}, seed={seed + k})"
        elif kind == 1:
            a = synth.make_slab_pair(n_per // 2, n_per - n_per // 2, seed=seed + k)
            desc = f"make_slab_pair({n_per // 2}, {n_per - n_per // 2}, seed={seed + k})"
        else:
            a = synth.make_random_cloud(n_per, seed=seed + k)
            desc = f"make_random_cloud({n_per}, seed={seed + k})"
        out.append((prepare(a), desc))
    return out


def config3(n_per: int = 100_000, n_instances: int = 1000, width: int = 1920, height: int = 1080,
            with_model: bool = True, seed: int = 0, keep_target: float | None = 0.65) -> Workload:
    """~1,000 instances of 8 synthetic assets (~100M instantiated), near / mid / far views.

    Layout: jittered square grid on the z = 0 plane (pitch 6 units), seeded
    quaternions, scale in [0.5, 2].  Cameras: near (inside the layout, low),
    mid and far (whole layout in view).
    """
    assets = _cfg3_assets(n_per, seed)
    sc = ComposedScene()
    for k, (a, _d) in enumerate(assets):
        sc.add_asset(a, calibrated_model(a, seed + k, keep_target) if with_model else None)
    rng = np.random.default_rng(seed + 1000)
    side = int(math.ceil(math.sqrt(n_instances)))
    pitch = 6.0
    per_asset = [[] for _ in range(8)]
    for i in range(n_instances):
        gx, gy = i % side, i // side
        t = np.array([(gx - (side - 1) / 2.0) * pitch + rng.uniform(-1.5, 1.5),
                      (gy - (side - 1) / 2.0) * pitch + rng.uniform(-1.5, 1.5),
                      rng.uniform(-1.0, 1.0)])
        q = random_unit_quats(rng, 1)[0]
        s = float(np.exp(rng.uniform(math.log(0.5), math.log(2.0))))
        per_asset[int(rng.integers(0, 8))].append(InstanceTransform(t, q, s))
    for k in range(8):
        for tr in per_asset[k]:
            sc.add_instance(k, tr)
    half = side * pitch / 2.0
    cams = [
        Camera.look_at([0.15 * half, -0.35 * half, 6.0], [0.0, 0.3 * half, 0.0], math.radians(60), width, height),
        Camera.look_at([0.0, -1.4 * half, 0.9 * half], [0, 0, 0], math.radians(50), width, height),
        Camera.look_at([0.0, -2.6 * half, 1.8 * half], [0, 0, 0], math.radians(45), width, height),
    ]
    return Workload("cfg3", sc, cams, {"assets": [d for _a, d in assets], "instances": n_instances,
                                       "instantiated": sc.n_instantiated, "views": ["near", "mid", "far"],
                                       "layout": "jittered grid pitch 6, s in [0.5, 2]", "seed": seed})


def camera_path(wl: Workload, frames: int, width: int, height: int) -> list[Camera]:
    """Orbit around the layout centre at the mid view's distance (configs 2/5 style paths)."""
    mid = wl.cameras[min(1, len(wl.cameras) - 1)]
    rad = float(np.hypot(mid.position[0], mid.position[1]))
    z = float(mid.position[2])
    out = []
    for f in range(frames):
        ang = -math.pi / 2.0 + 2.0 * math.pi * f / frames
        out.append(Camera.look_at([rad * math.cos(ang), rad * math.sin(ang), z], [0, 0, 0], mid.fov_y, width,
                                  height))
    return out


def config5(frames: int = 120, width: int = 3840, height: int = 2160, **kw) -> Workload:
    """Config 5: the config-3 scene (~100M instantiated) on a 4K orbit camera path
    (sharded by frames or screen bands across GPUs)."""
    wl = config3(width=width, height=height, **kw)
    cams = camera_path(wl, frames, width, height)
    meta = dict(wl.meta)
    meta.update({"views": f"{frames}-frame orbit at the mid view's distance", "resolution": f"{width}x{height}"})
    return Workload("cfg5", wl.scene, cams, meta)
