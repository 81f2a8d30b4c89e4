"""Scene-layout files and the orbit evaluation (SPEC.md scene module).

Layout JSON: ``{"assets": [{"id", "ply", "vismlp"?}],
"instances": [{"asset_id", "translation", "rotation_quat", "scale"}],
"camera"?: {...}}``.  Paths are relative to the layout file.  An asset entry
may carry ``"prepare": false`` plus ``"d_near"``/``"d_far"``: the PLY is then
used as stored (already pruned and recentred, so the asset hash a saved
visibility model was trained against survives the round trip); otherwise the
PLY goes through ``prepare`` (prune -> recenter -> sampling distances,
sc/asset.py:376-386).  ``save_scene`` writes that exact form.

``orbit_eval`` is the SPEC's Table 5 harness: average passed / used counts over
a circular trajectory, ground truth from contribution records of the full
asset, "ours" with the visibility model gating the same frames.
"""

from __future__ import annotations

import json
import math
import os
from dataclasses import replace

import numpy as np

from .asset import Asset, compute_sampling_distances, prepare
from .camera import Camera
from .nn import VisibilityModel, load_model, save_model
from .ply import load_ply, save_ply
from .scene import ComposedScene, InstanceTransform, RenderOptions, render_composed


def _vec(x, n, what):
    a = np.asarray(x, dtype=np.float64).reshape(-1)
    if a.shape != (n,) or not np.isfinite(a).all():
        raise ValueError(f"{what} must be {n} finite numbers")
    return a


def camera_from_dict(d: dict) -> Camera:
    """{"position", "target", "fov_y_deg", "width", "height", "near"?} -> Camera.look_at."""
    return Camera.look_at(_vec(d["position"], 3, "camera position"), _vec(d["target"], 3, "camera target"),
                          math.radians(float(d.get("fov_y_deg", 50.0))), int(d.get("width", 1920)),
                          int(d.get("height", 1080)), near=float(d.get("near", 0.05)))


def load_scene(path, fov: float = math.radians(60.0)) -> tuple[ComposedScene, Camera | None]:
    """Read a layout file -> (ComposedScene, default camera or None)."""
    base = os.path.dirname(os.path.abspath(path))
    with open(path) as fh:
        try:
            doc = json.load(fh)
        except json.JSONDecodeError as e:
            raise ValueError(f"{path}: invalid JSON ({e})") from None
    if not isinstance(doc, dict) or not isinstance(doc.get("assets"), list) or not doc["assets"]:
        raise ValueError(f"{path}: layout needs a non-empty 'assets' list")
    scene, ids = ComposedScene(), {}
    for ent in doc["assets"]:
        if "ply" not in ent or "id" not in ent:
            raise ValueError(f"{path}: asset entries need 'id' and 'ply'")
        if ent["id"] in ids:
            raise ValueError(f"{path}: duplicate asset id {ent['id']!r}")
        a = load_ply(os.path.join(base, ent["ply"]))
        if ent.get("prepare", True):
            a = prepare(a, fov=fov)
        elif "d_near" in ent and "d_far" in ent:
            a = replace(a, d_near=float(ent["d_near"]), d_far=float(ent["d_far"]))
        else:
            dn, df = compute_sampling_distances(a, fov)
            a = replace(a, d_near=dn, d_far=df)
        model = load_model(os.path.join(base, ent["vismlp"])) if ent.get("vismlp") else None
        ids[ent["id"]] = scene.add_asset(a, model)
    for k, inst in enumerate(doc.get("instances", [])):
        aid = inst.get("asset_id")
        if aid not in ids:
            raise ValueError(f"{path}: instance {k} references unknown asset id {aid!r}")
        tr = InstanceTransform(_vec(inst.get("translation", [0, 0, 0]), 3, "translation"),
                               _vec(inst.get("rotation_quat", [1, 0, 0, 0]), 4, "rotation_quat"),
                               float(inst.get("scale", 1.0)))
        scene.add_instance(ids[aid], tr)
    cam = camera_from_dict(doc["camera"]) if doc.get("camera") else None
    return scene, cam


def save_scene(scene: ComposedScene, path, camera: dict | None = None) -> None:
    """Write ``path`` plus one PLY (and .scvm when a model is attached) per asset beside it."""
    base = os.path.dirname(os.path.abspath(path))
    stem = os.path.splitext(os.path.basename(path))[0]
    assets, instances = [], []
    for k, sa in enumerate(scene.assets):
        ply = f"{stem}_asset{k}.ply"
        save_ply(sa.asset, os.path.join(base, ply))
        ent = {"id": k, "ply": ply, "prepare": False}
        if sa.asset.d_near is not None:
            ent.update(d_near=float(sa.asset.d_near), d_far=float(sa.asset.d_far))
        if sa.model is not None:
            ent["vismlp"] = f"{stem}_asset{k}.scvm"
            save_model(sa.model, os.path.join(base, ent["vismlp"]))
        assets.append(ent)
        for tr in scene.instances[k]:
            instances.append({"asset_id": k, "translation": tr.translation.tolist(),
                              "rotation_quat": tr.rotation.tolist(), "scale": tr.scale})
    doc = {"assets": assets, "instances": instances}
    if camera is not None:
        doc["camera"] = camera
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)


def orbit_cameras(asset: Asset, n_views: int, distance: float, height_frac: float = 0.0, fov_y: float | None = None,
                  size: int = 256) -> list[Camera]:
    """Circular trajectory in the z = height plane around the asset origin, looking at it."""
    if n_views < 1 or not distance > 0.0:
        raise ValueError("need n_views >= 1 and distance > 0")
    from .camera import diag_to_fov_y

    fy = diag_to_fov_y(math.radians(60.0), size, size) if fov_y is None else fov_y
    out = []
    for k in range(n_views):
        ang = 2.0 * math.pi * k / n_views
        eye = [distance * math.cos(ang), distance * math.sin(ang), height_frac * distance]
        out.append(Camera.look_at(eye, [0.0, 0.0, 0.0], fy, size, size))
    return out


def orbit_eval(asset: Asset, model: VisibilityModel, n_views: int, distance: float, size: int = 256,
               height_frac: float = 0.0) -> dict:
    """SPEC orbit_eval (supplementary Table 5): mean passed / used over an orbit.

    GT: full asset, passed = splats reaching the rasteriser, used = splats with a
    non-zero recorded contribution.  Ours: the same frames with the model gating.
    delta_passed_pct = 100 (passed_ours - passed_gt) / passed_gt.
    """
    if model is None:
        raise ValueError("orbit_eval needs a model")
    sums = {"passed_gt": 0.0, "used_gt": 0.0, "passed_ours": 0.0, "used_ours": 0.0}
    scenes = {}
    for key, m in (("gt", None), ("ours", model)):
        sc = ComposedScene()
        sc.add_asset(asset, m)
        sc.add_instance(0, InstanceTransform())
        scenes[key] = sc
    for cam in orbit_cameras(asset, n_views, distance, height_frac, size=size):
        for key, sc in scenes.items():
            out, st = render_composed(sc, cam, RenderOptions(use_mlp=key == "ours", record_contributions=True))
            sums[f"passed_{key}"] += out.passed_count
            sums[f"used_{key}"] += out.used_count
    res = {k: v / n_views for k, v in sums.items()}
    res["delta_passed_pct"] = 100.0 * (res["passed_ours"] - res["passed_gt"]) / max(res["passed_gt"], 1e-12)
    return res
