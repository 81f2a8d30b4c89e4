"""Oracle restatement of SPEC ``scene`` / ``nn`` (TEST INFRASTRUCTURE ONLY).

The reference package ships no scene / nn code, so these
stages are restated from SPEC.md:325-389 and SPEC.md:240-323 with every open
choice pinned here.  Parity status: unpinned against
reference code (none exists); pinned against the SPEC's known-answer
examples and invariants in tests/test_oracle_scene.py.

Pinned decisions
  B1  flat order: assets in scene order, each asset's instances in order,
      gaussians in asset order; survivors keep that order.
  B2  instanced gaussian: mean' = f32(s * (R m) + t) in f64 with the scalar
      association of orc_instantiate; q' = f32(q_i (x) q); log_s' =
      f32(log_s + ln s); opacity and SH unchanged (world-space SH direction on
      unrotated coefficients, exactly what flatten-then-render does).
  B3  frustum: on the f32 instanced mean, camera-space (tx, ty, tz) as the
      reference projection; cull if tz <= near; "margin" mode keeps a pair iff
      mx + Rb >= 0, mx - Rb < 16 n_tx, my + Rb >= 0, my - Rb < 16 n_ty with
      Rb = 3 (f / tz) s sigma_max G + pad, pad = max(3, 3 sqrt(dilation) + 1 +
      1e-6) px (3 px at the default dilation), and 16 = the render tile size —
      a superset of the splats the rasterizer passes, so culling never changes
      the image; "strict" mode
      keeps a pair iff the mean projects inside [0, W-1] x [0, H-1].
  B4  direction input: R_i^T (m' - c) / |m' - c| (camera -> gaussian, local);
      forward input: R_i^T cam.forward.
  B5  mean input: local mean / model.mean_scale.
  B6  d_r = |c - m'|; d_t = d_r * ((f_t / f_r) / s); normalised distance
      clamp(2 (d_t - d_near) / (d_far - d_near) - 1, -1, 1).
  B7  query iff a model exists and d_t >= d_near; keep iff logit >= logit(tau).
  B8  vis MLP 16->32->32->1 ReLU, feature MLP 14->32->32->6 ReLU / linear
      output; oracle evaluates both in float64 from the f32 weights.
  B9  FrameStats: instantiated = frustum_passed - mlp_culled.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import raster_ref as rr

SH_C0 = 0.28209479177387814

INSTANCE_DTYPE = np.dtype([("R", "<f8", 9), ("t", "<f8", 3), ("q", "<f8", 4), ("s", "<f8"), ("ln_s", "<f8"),
                           ("corr", "<f8"), ("fwd_local", "<f8", 3), ("asset", "<i8")])
ASSET_DTYPE = np.dtype([("offset", "<i8"), ("count", "<i8"), ("d_near", "<f8"), ("d_far", "<f8"),
                        ("bound_radius", "<f8"), ("model", "<i8")])
CAMERA_DTYPE = np.dtype([("pos", "<f8", 3), ("rot", "<f8", 9), ("focal", "<f8"), ("tan_x", "<f8"),
                         ("tan_y", "<f8"), ("near_", "<f8"), ("width", "<i8"), ("height", "<i8"),
                         ("tile_size", "<i8")])


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def quat_rotation(q):
    """Normalised quaternion and its rotation matrix (formula of sc/raster.py:111-126)."""
    w, x, y, z = (float(v) for v in q)
    n = math.sqrt(w * w + x * x + y * y + z * z)
    w, x, y, z = w / n, x / n, y / n, z / n
    R = np.array([[1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)],
                  [2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)],
                  [2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)]])
    return np.array([w, x, y, z]), R


def jacobian_bound(tan_x, tan_y):
    """G of B3: sqrt(1 + 1.69 (tan_x^2 + tan_y^2)) with 1e-5 slack."""
    return math.sqrt(1.0 + 1.69 * (tan_x * tan_x + tan_y * tan_y)) * 1.00001


def feature_inputs(asset, mean_scale):
    x = np.empty((len(asset.means), 14), dtype=np.float64)
    x[:, 0:3] = asset.means.astype(np.float64) / mean_scale
    x[:, 3:6] = np.exp(asset.log_scales.astype(np.float64)) / mean_scale
    x[:, 6:10] = asset.rotations.astype(np.float64)
    x[:, 10] = rr.sigmoid(asset.opacity_logits)
    x[:, 11:14] = SH_C0 * asset.sh_coeffs[:, 0, :].astype(np.float64) + 0.5
    return x.astype(np.float32).astype(np.float64)


def mlp_params(mlp):
    """Flat f64 parameter vector [W1, b1, W2, b2, ...] and widths."""
    parts = []
    for W, b in zip(mlp.weights, mlp.biases):
        parts += [np.asarray(W, np.float64).reshape(-1), np.asarray(b, np.float64).reshape(-1)]
    widths = [int(mlp.weights[0].shape[1])] + [int(W.shape[0]) for W in mlp.weights]
    return np.concatenate(parts), np.array(widths, dtype=np.int64)


def mlp_forward(mlp, x):
    params, widths = mlp_params(mlp)
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty((x.shape[0], int(widths[-1])))
    rr.lib().orc_mlp_forward(x.shape[0], _p(params), _p(widths), len(widths) - 1, _p(x), _p(out))
    return out


def encode_features(model, asset):
    return mlp_forward(model.feature_mlp, feature_inputs(asset, model.mean_scale))


def sigma_max(asset):
    return np.exp(asset.log_scales.max(axis=1).astype(np.float64)).astype(np.float32)


@dataclass
class CullResult:
    keep: np.ndarray          # (pairs,) u8
    flags: np.ndarray         # (pairs,) bit0 frustum pass, bit1 queried
    logit: np.ndarray         # (pairs,) f64, NaN where not queried
    pair_inst: np.ndarray     # (pairs,) instance index of each pair
    pair_gid: np.ndarray      # (pairs,) gaussian index within its asset
    surv_inst: np.ndarray
    surv_gid: np.ndarray


class SceneTables:
    """Concatenated gaussian arrays and host-derived instance records."""

    def __init__(self, scene):
        assets = [sa.asset for sa in scene.assets]
        self.assets = assets
        self.models = [sa.model for sa in scene.assets]
        counts = [len(a.means) for a in assets]
        self.offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        self.means = np.ascontiguousarray(np.concatenate([a.means for a in assets]), dtype=np.float32)
        self.sigma_max = np.ascontiguousarray(np.concatenate([sigma_max(a) for a in assets]))
        feats = []
        for a, m in zip(assets, self.models):
            feats.append(encode_features(m, a) if m is not None else np.zeros((len(a.means), 6)))
        self.features = np.ascontiguousarray(np.concatenate(feats), dtype=np.float64)
        self.flat = list(scene.flat_instances())
        model_ids, params, poffs = [], [], []
        for m in self.models:
            if m is None:
                model_ids.append(-1)
            else:
                p, w = mlp_params(m.vis_mlp)
                model_ids.append(len(params))
                poffs.append(sum(len(x) for x in params))
                params.append(p)
                self.vis_widths = w
        if not params:
            self.vis_widths = np.array([16, 32, 32, 1], dtype=np.int64)
        self.model_ids = model_ids
        self.params = np.concatenate(params) if params else np.zeros(1)
        self.param_offsets = np.array(poffs if poffs else [0], dtype=np.int64)
        self.asset_tab = np.zeros(len(assets), dtype=ASSET_DTYPE)
        for i, (a, m) in enumerate(zip(assets, self.models)):
            r = self.asset_tab[i]
            r["offset"], r["count"] = self.offsets[i], counts[i]
            if m is not None:
                r["d_near"], r["d_far"], r["bound_radius"] = m.d_near, m.d_far, m.mean_scale
            else:
                r["d_near"], r["d_far"], r["bound_radius"] = 0.0, 1.0, 1.0
            r["model"] = model_ids[i]
        self.pair_offset = np.concatenate([[0], np.cumsum([counts[a] for a, _ in self.flat])]).astype(np.int64)

    def instances(self, cam):
        tab = np.zeros(len(self.flat), dtype=INSTANCE_DTYPE)
        fwd = np.asarray(cam.rotation, dtype=np.float64)[2]
        focal = cam.height / (2.0 * math.tan(cam.fov_y / 2.0))
        for k, (ai, tr) in enumerate(self.flat):
            q, R = quat_rotation(tr.rotation)
            s = float(tr.scale)
            r = tab[k]
            r["R"] = R.reshape(-1)
            r["t"] = np.asarray(tr.translation, dtype=np.float64)
            r["q"] = q
            r["s"] = s
            r["ln_s"] = math.log(s)
            m = self.models[ai]
            r["corr"] = (m.f_train / focal) / s if m is not None else 0.0
            r["fwd_local"] = [R[0, j] * fwd[0] + R[1, j] * fwd[1] + R[2, j] * fwd[2] for j in range(3)]
            r["asset"] = ai
        return tab


def camera_record(cam, tile_size=16):
    rot, pos, focal, tx, ty = rr.cam_params(cam)
    c = np.zeros(1, dtype=CAMERA_DTYPE)
    c["pos"], c["rot"], c["focal"] = pos, rot.reshape(-1), focal
    c["tan_x"], c["tan_y"], c["near_"] = tx, ty, float(cam.near)
    c["width"], c["height"], c["tile_size"] = int(cam.width), int(cam.height), tile_size
    return c


def cull(tables: SceneTables, cam, frustum="margin", use_mlp=True, tile_size=16, dilation=0.3) -> CullResult:
    """Stages (a)+(b) for every (instance, gaussian) pair."""
    inst = tables.instances(cam)
    camr = camera_record(cam, tile_size)
    n_pairs = int(tables.pair_offset[-1])
    keep = np.zeros(n_pairs, np.uint8)
    flags = np.zeros(n_pairs, np.uint8)
    logit = np.empty(n_pairs, np.float64)
    _, _, _, tx, ty = rr.cam_params(cam)
    thr = 0.0
    ms = [m for m in tables.models if m is not None]
    if ms:
        t = ms[0].threshold
        thr = math.log(t) - math.log1p(-t)
    if frustum == "off":
        raise ValueError("the scene oracle always culls; use raster_ref.render for frustum='off'")
    rr.lib().orc_scene_cull(len(inst), _p(inst), _p(tables.pair_offset), _p(tables.asset_tab), _p(camr),
                            _p(tables.means), _p(tables.sigma_max), _p(tables.features), _p(tables.params),
                            _p(tables.param_offsets), _p(tables.vis_widths), len(tables.vis_widths) - 1,
                            jacobian_bound(tx, ty), float(dilation), 1 if frustum == "strict" else 0,
                            1 if use_mlp else 0, thr,
                            _p(keep), _p(flags), _p(logit))
    counts = np.array([len(tables.assets[a].means) for a, _ in tables.flat], dtype=np.int64)
    pair_inst = np.repeat(np.arange(len(tables.flat), dtype=np.int64), counts)
    pair_gid = np.arange(n_pairs, dtype=np.int64) - np.repeat(tables.pair_offset[:-1], counts)
    sel = np.flatnonzero(keep)
    return CullResult(keep, flags, logit, pair_inst, pair_gid, pair_inst[sel], pair_gid[sel])


def instantiate(tables: SceneTables, cam, surv_inst, surv_gid):
    """Flattened f32 survivor arrays (B2) — what render() receives."""
    inst = tables.instances(cam)
    sh_deg = max(a.sh_degree for a in tables.assets)
    k = (sh_deg + 1) ** 2
    n = len(surv_inst)
    means = np.concatenate([a.means for a in tables.assets]).astype(np.float32)
    ls = np.concatenate([a.log_scales for a in tables.assets]).astype(np.float32)
    q = np.concatenate([a.rotations for a in tables.assets]).astype(np.float32)
    op = np.concatenate([a.opacity_logits for a in tables.assets]).astype(np.float32)
    sh = np.zeros((len(means), k, 3), np.float32)
    for i, a in enumerate(tables.assets):
        sh[tables.offsets[i]:tables.offsets[i + 1], :a.sh_coeffs.shape[1]] = a.sh_coeffs
    inst_asset = np.asarray([a for a, _ in tables.flat], dtype=np.int64)
    gid_global = (np.asarray(surv_gid, np.int64) + tables.offsets[inst_asset[np.asarray(surv_inst, np.int64)]]
                  if n else np.zeros(0, np.int64))
    si = np.ascontiguousarray(surv_inst, dtype=np.int64)
    sg = np.ascontiguousarray(gid_global, dtype=np.int64)
    o_means = np.empty((n, 3), np.float32)
    o_ls = np.empty((n, 3), np.float32)
    o_q = np.empty((n, 4), np.float32)
    o_op = np.empty(n, np.float32)
    o_sh = np.empty((n, k, 3), np.float32)
    rr.lib().orc_instantiate(n, _p(si), _p(sg), _p(inst), _p(means), _p(ls), _p(q), _p(op), _p(sh), 3 * k,
                             _p(o_means), _p(o_ls), _p(o_q), _p(o_op), _p(o_sh))
    return o_means, o_ls, o_q, o_op, o_sh, sh_deg


@dataclass
class ComposedResult:
    out: rr.RenderOutput
    stats: dict
    cull: CullResult
    stages: rr.Stages


def render_composed(scene, cam, *, frustum="margin", use_mlp=True, tables: SceneTables | None = None,
                    **render_kw) -> ComposedResult:
    """Oracle render_composed: cull + MLP, instantiate survivors, raster_ref.render."""
    tables = tables or SceneTables(scene)
    c = cull(tables, cam, frustum=frustum, use_mlp=use_mlp, tile_size=render_kw.get("tile_size", 16),
             dilation=render_kw.get("dilation", rr.COV_DILATION))
    m, ls, q, op, sh, deg = instantiate(tables, cam, c.surv_inst, c.surv_gid)
    stages = rr.Stages()
    out = rr.render_arrays(m, ls, q, op, sh, deg, cam, stages=stages, **render_kw)
    fp = int(np.count_nonzero(c.flags & 1))
    culled = int(np.count_nonzero((c.flags & 1) & (c.keep == 0)))
    stats = {"frustum_passed": fp, "mlp_queried": int(np.count_nonzero(c.flags & 2)), "mlp_culled": culled,
             "instantiated": fp - culled, "passed": out.passed_count, "skipped": out.skipped_count,
             "used": out.used_count}
    return ComposedResult(out, stats, c, stages)
