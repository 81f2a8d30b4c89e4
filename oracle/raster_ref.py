"""Oracle for the reference render path (TEST INFRASTRUCTURE ONLY).

Restates ``splatcull.raster.render`` (reference sc/raster.py:240-339) with the
same numpy glue operations, and runs the three numba kernels through their C
restatement in ``sc_oracle.c``:

    project_kernel   sc/_kernels.py:13-134   -> orc_project
    bin_tiles        sc/_kernels.py:137-165  -> orc_bin_count / orc_bin_fill
    composite_tiles  sc/_kernels.py:168-275  -> orc_composite

Inputs are duck-typed (any object with the reference ``Asset`` / ``Camera``
attributes), so this module never imports the product package.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

# reference constants, sc/raster.py:22-25
MIN_ALPHA = 1.0 / 255.0
STOP_TRANSMITTANCE = 1.0 / 255.0
COV_DILATION = 0.3
DET_EPS = 1e-12

# real SH basis constants, sc/raster.py:30-37
SH_C0 = 0.28209479177387814
SH_C1 = 0.4886025119029199
SH_C2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
         -1.0925484305920792, 0.5462742152960396)
SH_C3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
         -0.5900435899266435)

_lib = None


def build_lib() -> str:
    """Compile sc_oracle.c (gcc, -ffp-contract=off) into oracle/liboracle.so."""
    src = os.path.join(_HERE, "sc_oracle.c")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE, "liboracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build_lib()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        i64, f64, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_int32
        L.orc_project.restype = i64
        L.orc_project.argtypes = [i64, P, P, P, P, P, f64, f64, f64, f64, i64, i64, f64, f64,
                                  P, P, P, P, P, P]
        L.orc_bin_count.restype = None
        L.orc_bin_count.argtypes = [i64, P, P, P, P, P, i64, i64, P]
        L.orc_bin_fill.restype = None
        L.orc_bin_fill.argtypes = [i64, P, P, P, P, P, i64, i64, P, P]
        L.orc_composite.restype = None
        L.orc_composite.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, i64, i64, i64, i64,
                                    f64, f64, f64, i32, P, P, P, P]
        L.orc_instantiate.restype = None
        L.orc_instantiate.argtypes = [i64, P, P, P, P, P, P, P, P, i64, P, P, P, P, P]
        L.orc_scene_cull.restype = None
        L.orc_scene_cull.argtypes = [i64, P, P, P, P, P, P, P, P, P, P, i64, f64, f64, i32, i32, f64,
                                     P, P, P]
        L.orc_margin_pad.restype = f64
        L.orc_margin_pad.argtypes = [f64]
        L.orc_mlp_forward.restype = None
        L.orc_mlp_forward.argtypes = [i64, P, P, i64, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def sigmoid(x):
    """Numerically stable logistic in float64 (sc/asset.py:44-51), numpy exp."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    nonneg = x >= 0
    out[nonneg] = 1.0 / (1.0 + np.exp(-x[nonneg]))
    e = np.exp(x[~nonneg])
    out[~nonneg] = e / (1.0 + e)
    return out


def cam_params(cam):
    """(rotation, position, focal, tan_x, tan_y) exactly as sc/raster.py:67-78."""
    focal = cam.height / (2.0 * math.tan(cam.fov_y / 2.0))
    ty = math.tan(cam.fov_y / 2.0)
    tx = ty * cam.width / cam.height
    rot = _c(cam.rotation, np.float64).reshape(3, 3)
    pos = _c(cam.position, np.float64).reshape(3)
    return rot, pos, focal, tx, ty


@dataclass
class Projection:
    mean2d: np.ndarray
    cov2d: np.ndarray
    conic: np.ndarray
    depth: np.ndarray
    radius: np.ndarray
    valid: np.ndarray
    n_skipped: int


def project(means, log_scales, quats, cam, dilation=COV_DILATION) -> Projection:
    """Stage (c) projection; inputs are upcast to f8 like sc/raster.py:158-159."""
    n = means.shape[0]
    m = _c(means, np.float64)
    ls = _c(log_scales, np.float64)
    q = _c(quats, np.float64)
    rot, pos, focal, tx, ty = cam_params(cam)
    mean2d = np.empty((n, 2))
    cov2d = np.empty((n, 3))
    conic = np.empty((n, 3))
    depth = np.empty(n)
    radius = np.empty(n)
    valid = np.empty(n, dtype=np.uint8)
    skipped = lib().orc_project(n, _p(m), _p(ls), _p(q), _p(rot), _p(pos), focal, tx, ty,
                                float(cam.near), int(cam.width), int(cam.height), float(dilation),
                                DET_EPS, _p(mean2d), _p(cov2d), _p(conic), _p(depth), _p(radius),
                                _p(valid))
    return Projection(mean2d, cov2d, conic, depth, radius, valid.astype(bool), int(skipped))


def eval_sh(sh_coeffs, sh_degree, means, cam_pos, sh_degree_eval=None):
    """Real SH colour, degrees 0..3, +0.5 and clip (sc/raster.py:198-226)."""
    deg = sh_degree if sh_degree_eval is None else min(sh_degree_eval, sh_degree)
    sh = np.asarray(sh_coeffs, dtype=np.float64)
    col = SH_C0 * sh[:, 0, :]
    if deg >= 1:
        d = np.asarray(means, dtype=np.float64) - np.asarray(cam_pos, dtype=np.float64)
        d = d / np.linalg.norm(d, axis=1, keepdims=True)
        x = d[:, 0:1]
        y = d[:, 1:2]
        z = d[:, 2:3]
        col = col - SH_C1 * y * sh[:, 1] + SH_C1 * z * sh[:, 2] - SH_C1 * x * sh[:, 3]
        if deg >= 2:
            xx, yy, zz = x * x, y * y, z * z
            xy, yz, xz = x * y, y * z, x * z
            col = (col
                   + SH_C2[0] * xy * sh[:, 4]
                   + SH_C2[1] * yz * sh[:, 5]
                   + SH_C2[2] * (2.0 * zz - xx - yy) * sh[:, 6]
                   + SH_C2[3] * xz * sh[:, 7]
                   + SH_C2[4] * (xx - yy) * sh[:, 8])
            if deg >= 3:
                col = (col
                       + SH_C3[0] * y * (3.0 * xx - yy) * sh[:, 9]
                       + SH_C3[1] * xy * z * sh[:, 10]
                       + SH_C3[2] * y * (4.0 * zz - xx - yy) * sh[:, 11]
                       + SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy) * sh[:, 12]
                       + SH_C3[4] * x * (4.0 * zz - xx - yy) * sh[:, 13]
                       + SH_C3[5] * z * (xx - yy) * sh[:, 14]
                       + SH_C3[6] * x * (xx - 3.0 * yy) * sh[:, 15])
    return np.clip(col + 0.5, 0.0, 1.0)


@dataclass
class RenderOutput:
    image: np.ndarray
    final_transmittance: np.ndarray
    contribution_max: np.ndarray | None
    contribution_sum: np.ndarray | None
    used_count: int | None
    passed_count: int
    skipped_count: int


@dataclass
class Stages:
    """Intermediates of one oracle render, for stage-level parity tests."""
    proj: Projection | None = None
    valid: np.ndarray | None = None          # after radius clip
    tx0: np.ndarray | None = None
    tx1: np.ndarray | None = None
    ty0: np.ndarray | None = None
    ty1: np.ndarray | None = None
    passed_idx: np.ndarray | None = None     # passed splats, ascending index
    order_idx: np.ndarray | None = None      # passed splats in (depth, index) order
    entry_idx: np.ndarray | None = None      # tile-binned entries
    counts: np.ndarray | None = None         # (n_tiles + 1,) segment offsets
    colors: np.ndarray | None = None
    opacity: np.ndarray | None = None
    entry_contrib: np.ndarray | None = None


def tile_rects(mean2d, radius, idx, n, n_tx, n_ty, ts):
    """Per-splat tile rectangle (sc/raster.py:297-311), int64, zero outside idx."""
    tx0 = np.zeros(n, dtype=np.int64)
    tx1 = np.zeros(n, dtype=np.int64)
    ty0 = np.zeros(n, dtype=np.int64)
    ty1 = np.zeros(n, dtype=np.int64)
    mx = mean2d[idx, 0]
    my = mean2d[idx, 1]
    r = radius[idx]
    tx0[idx] = np.clip(np.floor((mx - r) / ts).astype(np.int64), 0, n_tx)
    tx1[idx] = np.clip(np.floor((mx + r) / ts).astype(np.int64) + 1, 0, n_tx)
    ty0[idx] = np.clip(np.floor((my - r) / ts).astype(np.int64), 0, n_ty)
    ty1[idx] = np.clip(np.floor((my + r) / ts).astype(np.int64) + 1, 0, n_ty)
    return tx0, tx1, ty0, ty1


def bin_tiles(order_idx, tx0, tx1, ty0, ty1, n_tx, n_tiles):
    L = lib()
    order_idx = _c(order_idx, np.int64)
    counts = np.zeros(n_tiles + 1, dtype=np.int64)
    L.orc_bin_count(order_idx.size, _p(order_idx), _p(tx0), _p(tx1), _p(ty0), _p(ty1), n_tx,
                    n_tiles, _p(counts))
    entry_idx = np.empty(int(counts[n_tiles]), dtype=np.int64)
    L.orc_bin_fill(order_idx.size, _p(order_idx), _p(tx0), _p(tx1), _p(ty0), _p(ty1), n_tx,
                   n_tiles, _p(counts), _p(entry_idx))
    return entry_idx, counts


def render_arrays(means, log_scales, rotations, opacity_logits, sh_coeffs, sh_degree, cam, *,
                  sh_degree_eval=None, record_contributions=False, radius_clip=None,
                  tile_size=16, stop_transmittance=STOP_TRANSMITTANCE,
                  background=(1.0, 1.0, 1.0), dilation=COV_DILATION,
                  stages: Stages | None = None) -> RenderOutput:
    """``render`` on raw struct-of-arrays (sc/raster.py:240-339)."""
    h, w = int(cam.height), int(cam.width)
    n = means.shape[0]
    bg = np.asarray(background, dtype=np.float64)
    image = np.zeros((h, w, 3))
    trans = np.ones((h, w))
    contrib_sum = np.zeros((h, w)) if record_contributions else np.zeros((0, 0))
    cmax = np.zeros(n) if record_contributions else None

    def done(passed, skipped, entry_idx=None, entry_contrib=None):
        used = None
        if record_contributions:
            if entry_idx is not None and entry_idx.size:
                np.maximum.at(cmax, entry_idx, entry_contrib)
            used = int(np.count_nonzero(cmax > 0.0))
        return RenderOutput(image + trans[:, :, None] * bg, trans, cmax,
                            contrib_sum if record_contributions else None, used, passed, skipped)

    if n == 0:
        return done(0, 0)
    proj = project(means, log_scales, rotations, cam, dilation)
    valid = proj.valid.copy()
    if radius_clip is not None and radius_clip > 0.0:
        det = proj.cov2d[:, 0] * proj.cov2d[:, 2] - proj.cov2d[:, 1] ** 2
        valid &= ~(det < radius_clip)
    if stages is not None:
        stages.proj = proj
        stages.valid = valid
    idx = np.flatnonzero(valid)
    if idx.size == 0:
        return done(0, proj.n_skipped)
    ts = int(tile_size)
    n_tx = (w + ts - 1) // ts
    n_ty = (h + ts - 1) // ts
    n_tiles = n_tx * n_ty
    tx0, tx1, ty0, ty1 = tile_rects(proj.mean2d, proj.radius, idx, n, n_tx, n_ty, ts)
    idx = idx[(tx1[idx] > tx0[idx]) & (ty1[idx] > ty0[idx])]
    if stages is not None:
        stages.tx0, stages.tx1, stages.ty0, stages.ty1 = tx0, tx1, ty0, ty1
        stages.passed_idx = idx
    passed = int(idx.size)
    if passed == 0:
        return done(0, proj.n_skipped)
    order_idx = idx[np.argsort(proj.depth[idx], kind="stable")]
    entry_idx, seg = bin_tiles(order_idx, tx0, tx1, ty0, ty1, n_tx, n_tiles)
    active = np.flatnonzero(seg[1:] > seg[:-1]).astype(np.int64)
    starts = _c(seg[:-1][active], np.int64)
    ends = _c(seg[1:][active], np.int64)
    colors = eval_sh(sh_coeffs, sh_degree, means, cam.position, sh_degree_eval)
    opac = sigmoid(opacity_logits)
    log_opac = np.log(np.maximum(opac, 1e-300))
    entry_contrib = np.zeros(entry_idx.size) if record_contributions else np.zeros(0)
    if stages is not None:
        stages.order_idx, stages.entry_idx, stages.counts = order_idx, entry_idx, seg
        stages.colors, stages.opacity = colors, opac
    mean2d = _c(proj.mean2d, np.float64)
    conic = _c(proj.conic, np.float64)
    colors_c = _c(colors, np.float64)
    lib().orc_composite(active.size, _p(active), _p(starts), _p(ends), _p(entry_idx), _p(mean2d),
                        _p(conic), _p(opac), _p(log_opac), _p(colors_c), _p(proj.radius), h, w, ts,
                        n_tx, float(stop_transmittance), MIN_ALPHA, math.log(MIN_ALPHA),
                        1 if record_contributions else 0, _p(image), _p(trans), _p(contrib_sum),
                        _p(entry_contrib))
    if stages is not None:
        stages.entry_contrib = entry_contrib
    return done(passed, proj.n_skipped, entry_idx, entry_contrib)


def render(asset, cam, **kw) -> RenderOutput:
    """Oracle ``render(asset, cam, **opts)`` (sc/raster.py:240)."""
    return render_arrays(asset.means, asset.log_scales, asset.rotations, asset.opacity_logits,
                         asset.sh_coeffs, int(asset.sh_degree), cam, **kw)


# ---------------------------------------------------------------------------
# image metrics (sc/raster.py:346-399)
# ---------------------------------------------------------------------------

def psnr(a, b, cap=99.0):
    mse = float(np.mean((np.asarray(a, np.float64) - np.asarray(b, np.float64)) ** 2))
    if mse <= 0.0:
        return cap if cap is not None else math.inf
    v = -10.0 * math.log10(mse)
    return min(cap, v) if cap is not None else v


def ssim(a, b):
    from scipy.ndimage import correlate1d
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.ndim == 2:
        a, b = a[:, :, None], b[:, :, None]
    half = 5
    xs = np.arange(-half, half + 1, dtype=np.float64)
    win = np.exp(-0.5 * xs * xs / (1.5 ** 2))
    win = win / win.sum()
    c1, c2 = 0.01 ** 2, 0.03 ** 2

    def blur(im):
        return correlate1d(correlate1d(im, win, axis=0, mode="nearest"), win, axis=1, mode="nearest")

    vals = []
    for ch in range(a.shape[2]):
        x, y = a[:, :, ch], b[:, :, ch]
        mx, my = blur(x), blur(y)
        vx = blur(x * x) - mx * mx
        vy = blur(y * y) - my * my
        cxy = blur(x * y) - mx * my
        s = ((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx ** 2 + my ** 2 + c1) * (vx + vy + c2))
        vals.append(float(np.mean(s[half:-half, half:-half])))
    return float(np.mean(vals))
