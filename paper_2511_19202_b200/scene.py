"""Composed scenes and the instanced, occlusion-culled render path.

The reference package does not ship its ``scene`` module; this implements
SPEC.md:325-389 (InstanceTransform, ComposedScene, FrameStats, local_inputs,
render_composed) with every per-frame stage on the B200:

    sc_render_composed (libsplatcull_b200.so)
      prep     per-instance Eq. 2 factor + bounding-sphere cull
      cull     per-(instance, gaussian) frustum test, d_near gate, tcgen05 MLP,
               order-preserving survivor compaction           stages (a)+(b)
      project  instancing + EWA projection + SH on survivors  stage (c)
      bin      depth radix sort + tie-fix + tile binning      stage (d)
      blend    per-tile front-to-back compositing             stage (e)

Assets are stored once (struct-of-arrays in HBM) with a list of similarity
transforms; culled Gaussians are never instantiated in HBM.  The host only
passes the camera per frame and reads back the image and the counters.

Pinned restatement decisions (shared with oracle/scene_ref.py):
flat order (asset, instance, gaussian); instanced mean s R m + t in f64 then
f32; q' = q_i (x) q; log_s' = log_s + ln s; frustum = conservative superset
of what the rasterizer passes (``frustum="margin"``) or mean-in-image
(``"strict"``); gate d_t = |c - m'| (f_t / f_r) / s >= d_near; keep iff
logit >= logit(threshold).
"""

from __future__ import annotations

import ctypes
import math
import threading
import time
import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from . import ops
from .asset import Asset
from .nn import VisibilityModel, feature_inputs

FRUSTUM_MODES = {"margin": nat.SC_FRUSTUM_MARGIN, "strict": nat.SC_FRUSTUM_STRICT, "off": nat.SC_FRUSTUM_OFF}


@dataclass
class InstanceTransform:
    """Similarity transform: x' = s R(q) x + t."""

    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))
    rotation: np.ndarray = field(default_factory=lambda: np.array([1.0, 0.0, 0.0, 0.0]))  # (w, x, y, z)
    scale: float = 1.0

    def __post_init__(self):
        self.translation = np.asarray(self.translation, dtype=np.float64).reshape(3)
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(4)
        self.scale = float(self.scale)
        if not (self.scale > 0.0 and math.isfinite(self.scale)):
            raise ValueError(f"instance scale must be > 0, got {self.scale}")
        if not np.isfinite(self.translation).all() or not np.isfinite(self.rotation).all():
            raise ValueError("non-finite instance transform")
        n = float(np.sqrt((self.rotation ** 2).sum()))
        if abs(n - 1.0) > 1e-6:
            raise ValueError(f"instance rotation must be a unit quaternion (norm {n})")

    @classmethod
    def identity(cls) -> "InstanceTransform":
        return cls()


def instance_frame(tr: InstanceTransform) -> tuple[list[float], list[float], float, float]:
    """(R row-major, normalised q, s, ln s) with plain float64 scalar math.

    R follows the reference quaternion formula (sc/raster.py:111-126).
    """
    w, x, y, z = (float(v) for v in tr.rotation)
    n = math.sqrt(w * w + x * x + y * y + z * z)
    w, x, y, z = w / n, x / n, y / n, z / n
    R = [1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y),
         2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x),
         2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)]
    return R, [w, x, y, z], float(tr.scale), math.log(float(tr.scale))


@dataclass
class SceneAsset:
    asset: Asset
    model: VisibilityModel | None = None


class ComposedScene:
    """Assets stored once, each with a list of instance transforms."""

    def __init__(self):
        self.assets: list[SceneAsset] = []
        self.instances: list[list[InstanceTransform]] = []
        self._version = 0
        self._device = None

    def add_asset(self, asset: Asset, model: VisibilityModel | None = None) -> int:
        if len(asset) == 0:
            raise ValueError("cannot add an empty asset")
        if model is not None and model.asset_hash is not None:
            from .asset import asset_hash
            if asset_hash(asset) != model.asset_hash:
                raise ValueError("visibility model was trained for a different asset (hash mismatch)")
        self.assets.append(SceneAsset(asset, model))
        self.instances.append([])
        self._touch()
        return len(self.assets) - 1

    def add_instance(self, asset_id: int, transform: InstanceTransform | None = None) -> None:
        if not (0 <= asset_id < len(self.assets)):
            raise ValueError(f"unknown asset id {asset_id}")
        self.instances[asset_id].append(transform if transform is not None else InstanceTransform())
        self._touch()

    def set_model(self, asset_id: int, model: VisibilityModel | None) -> None:
        self.assets[asset_id].model = model
        self._touch()

    def _touch(self):
        self._version += 1
        self._device = None

    @property
    def n_instances(self) -> int:
        return sum(len(v) for v in self.instances)

    @property
    def n_instantiated(self) -> int:
        """Gaussians if every instance were flattened."""
        return sum(len(a.asset) * len(v) for a, v in zip(self.assets, self.instances))

    def flat_instances(self):
        """(asset index, transform) in flat order (asset-major)."""
        for a, lst in enumerate(self.instances):
            for tr in lst:
                yield a, tr


@dataclass
class FrameStats:
    """Per-frame counters plus device-side extras."""

    frustum_passed: int
    mlp_culled: int
    instantiated: int
    used: int | None
    mem_bytes_instantiated: int
    render_ms: float
    mlp_ms: float
    preprocess_ms: float
    mlp_queried: int = 0
    instances_visible: int = 0
    pairs_tested: int = 0
    passed: int = 0
    skipped: int = 0
    entries: int = 0
    max_tie_run: int = 0
    block_entries: int = 0
    exact_fallbacks: int = 0


@dataclass
class RenderOptions:
    """render() keywords (sc/raster.py:240-251) plus the scene-path switches."""

    sh_degree_eval: int | None = None
    record_contributions: bool = False
    radius_clip: float | None = None
    tile_size: int = 16
    stop_transmittance: float = 1.0 / 255.0
    background: tuple = (1.0, 1.0, 1.0)
    dilation: float = 0.3
    use_mlp: bool = True
    frustum: str = "margin"
    exact_projection: bool = False   # True: all-f64 projection (False: f32 covariance, exact f64 fallback)
    band: tuple | None = None        # (y0, y1) pixel rows, y0 a multiple of 16: render only this screen band

    def struct(self, cam) -> nat.ScOpts:
        ts = check_tile_size(self.tile_size)
        if self.frustum not in FRUSTUM_MODES:
            raise ValueError(f"frustum must be one of {sorted(FRUSTUM_MODES)}")
        o = nat.ScOpts()
        o.tile_size = ts
        o.sh_degree_eval = -1 if self.sh_degree_eval is None else int(self.sh_degree_eval)
        o.record_contributions = 1 if self.record_contributions else 0
        o.use_mlp = 1 if self.use_mlp else 0
        o.frustum_mode = FRUSTUM_MODES[self.frustum]
        o.exact_projection = 1 if self.exact_projection else 0
        if self.band is not None:
            if ts != 16:
                raise ValueError("screen bands need tile_size 16")
            y0, y1 = int(self.band[0]), int(self.band[1])
            if y0 < 0 or y0 % 16 or y1 <= y0 or y0 >= int(cam.height):
                raise ValueError(f"band must be (y0, y1) with 0 <= y0 < height, y0 % 16 == 0, y1 > y0; got {self.band}")
            o.band_y0, o.band_y1 = y0, min(y1, int(cam.height))
        o.radius_clip = float(self.radius_clip) if self.radius_clip is not None else 0.0
        o.stop_transmittance = float(self.stop_transmittance)
        o.background[:] = [float(v) for v in self.background]
        o.dilation = float(self.dilation)
        o.frustum_G = frustum_G(cam)
        return o


def check_tile_size(tile_size) -> int:
    """The reference accepts any positive tile size (sc/raster.py:245, :297-311); the image depends on it."""
    if isinstance(tile_size, bool) or int(tile_size) != tile_size:
        raise ValueError(f"tile_size must be an integer, got {tile_size!r}")
    ts = int(tile_size)
    if not 1 <= ts <= 65535:
        raise ValueError(f"tile_size must be in [1, 65535], got {ts}")
    return ts


def frustum_G(cam) -> float:
    """Bound on |J W| in units of f/z for the clamped Jacobian."""
    tx, ty = cam.tan_half_fov
    return math.sqrt(1.0 + 1.69 * (tx * tx + ty * ty)) * 1.00001


def appearance(asset: Asset) -> np.ndarray:
    """(n, 4) float32 per-gaussian view-independent appearance (sc_scene.appear), computed
    in f64 with the reference's formulas and rounded once:
    [p_min = ln(1/255) - ln(sigmoid(logit)) (+inf when opacity < 1/255: the reference
    skips the splat, sc/_kernels.py:215-219; sigmoid sc/asset.py:44-51),
    fp16 bits r | g << 16, fp16 bits b, 0] with the degree-0 colour
    clip(C0 f_dc + 0.5, 0, 1) (sc/raster.py:198-226 at degree 0)."""
    from .asset import SH_C0, sigmoid

    n = len(asset)
    out = np.zeros((n, 4), np.float32)
    op = sigmoid(asset.opacity_logits)
    with np.errstate(divide="ignore"):
        p_min = math.log(1.0 / 255.0) - np.log(np.maximum(op, 1e-300))
    out[:, 0] = np.where(op < 1.0 / 255.0, np.inf, p_min).astype(np.float32)
    rgb = np.clip(SH_C0 * asset.sh_coeffs[:, 0, :].astype(np.float64) + 0.5, 0.0, 1.0).astype(np.float16)
    bits = rgb.view(np.uint16).astype(np.uint32)
    out[:, 1] = (bits[:, 0] | (bits[:, 1] << 16)).view(np.float32)
    out[:, 2] = bits[:, 2].view(np.float32)
    return out


def sigma_max(asset: Asset) -> np.ndarray:
    """Per-gaussian largest std-dev exp(max log_scale), f32 (frustum margin input)."""
    return np.exp(asset.log_scales.max(axis=1).astype(np.float64)).astype(np.float32)


def vis_weights_struct(model: VisibilityModel) -> nat.ScVisWeights:
    w = nat.ScVisWeights()
    W1, W2, W3 = model.vis_mlp.weights
    b1, b2, b3 = model.vis_mlp.biases
    if W1.shape != (32, 16) or W2.shape != (32, 32) or W3.shape != (1, 32):
        raise ValueError(f"device MLP supports 16->32->32->1 only, got {model.vis_mlp.widths}")
    w.w1[:] = W1.astype(np.float16).view(np.uint16).reshape(-1).tolist()
    w.w2[:] = W2.astype(np.float16).view(np.uint16).reshape(-1).tolist()
    w.b1[:] = b1.astype(np.float32).tolist()
    w.b2[:] = b2.astype(np.float32).tolist()
    w.w3[:] = W3.reshape(-1).astype(np.float32).tolist()
    w.b3 = float(b3[0])
    return w


def feature_params(model: VisibilityModel) -> np.ndarray:
    m = model.feature_mlp
    parts = []
    for W, b in zip(m.weights, m.biases):
        parts += [W.astype(np.float32).reshape(-1), b.astype(np.float32).reshape(-1)]
    p = np.concatenate(parts)
    if m.widths != (14, 32, 32, 6):
        raise ValueError(f"device feature MLP supports 14->32->32->6 only, got {m.widths}")
    return p


class DeviceScene:
    """The scene in HBM: concatenated gaussian SoA + asset / instance / weight tables."""

    def __init__(self, scene: ComposedScene, device=None):
        import torch

        nat.load()
        self.device = torch.device(device or "cuda")
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self._scene_version = scene._version
        assets = scene.assets
        if not assets:
            raise ValueError("scene has no assets")
        counts = [len(a.asset) for a in assets]
        offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        n = int(offsets[-1])
        max_deg = max(a.asset.sh_degree for a in assets)
        sh_stride = 3 * (max_deg + 1) ** 2
        mean_opa = np.empty((n, 4), np.float32)
        quat = np.empty((n, 4), np.float32)
        scale_smax = np.empty((n, 4), np.float32)
        sh = np.zeros((n, sh_stride), np.float32)
        appear = np.zeros((n, 4), np.float32)
        arecs = (nat.ScAssetRec * len(assets))()
        models: list[VisibilityModel] = []
        feat_jobs = []
        for i, sa in enumerate(assets):
            a = sa.asset
            lo, hi = int(offsets[i]), int(offsets[i + 1])
            mean_opa[lo:hi, :3] = a.means
            mean_opa[lo:hi, 3] = a.opacity_logits
            quat[lo:hi] = a.rotations
            scale_smax[lo:hi, :3] = a.log_scales
            smax = sigma_max(a)
            scale_smax[lo:hi, 3] = smax
            k = 3 * (a.sh_degree + 1) ** 2
            sh[lo:hi, :k] = a.sh_coeffs.reshape(hi - lo, k)
            appear[lo:hi] = appearance(a)
            r = arecs[i]
            r.offset, r.count = lo, hi - lo
            r.bound_local = float(np.sqrt((a.means.astype(np.float64) ** 2).sum(axis=1)).max())
            r.sigma_max = float(smax.astype(np.float64).max())
            r.sh_degree = a.sh_degree
            m = sa.model
            if m is not None:
                r.model = len(models)
                models.append(m)
                r.d_near, r.d_far = float(m.d_near), float(m.d_far)
                r.inv_mean_scale = 1.0 / float(m.mean_scale)
                r.f_train = float(m.f_train)
                r.logit_threshold = float(m.logit_threshold)
                feat_jobs.append((lo, hi, m, a))
            else:
                r.model = -1
                r.d_near = float(a.d_near) if a.d_near is not None else 0.0
                r.d_far = float(a.d_far) if a.d_far is not None else 1.0
                r.inv_mean_scale = 1.0
                r.f_train = 0.0
                r.logit_threshold = 0.0
        flat = list(scene.flat_instances())
        irecs = (nat.ScInstanceRec * max(1, len(flat)))()
        for k, (ai, tr) in enumerate(flat):
            R, q, s, ln_s = instance_frame(tr)
            rec = irecs[k]
            rec.R[:] = R
            rec.t[:] = [float(v) for v in tr.translation]
            rec.q[:] = q
            rec.s, rec.ln_s = s, ln_s
            rec.asset = ai
        wrecs = (nat.ScVisWeights * max(1, len(models)))()
        for k, m in enumerate(models):
            wrecs[k] = vis_weights_struct(m)

        dev = self.device
        with torch.cuda.device(dev):
            self._upload(mean_opa, quat, scale_smax, sh, appear, arecs, irecs, wrecs, n, flat, models, counts,
                         offsets, sh_stride, feat_jobs, assets)

    def _upload(self, mean_opa, quat, scale_smax, sh, appear, arecs, irecs, wrecs, n, flat, models, counts, offsets,
                sh_stride, feat_jobs, assets):
        import torch

        dev = self.device
        T = torch.from_numpy
        self.mean_opa = T(mean_opa).to(dev)
        self.quat = T(quat).to(dev)
        self.scale_smax = T(scale_smax).to(dev)
        self.sh = T(sh).to(dev)
        self.appear = T(appear).to(dev)
        self.features = torch.zeros((max(n, 1), 8), dtype=torch.float16, device=dev)
        self.assets_t = nat.struct_tensor(arecs, dev)
        self.instances_t = nat.struct_tensor(irecs, dev)
        self.weights_t = nat.struct_tensor(wrecs, dev)
        self.n_gauss, self.n_instances, self.n_models = n, len(flat), len(models)
        self.max_pairs = int(sum(counts[ai] for ai, _ in flat))
        self.sh_stride = sh_stride
        self.asset_offsets = offsets
        self.inst_asset = np.array([ai for ai, _ in flat], dtype=np.int64)
        self.scene_version = self._scene_version
        for lo, hi, m, a in feat_jobs:
            self.features[lo:hi] = encode_features_device(m, a, dev)
        self.struct = nat.ScScene()
        s = self.struct
        s.mean_opa, s.quat, s.scale_smax = nat.ptr(self.mean_opa), nat.ptr(self.quat), nat.ptr(self.scale_smax)
        s.sh, s.features = nat.ptr(self.sh), nat.ptr(self.features)
        s.n_gauss, s.sh_stride, s.n_assets = n, sh_stride, len(assets)
        s.assets, s.instances, s.n_instances = nat.ptr(self.assets_t), nat.ptr(self.instances_t), len(flat)
        s.vis_weights, s.n_models = nat.ptr(self.weights_t), len(models)
        s.n_pairs = self.max_pairs
        s.appear = nat.ptr(self.appear)
        self.nbytes = sum(int(t.numel() * t.element_size()) for t in
                          (self.mean_opa, self.quat, self.scale_smax, self.sh, self.features, self.appear,
                           self.assets_t, self.instances_t, self.weights_t))
        # packed form for torch.ops.splatcull (ops.py)
        self.op_scene = [self.mean_opa, self.quat, self.scale_smax, self.sh, self.features, self.appear,
                         self.assets_t, self.instances_t, self.weights_t]
        self.op_meta = [n, sh_stride, len(assets), len(flat), len(models), self.max_pairs]
        self.payload_bytes = [44 + 12 * (a.asset.sh_degree + 1) ** 2 for a in assets]


def encode_features_device(model: VisibilityModel, asset: Asset, device) -> "torch.Tensor":
    """nn.encode_features on the GPU (torch.ops.splatcull.encode_features): (n, 8) fp16 (6 used)."""
    import torch

    nat.load()
    x = torch.from_numpy(feature_inputs(asset, model.mean_scale)).to(device)
    p = torch.from_numpy(feature_params(model)).to(device)
    with torch.cuda.device(x.device):
        return ops.encode_features(p, x)


class Workspace:
    """Device workspace sized from the previous frame's counts (grows on overflow)."""

    def __init__(self, dscene: DeviceScene, width: int, height: int, cap_s: int | None = None,
                 cap_e: int | None = None, tile_size: int = 16):
        self.dscene, self.width, self.height = dscene, int(width), int(height)
        self.tile_size = check_tile_size(tile_size)
        mp = max(1, dscene.max_pairs)
        self.cap_s = int(cap_s if cap_s is not None else min(mp, 1 << 24))
        self.cap_e = int(cap_e if cap_e is not None else max(4 * self.cap_s, 1 << 16))
        self._alloc()

    def _alloc(self):
        import torch

        lib = nat.load()
        nbytes = lib.sc_workspace_bytes(self.dscene.n_instances, self.dscene.max_pairs, self.cap_s, self.cap_e,
                                        self.width, self.height, self.tile_size)
        if nbytes == 0:
            raise ValueError("invalid workspace request")
        self.buf = torch.empty(int(nbytes), dtype=torch.uint8, device=self.dscene.device)
        self.struct = nat.ScWorkspace()
        w = self.struct
        w.base, w.bytes = nat.ptr(self.buf), int(nbytes)
        w.n_instances, w.max_pairs = self.dscene.n_instances, self.dscene.max_pairs
        w.cap_survivors, w.cap_entries = self.cap_s, self.cap_e

    def grow(self, need_s: int, need_e: int) -> None:
        # 5 % headroom: a camera path's next frames rarely need more, and an overflow only
        # costs one re-render of that frame
        self.cap_s = max(self.cap_s, int(need_s * 1.05) + 4096)
        self.cap_e = max(self.cap_e, int(need_e * 1.05) + 16384)
        self.buf = None
        self._alloc()

    @property
    def nbytes(self) -> int:
        return int(self.buf.numel())

    @property
    def op_meta(self) -> list[int]:
        w = self.struct
        return [int(w.n_instances), int(w.max_pairs), int(w.cap_survivors), int(w.cap_entries)]


@dataclass
class DeviceFrame:
    """A rendered frame still on the device (torch tensors)."""

    image: "torch.Tensor"          # (H, W, 3) f32
    trans: "torch.Tensor"          # (H, W) f32
    stats_raw: "torch.Tensor"      # sc_frame_stats bytes
    contrib_sum: "torch.Tensor | None" = None
    contrib_max: "torch.Tensor | None" = None
    survivors: "torch.Tensor | None" = None


class _PinnedPool:
    """Pinned host buffers for the per-frame device->host copies, recycled once
    the numpy arrays handed out over them are garbage-collected (a fresh
    pinned allocation of a 1080p image costs ~1.5 ms of host time, about what
    the frame's GPU work leaves the host per frame).  At most ``limit_bytes``
    of pinned memory stays handed out: beyond that (a caller keeping many
    frames alive) the arrays are copied into pageable memory and the pinned
    buffer returns to the pool at once."""

    def __init__(self, limit_bytes: int = 2 << 30):
        self._free: dict = {}
        self._lock = threading.Lock()
        self.limit_bytes = int(limit_bytes)
        self.out_bytes = 0

    def take(self, shape, dtype):
        import torch

        key = (tuple(shape), dtype)
        with self._lock:
            lst = self._free.get(key)
            if lst:
                return lst.pop()
        return torch.empty(tuple(shape), dtype=dtype, pin_memory=True)

    def give(self, t) -> None:
        with self._lock:
            self._free.setdefault((tuple(t.shape), t.dtype), []).append(t)

    def _release(self, t, nbytes: int) -> None:
        with self._lock:
            self.out_bytes -= nbytes
        self.give(t)

    def numpy(self, t):
        """numpy view of pinned ``t`` (``t`` returns to the pool when the view is collected),
        or a pageable copy once ``limit_bytes`` of pinned memory is handed out."""
        nbytes = t.numel() * t.element_size()
        with self._lock:
            keep = self.out_bytes + nbytes <= self.limit_bytes
            if keep:
                self.out_bytes += nbytes
        if not keep:
            a = t.numpy().copy()
            self.give(t)
            return a
        a = t.numpy()
        weakref.finalize(a, self._release, t, nbytes)
        return a


_PINNED = _PinnedPool()


def _to_pinned(t):
    """Asynchronous device->host copy into a pooled pinned tensor (caller synchronises)."""
    h = _PINNED.take(t.shape, t.dtype)
    h.copy_(t, non_blocking=True)
    return h


class _StageEvents:
    """Five timing events the library records at the stage boundaries of one frame
    (frame start, after cull + MLP, projection, sort / binning, blend), reused
    frame after frame by one workspace slot."""

    def __init__(self):
        import torch

        self.events = [torch.cuda.Event(enable_timing=True) for _ in range(nat.N_STAGE_EVENTS)]
        for ev in self.events:
            ev.record()   # torch creates the CUDA event lazily
        self.handles = (ctypes.c_void_p * nat.N_STAGE_EVENTS)(*[ev.cuda_event for ev in self.events])

    def timings(self) -> tuple[float, float, float]:
        """(render_ms, mlp_ms, preprocess_ms) of the last recorded frame (its events have completed):
        the whole frame, the cull + MLP stage, and projection + sort / binning."""
        e = self.events
        return (float(e[0].elapsed_time(e[4])), float(e[0].elapsed_time(e[1])), float(e[1].elapsed_time(e[3])))


def _frame_stats(st: dict, timings, payload: int, record: bool) -> FrameStats:
    render_ms, mlp_ms, pre_ms = timings
    return FrameStats(frustum_passed=st["frustum_passed"], mlp_culled=st["mlp_culled"], instantiated=st["survivors"],
                      used=st["used"] if record else None, mem_bytes_instantiated=payload, render_ms=render_ms,
                      mlp_ms=mlp_ms, preprocess_ms=pre_ms, mlp_queried=st["mlp_queried"],
                      instances_visible=st["instances_visible"], pairs_tested=st["pairs_tested"], passed=st["passed"],
                      skipped=st["skipped"], entries=st["entries"], max_tie_run=st["max_tie_run"],
                      block_entries=st["block_entries"], exact_fallbacks=st["exact_fallbacks"])


class FrameDebug:
    """Device buffers for the frame path's internals (sc_frame_debug): the
    (depth, index) order of the passed survivors and the per-(16x16 tile, 8x4
    block) entry lists the blend walks.  Parity tests only."""

    def __init__(self, ws: Workspace):
        import torch

        dev = ws.dscene.device
        n_tiles16 = ((ws.width + 15) // 16) * ((ws.height + 15) // 16)
        self.order = torch.empty(max(ws.cap_s, 1), dtype=torch.int32, device=dev)
        self.block_offsets = torch.empty(8 * n_tiles16 + 1, dtype=torch.int32, device=dev)
        self.block_entries = torch.empty(max(ws.cap_e, 1), dtype=torch.int32, device=dev)
        self.block_codes = torch.empty(max(ws.cap_e, 1), dtype=torch.int32, device=dev)

    def host(self, stats: dict) -> dict:
        """numpy copies: order [passed], block offsets, entries / codes [block_entries] (uint32 as int64)."""
        u = lambda t, n: t[:n].cpu().numpy().view(np.uint32).astype(np.int64)   # noqa: E731
        nb = stats["block_entries"]
        return {"order": u(self.order, stats["passed"]),
                "block_offsets": u(self.block_offsets, self.block_offsets.numel()),
                "block_entries": u(self.block_entries, nb), "block_codes": u(self.block_codes, nb)}


class Renderer:
    """Renders frames of one ComposedScene on one GPU (the scene's device)."""

    def __init__(self, scene: ComposedScene, device=None):
        self.scene = scene
        self.dscene = DeviceScene(scene, device)
        self.workspaces: dict[tuple, Workspace] = {}
        self._path_streams: list = []
        self._path_frames: dict = {}
        self._events: dict = {}
        self.path_wait_s = 0.0   # host time render_path spent waiting on frames (diagnostics)

    @staticmethod
    def ws_key(cam, slot: int = 0, tile_size: int = 16) -> tuple:
        return (int(cam.width), int(cam.height), int(slot), int(tile_size))

    def workspace(self, cam, slot: int = 0, tile_size: int = 16) -> Workspace:
        """The workspace of this resolution / tile size (``slot`` > 0: one more per frame in flight)."""
        key = self.ws_key(cam, slot, tile_size)
        if key not in self.workspaces:
            base = self.workspaces.get(self.ws_key(cam, 0, tile_size)) if slot else None   # extra slots start at slot 0's
            self.workspaces[key] = Workspace(self.dscene, int(cam.width), int(cam.height),
                                             cap_s=base.cap_s if base else None, cap_e=base.cap_e if base else None,
                                             tile_size=tile_size)
        return self.workspaces[key]

    def stage_events(self, slot: int = 0) -> _StageEvents:
        if slot not in self._events:
            import torch

            with torch.cuda.device(self.dscene.device):
                self._events[slot] = _StageEvents()
        return self._events[slot]

    def render_device(self, cam, opts: RenderOptions | None = None, out: DeviceFrame | None = None,
                      return_survivors: bool = False, stage_events=None, slot: int = 0,
                      survivors=None, debug: FrameDebug | None = None) -> DeviceFrame:
        """Enqueue one frame on the current stream of the scene's device; no host synchronisation.

        ``stage_events``: optional 5 timing-enabled torch.cuda.Event objects (or a
        _StageEvents), recorded by the library at the stage boundaries (frame
        start, after cull+MLP, projection, sort/binning, blend).  ``slot``: which
        of the per-frame-in-flight workspaces to use (frames rendered
        concurrently on different streams need different slots).
        ``survivors``: an explicit (S, 2) int32 [instance, gaussian] device list
        rendered through stages (c)-(e) of the frame path instead of the cull
        (sc_render_survivors).  ``debug``: FrameDebug buffers to copy the depth
        order and block lists into.  Calls torch.ops.splatcull.render_frame_.
        """
        import torch

        opts = opts or RenderOptions()
        nat.load()
        dev = self.dscene.device
        with torch.cuda.device(dev):
            ws = self.workspace(cam, slot, opts.tile_size)
            h, w = int(cam.height), int(cam.width)
            if out is None or out.image.shape != (h, w, 3):
                out = DeviceFrame(torch.empty((h, w, 3), dtype=torch.float32, device=dev),
                                  torch.empty((h, w), dtype=torch.float32, device=dev),
                                  torch.empty(nat.STATS_BYTES, dtype=torch.uint8, device=dev))
            if opts.record_contributions:
                if out.contrib_sum is None or out.contrib_sum.shape != (h, w):
                    out.contrib_sum = torch.empty((h, w), dtype=torch.float32, device=dev)
                if out.contrib_max is None or out.contrib_max.numel() != ws.cap_s:
                    out.contrib_max = torch.empty(ws.cap_s, dtype=torch.float32, device=dev)
            if return_survivors and (out.survivors is None or out.survivors.shape[0] != ws.cap_s):
                out.survivors = torch.empty((ws.cap_s, 2), dtype=torch.int32, device=dev)
            handles: list[int] = []
            if isinstance(stage_events, _StageEvents):
                handles = [int(h) for h in stage_events.handles]
            elif stage_events is not None:
                for ev in stage_events[:nat.N_STAGE_EVENTS]:
                    if not ev.cuda_event:
                        ev.record()            # torch creates the CUDA event lazily
                    handles.append(int(ev.cuda_event))
            dbg: list = []
            if debug is not None:
                if debug.order.numel() < ws.cap_s or debug.block_entries.numel() < ws.cap_e:
                    raise ValueError("FrameDebug buffers are smaller than the workspace capacities")
                dbg = [debug.order, debug.block_offsets, debug.block_entries, debug.block_codes]
            if survivors is not None and int(survivors.shape[0]) > ws.cap_s:
                if debug is not None:
                    raise ValueError("survivor list exceeds the workspace capacity (grow it before FrameDebug)")
                ws.grow(int(survivors.shape[0]), ws.cap_e)
            cam_f, cam_i = ops.pack_camera(cam)
            opt_f, opt_i = ops.pack_opts(opts.struct(cam))
            rec = opts.record_contributions
            ops.render_frame_(self.dscene.op_scene, self.dscene.op_meta, cam_f, cam_i, opt_f, opt_i, ws.buf,
                              ws.op_meta, out.image, out.trans, out.stats_raw, out.contrib_sum if rec else None,
                              out.contrib_max if rec else None, out.survivors if return_survivors else None,
                              survivors, handles, dbg)
        return out

    def render(self, cam, opts: RenderOptions | None = None, return_survivors: bool = False,
               to_host: bool = True, survivors=None, debug: bool = False):
        """One frame -> (RenderOutput, FrameStats); regrows the workspace on overflow.

        ``debug=True`` also returns the frame path's depth order and block lists
        (a dict of numpy arrays, FrameDebug.host) as a third element.
        """
        import torch

        from .raster import RenderOutput

        opts = opts or RenderOptions()
        with torch.cuda.device(self.dscene.device):
            evs = self.stage_events(0)
            if survivors is not None:
                ws = self.workspace(cam, 0, opts.tile_size)
                if int(survivors.shape[0]) > ws.cap_s:
                    ws.grow(int(survivors.shape[0]), ws.cap_e)
            for _attempt in range(4):
                dbg = FrameDebug(self.workspace(cam, 0, opts.tile_size)) if debug else None
                frame = self.render_device(cam, opts, return_survivors=return_survivors, stage_events=evs,
                                           survivors=survivors, debug=dbg)
                # one batch of asynchronous copies into pinned host memory (torch's caching host
                # allocator), then a single synchronisation
                host = {"stats": _to_pinned(frame.stats_raw)}
                if to_host:
                    host["image"] = _to_pinned(frame.image)
                    host["trans"] = _to_pinned(frame.trans)
                torch.cuda.current_stream().synchronize()
                st = nat.stats_dict(host["stats"].numpy())
                _PINNED.give(host["stats"])
                if not st["overflow"]:
                    break
                # the frame path bins (splat, 8x4 block) pairs: block_entries of them
                self.workspace(cam, 0, opts.tile_size).grow(st["survivors"], max(st["entries"], st["block_entries"]))
            else:
                raise nat.NativeError("workspace overflow persists after regrowing")
            n_s = st["survivors"]
            payload = self._payload_bytes_per_survivor(n_s, frame, return_survivors)
            stats = _frame_stats(st, evs.timings(), payload, opts.record_contributions)
            extra = (dbg.host(st),) if debug else ()
            if not to_host:
                return (frame, stats) + extra
            out = RenderOutput(
                image=_PINNED.numpy(host["image"]),
                final_transmittance=_PINNED.numpy(host["trans"]),
                contribution_max=frame.contrib_max[:n_s].cpu().numpy() if opts.record_contributions else None,
                contribution_sum=frame.contrib_sum.cpu().numpy() if opts.record_contributions else None,
                used_count=st["used"] if opts.record_contributions else None,
                passed_count=st["passed"], skipped_count=st["skipped"])
            if return_survivors:
                out.survivors = frame.survivors[:n_s].cpu().numpy().astype(np.int64)
            return (out, stats) + extra

    def render_path(self, cams, opts: RenderOptions | None = None, frames_in_flight: int = 2,
                    to_host: bool = True):
        """Render a camera path; yields (RenderOutput, FrameStats) per camera, in order.

        Frame i is rendered on stream i % F with workspace slot i % F (F =
        ``frames_in_flight``), so the kernels of consecutive frames overlap on
        the GPU and the device->host copies of frame i run while frame i + 1
        renders.  Each frame is bit-identical to ``render(cam, opts)``.
        ``to_host=False`` yields (DeviceFrame, FrameStats); the device frames
        rotate through F + 1 output buffers, so a DeviceFrame stays valid until
        the caller requests the frame after next (two consecutive frames can be
        held at once; work the caller enqueues on its current stream before
        that request is ordered before the buffer's reuse).
        """
        import torch

        from .raster import RenderOutput

        opts = opts or RenderOptions()
        F = max(1, int(frames_in_flight))
        R = F + 1   # output frames in the ring
        cams = list(cams)
        dev = self.dscene.device
        with torch.cuda.device(dev):
            main = torch.cuda.current_stream()
            # streams, per-slot events and the output ring persist across calls: a new stream's
            # first allocations would be fresh cudaMallocs (device-synchronising) inside the path
            while len(self._path_streams) < F:
                self._path_streams.append(torch.cuda.Stream(device=dev))
        streams = self._path_streams[:F]
        events = [self.stage_events(j) for j in range(F)]
        frames: list[DeviceFrame | None] = [self._path_frames.get(j) for j in range(R)]
        pending: list[dict | None] = [None] * F

        def launch(i):
            slot, ring = i % F, i % R
            st = streams[slot]
            with torch.cuda.device(dev):
                st.wait_stream(main)
                with torch.cuda.stream(st):
                    frames[ring] = self.render_device(cams[i], opts, out=frames[ring], slot=slot,
                                                      stage_events=events[slot])
                    f = frames[ring]
                    self._path_frames[ring] = f
                    host = {"stats": _to_pinned(f.stats_raw)}
                    if to_host:
                        host["image"] = _to_pinned(f.image)
                        host["trans"] = _to_pinned(f.trans)
                        if opts.record_contributions:
                            host["contrib_sum"] = _to_pinned(f.contrib_sum)
                            host["contrib_max"] = _to_pinned(f.contrib_max)
                    done = torch.cuda.Event()
                    done.record()
            pending[slot] = {"i": i, "host": host, "done": done}

        def collect(i, attempt=0):
            slot, ring = i % F, i % R
            p = pending[slot]
            t_sync = time.perf_counter()
            p["done"].synchronize()
            self.path_wait_s += time.perf_counter() - t_sync
            st = nat.stats_dict(p["host"]["stats"].numpy())
            _PINNED.give(p["host"]["stats"])
            if st["overflow"]:
                if attempt >= 3:
                    raise nat.NativeError("workspace overflow persists after regrowing")
                # regrow this slot's workspace and re-render the frame on its stream
                torch.cuda.synchronize(dev)
                self.workspace(cams[i], slot, opts.tile_size).grow(st["survivors"],
                                                                   max(st["entries"], st["block_entries"]))
                launch(i)
                return collect(i, attempt + 1)
            n_s = st["survivors"]
            stats = _frame_stats(st, events[slot].timings(),
                                 self._payload_bytes_per_survivor(n_s, frames[ring], False), opts.record_contributions)
            if not to_host:
                return frames[ring], stats
            h = p["host"]
            rec = opts.record_contributions
            cmax = None
            if rec:
                cmax = h["contrib_max"].numpy()[:n_s].copy()
                _PINNED.give(h["contrib_max"])
            out = RenderOutput(image=_PINNED.numpy(h["image"]), final_transmittance=_PINNED.numpy(h["trans"]),
                               contribution_max=cmax,
                               contribution_sum=_PINNED.numpy(h["contrib_sum"]) if rec else None,
                               used_count=st["used"] if rec else None,
                               passed_count=st["passed"], skipped_count=st["skipped"])
            return out, stats

        for i in range(min(F, len(cams))):
            launch(i)
        for i in range(len(cams)):
            res = collect(i)
            if i + F < len(cams):
                if not to_host:
                    yield res          # the caller reads the device frame before its slot is reused
                    launch(i + F)
                    continue
                launch(i + F)
            yield res
        with torch.cuda.device(dev):
            for st in streams:
                main.wait_stream(st)

    def _payload_bytes_per_survivor(self, n_s, frame, have_surv):
        # instantiated x per-gaussian Asset payload (56 B at SH degree 0)
        pb = self.dscene.payload_bytes
        if len(set(pb)) == 1:
            return int(n_s) * pb[0]
        if have_surv and frame.survivors is not None:
            inst = frame.survivors[:n_s, 0].cpu().numpy()
            per = np.array(pb)[self.dscene.inst_asset[inst]]
            return int(per.sum())
        return int(n_s) * int(np.mean(pb))


def render_composed(scene: ComposedScene, cam, opts: RenderOptions | None = None, *,
                    return_survivors: bool = False, **kw):
    """-> (RenderOutput, FrameStats).  The device scene is cached on ``scene``.

    Keyword options (``record_contributions=...``, ``frustum=...`` ...) build a
    RenderOptions when ``opts`` is not given.  ``return_survivors`` adds
    ``out.survivors`` (S, 2) [flat instance index, gaussian index].
    """
    r = scene._device
    if r is None or r.dscene.scene_version != scene._version:
        r = Renderer(scene)
        scene._device = r
    if kw:
        if opts is not None:
            raise ValueError("pass either opts or keyword options, not both")
        opts = RenderOptions(**kw)
    return r.render(cam, opts, return_survivors=return_survivors)


def render_path(scene: ComposedScene, cams, opts: RenderOptions | None = None, *, frames_in_flight: int = 2,
                **kw):
    """Render a camera path -> iterator of (RenderOutput, FrameStats), frames overlapped on the GPU.

    Same per-frame results as ``render_composed`` (bit-identical images);
    ``frames_in_flight`` frames are in flight on separate streams, so one
    frame's device->host copy and its kernels' tails overlap the next frame.
    """
    r = scene._device
    if r is None or r.dscene.scene_version != scene._version:
        r = Renderer(scene)
        scene._device = r
    if kw:
        if opts is not None:
            raise ValueError("pass either opts or keyword options, not both")
        opts = RenderOptions(**kw)
    return r.render_path(cams, opts, frames_in_flight=frames_in_flight)


def local_inputs(g_index: int, asset: Asset, inst: InstanceTransform, cam, model: VisibilityModel,
                 features: np.ndarray | None = None) -> np.ndarray:
    """The 16 visibility-MLP inputs of one (gaussian, instance) pair, host f64.

    [mean / r (3), local direction camera->gaussian (3), normalised corrected
    distance (1), local camera forward (3), feature (6)].  Inspection helper;
    the device builds the same vector inside the fused cull kernel.
    """
    R, _q, s, _ln = instance_frame(inst)
    Rm = np.array(R).reshape(3, 3)
    m = asset.means[g_index].astype(np.float64)
    mw = np.array([np.float32(s * (Rm[k, 0] * m[0] + Rm[k, 1] * m[1] + Rm[k, 2] * m[2]) + inst.translation[k])
                   for k in range(3)], dtype=np.float64)
    d = mw - cam.position
    d_r = math.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
    corr = (model.f_train / cam.focal) / s
    d_t = d_r * corr
    x = np.empty(16)
    x[0:3] = m / model.mean_scale
    x[3:6] = Rm.T @ d / d_r
    x[6] = min(1.0, max(-1.0, 2.0 * (d_t - model.d_near) / (model.d_far - model.d_near) - 1.0))
    x[7:10] = Rm.T @ cam.rotation[2]
    if features is None:
        features = model.feature_mlp.forward_host(feature_inputs(asset, model.mean_scale)[g_index:g_index + 1])[0]
    x[10:16] = np.asarray(features, dtype=np.float64)[:6]
    return x
