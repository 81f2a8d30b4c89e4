"""Visibility model: feature MLP 14->32->32->6 and visibility MLP 16->32->32->1.

The reference package does not ship its ``nn`` module; this follows
SPEC.md:240-323 (architecture, He-uniform init, 16-input layout, threshold)
and PAPER.md:171-179 (16 inputs so the MLP maps onto tensor cores).  Weights
live on the host as float32 (the SPEC checkpoint dtype); the device copies
them to fp16 in shared memory (``sc_vis_mlp_forward`` / the fused cull
kernel).  Training lives in train.py; checkpoints are
``save_model`` / ``load_model`` below.

Pinned decisions: hidden activations ReLU, feature
output linear, visibility output a logit, keep iff logit >= logit(threshold).
"""

from __future__ import annotations

import json
import math
import struct
from dataclasses import dataclass, field

import numpy as np

from .asset import SH_C0, Asset, asset_hash, sigmoid

VIS_WIDTHS = (16, 32, 32, 1)
FEATURE_WIDTHS = (14, 32, 32, 6)


@dataclass
class Mlp:
    """Dense ReLU chain; ``weights[l]`` is (out, in) row-major float32."""

    weights: list[np.ndarray]
    biases: list[np.ndarray]

    @property
    def widths(self) -> tuple[int, ...]:
        return (int(self.weights[0].shape[1]),) + tuple(int(w.shape[0]) for w in self.weights)

    @property
    def n_params(self) -> int:
        return int(sum(w.size + b.size for w, b in zip(self.weights, self.biases)))

    def forward_host(self, x: np.ndarray) -> np.ndarray:
        """float64 host evaluation (tests / small batches only)."""
        h = np.asarray(x, dtype=np.float64)
        last = len(self.weights) - 1
        for li, (w, b) in enumerate(zip(self.weights, self.biases)):
            h = h @ w.astype(np.float64).T + b.astype(np.float64)
            if li < last:
                h = np.maximum(h, 0.0)
        return h


def init_mlp(widths, seed: int = 0) -> Mlp:
    """Seeded He-uniform weights (bound sqrt(6 / fan_in)), zero biases."""
    if len(widths) < 2 or min(widths) < 1:
        raise ValueError(f"invalid MLP widths {widths}")
    rng = np.random.default_rng(seed)
    ws, bs = [], []
    for fan_in, fan_out in zip(widths[:-1], widths[1:]):
        bound = math.sqrt(6.0 / fan_in)
        ws.append(rng.uniform(-bound, bound, size=(fan_out, fan_in)).astype(np.float32))
        bs.append(np.zeros(fan_out, dtype=np.float32))
    return Mlp(ws, bs)


@dataclass
class VisibilityModel:
    """Per-asset model plus the normalisation constants of Eq. 2."""

    feature_mlp: Mlp
    vis_mlp: Mlp
    mean_scale: float          # bound_radius of the training asset
    d_near: float
    d_far: float
    f_train: float             # training-camera focal (pixels), f_t of Eq. 2
    threshold: float = 0.5
    asset_hash: int | None = None
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.vis_mlp.widths[0] != 16 or self.vis_mlp.widths[-1] != 1:
            raise ValueError(f"visibility MLP must be 16 -> ... -> 1, got {self.vis_mlp.widths}")
        if self.feature_mlp.widths[-1] != 6:
            raise ValueError(f"feature MLP must output 6 values, got {self.feature_mlp.widths}")
        if not (0.0 < self.threshold < 1.0):
            raise ValueError("threshold must be in (0, 1)")
        if not (0.0 < self.d_near < self.d_far):
            raise ValueError("need 0 < d_near < d_far")

    @property
    def logit_threshold(self) -> float:
        return math.log(self.threshold) - math.log1p(-self.threshold)


def make_model(asset: Asset, seed: int = 0, f_train: float | None = None,
               output_bias: float = 0.0, threshold: float = 0.5) -> VisibilityModel:
    """Random-init model for ``asset`` (the benchmarks have no trained weights).

    ``output_bias`` shifts the visibility logit; the benchmark sets it so the
    keep-rate approximates the paper's 60-70 % and records it.
    """
    from .camera import train_focal

    if asset.d_near is None or asset.d_far is None:
        raise ValueError("asset has no d_near/d_far; call prepare() first")
    feat = init_mlp(FEATURE_WIDTHS, seed=seed * 2 + 1)
    vis = init_mlp(VIS_WIDTHS, seed=seed * 2)
    vis.biases[-1] = np.full(1, output_bias, dtype=np.float32)
    return VisibilityModel(feat, vis, asset.bound_radius, float(asset.d_near), float(asset.d_far),
                           float(train_focal() if f_train is None else f_train),
                           threshold=threshold, asset_hash=asset_hash(asset))


def feature_inputs(asset: Asset, mean_scale: float) -> np.ndarray:
    """(n, 14) float32 feature-MLP inputs.

    [mean / r (3), exp(log_scale) / r (3), quaternion (4), sigmoid(opacity) (1),
    DC colour SH_C0 * f_dc + 0.5 (3)].
    """
    n = len(asset)
    x = np.empty((n, 14), dtype=np.float64)
    x[:, 0:3] = asset.means.astype(np.float64) / mean_scale
    x[:, 3:6] = np.exp(asset.log_scales.astype(np.float64)) / mean_scale
    x[:, 6:10] = asset.rotations.astype(np.float64)
    x[:, 10] = sigmoid(asset.opacity_logits)
    x[:, 11:14] = SH_C0 * asset.sh_coeffs[:, 0, :].astype(np.float64) + 0.5
    return x.astype(np.float32)


def forward(model: VisibilityModel, inputs) -> np.ndarray:
    """Batched visibility MLP on the GPU: (B, 16) -> (B, 1) logits.

    Inputs are materialised fp32 rows; the kernel converts them to fp16 and
    runs the 16->32->32 layers on tcgen05 tensor cores (torch.ops.splatcull.vis_mlp_forward).
    Accepts a numpy array or a CUDA torch tensor (then returns a tensor).
    """
    import torch

    from . import _native as nat
    from . import ops
    from .scene import vis_weights_struct

    nat.load()
    is_tensor = isinstance(inputs, torch.Tensor)
    x = inputs if is_tensor else torch.from_numpy(np.ascontiguousarray(inputs, dtype=np.float32))
    if x.ndim != 2 or x.shape[1] != 16:
        raise ValueError(f"visibility MLP expects (B, 16) inputs, got {tuple(x.shape)}")
    x = x.to("cuda" if not x.is_cuda else x.device, torch.float32).contiguous()
    w = nat.struct_tensor(vis_weights_struct(model), x.device)
    with torch.cuda.device(x.device):
        out = ops.vis_mlp_forward(w, x).view(-1, 1)
    return out if is_tensor else out.cpu().numpy()


def encode_features(model: VisibilityModel, asset: Asset) -> np.ndarray:
    """Per-gaussian 6-vectors from the feature MLP, on the GPU."""
    if model.asset_hash is not None and asset_hash(asset) != model.asset_hash:
        raise ValueError("asset hash does not match the model")
    from .scene import encode_features_device

    return encode_features_device(model, asset, "cuda")[:, :6].float().cpu().numpy()


# Checkpoint: header, layer widths, float32 weights/biases (row-major (out, in)),
# then the JSON meta.  SPEC.md nn.save_model: magic + version + normalisation
# constants + layer dims + f32 weights, under 32 kB for the paper's sizes.
MODEL_MAGIC = b"SCVM"
MODEL_VERSION = 1
_MODEL_HEADER = "<4sIQ?5dII"   # magic, version, asset hash, has hash, r, d_near, d_far, f_train, threshold, #feat, #vis


def save_model(model: VisibilityModel, path) -> None:
    fw, vw = model.feature_mlp.widths, model.vis_mlp.widths
    meta = json.dumps(model.meta, sort_keys=True, default=float).encode()
    with open(path, "wb") as fh:
        fh.write(struct.pack(_MODEL_HEADER, MODEL_MAGIC, MODEL_VERSION, model.asset_hash or 0,
                             model.asset_hash is not None, model.mean_scale, model.d_near, model.d_far,
                             model.f_train, model.threshold, len(fw), len(vw)))
        fh.write(struct.pack(f"<{len(fw) + len(vw)}I", *fw, *vw))
        for mlp in (model.feature_mlp, model.vis_mlp):
            for w, b in zip(mlp.weights, mlp.biases):
                fh.write(np.ascontiguousarray(w, dtype="<f4").tobytes())
                fh.write(np.ascontiguousarray(b, dtype="<f4").tobytes())
        fh.write(struct.pack("<I", len(meta)))
        fh.write(meta)


def load_model(path) -> VisibilityModel:
    with open(path, "rb") as fh:
        raw = fh.read()
    hsize = struct.calcsize(_MODEL_HEADER)
    if len(raw) < hsize:
        raise ValueError(f"{path}: truncated model header")
    magic, version, ahash, has_hash, r, dn, df, ft, thr, nf, nv = struct.unpack_from(_MODEL_HEADER, raw)
    if magic != MODEL_MAGIC:
        raise ValueError(f"{path}: bad magic {magic!r}")
    if version != MODEL_VERSION:
        raise ValueError(f"{path}: unsupported model version {version}")
    if not (2 <= nf <= 16 and 2 <= nv <= 16):
        raise ValueError(f"{path}: implausible layer counts {nf}, {nv}")
    off = hsize
    need = 4 * (nf + nv)
    if len(raw) < off + need:
        raise ValueError(f"{path}: truncated layer widths")
    widths = struct.unpack_from(f"<{nf + nv}I", raw, off)
    off += need

    def read_mlp(ws):
        nonlocal off
        weights, biases = [], []
        for fan_in, fan_out in zip(ws[:-1], ws[1:]):
            for shape in ((fan_out, fan_in), (fan_out,)):
                cnt = int(np.prod(shape))
                if len(raw) < off + 4 * cnt:
                    raise ValueError(f"{path}: truncated weights")
                arr = np.frombuffer(raw, dtype="<f4", count=cnt, offset=off).reshape(shape).astype(np.float32)
                (weights if len(shape) == 2 else biases).append(arr)
                off += 4 * cnt
        return Mlp(weights, biases)

    feat, vis = read_mlp(widths[:nf]), read_mlp(widths[nf:])
    if len(raw) < off + 4:
        raise ValueError(f"{path}: truncated meta")
    (mlen,) = struct.unpack_from("<I", raw, off)
    off += 4
    if len(raw) < off + mlen:
        raise ValueError(f"{path}: truncated meta")
    meta = json.loads(raw[off:off + mlen].decode()) if mlen else {}
    for mlp in (feat, vis):
        if not all(np.isfinite(a).all() for a in mlp.weights + mlp.biases):
            raise ValueError(f"{path}: non-finite weights")
    return VisibilityModel(feat, vis, r, dn, df, ft, threshold=thr, asset_hash=int(ahash) if has_hash else None,
                           meta=meta)
