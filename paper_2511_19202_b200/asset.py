"""Gaussian assets — the host-side data model the renderer consumes.

Mirrors the reference ``splatcull.asset`` surface (reference
sc/asset.py:44-171, :324-386) so that code written against the reference keeps
working: a struct-of-arrays :class:`Asset` in float32, the stable float64
``sigmoid``, ``prune`` -> ``recenter`` -> ``compute_sampling_distances`` via
``prepare``, and ``asset_hash``.  Uploading to HBM happens in
:mod:`paper_2511_19202_b200.scene`; nothing here touches the GPU.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field, replace

import numpy as np

SH_C0 = 0.28209479177387814          # degree-0 real SH basis constant
DEFAULT_PRUNE_THRESHOLD = 1.0 / 255.0


def sigmoid(x):
    """float64 logistic, split on sign to avoid overflow (sc/asset.py:44-51)."""
    v = np.asarray(x, dtype=np.float64)
    res = np.empty_like(v)
    neg = v < 0
    e = np.exp(v[neg])
    res[neg] = e / (1.0 + e)
    res[~neg] = 1.0 / (1.0 + np.exp(-v[~neg]))
    return res


def logit(p):
    p = np.asarray(p, dtype=np.float64)
    return np.log(p) - np.log1p(-p)


@dataclass
class Gaussian:
    """One splat primitive (sc/asset.py:59-71)."""

    mean: np.ndarray
    log_scale: np.ndarray
    rotation: np.ndarray        # (w, x, y, z)
    opacity_logit: float
    sh_coeffs: np.ndarray       # ((deg+1)^2, 3)

    @property
    def opacity(self) -> float:
        return float(sigmoid(self.opacity_logit))


@dataclass
class Asset:
    """Struct-of-arrays splat collection (sc/asset.py:74-140).

    Arrays are float32; ``d_near``/``d_far`` are the Eq. 1 camera distance
    bounds that gate the visibility MLP.
    """

    means: np.ndarray            # (n, 3) f32
    log_scales: np.ndarray       # (n, 3) f32
    rotations: np.ndarray        # (n, 4) f32 unit (w, x, y, z)
    opacity_logits: np.ndarray   # (n,) f32
    sh_coeffs: np.ndarray        # (n, (deg+1)^2, 3) f32
    sh_degree: int
    center_offset: np.ndarray = field(default_factory=lambda: np.zeros(3, dtype=np.float64))
    d_near: float | None = None
    d_far: float | None = None

    def __len__(self) -> int:
        return int(self.means.shape[0])

    def _require_nonempty(self):
        if len(self) == 0:
            raise ValueError("empty asset has no bounding box")

    @property
    def bbox_min(self) -> np.ndarray:
        self._require_nonempty()
        return self.means.min(axis=0).astype(np.float64)

    @property
    def bbox_max(self) -> np.ndarray:
        self._require_nonempty()
        return self.means.max(axis=0).astype(np.float64)

    @property
    def bound_radius(self) -> float:
        """Half the bbox diagonal of the means (symbol r of Eq. 1)."""
        return float(np.linalg.norm(self.bbox_max - self.bbox_min) / 2.0)

    @property
    def opacities(self) -> np.ndarray:
        return sigmoid(self.opacity_logits)

    def gaussian(self, i: int) -> Gaussian:
        return Gaussian(self.means[i].copy(), self.log_scales[i].copy(), self.rotations[i].copy(),
                        float(self.opacity_logits[i]), self.sh_coeffs[i].copy())

    @classmethod
    def from_gaussians(cls, gaussians: list[Gaussian]) -> "Asset":
        if not gaussians:
            raise ValueError("cannot build an asset from zero gaussians")
        k = int(np.asarray(gaussians[0].sh_coeffs).shape[0])
        deg = int(round(math.sqrt(k))) - 1
        if (deg + 1) ** 2 != k:
            raise ValueError(f"sh_coeffs length {k} is not a perfect square")

        def col(name):
            return np.array([getattr(g, name) for g in gaussians], dtype=np.float32)

        return cls(col("mean"), col("log_scale"), col("rotation"), col("opacity_logit"),
                   col("sh_coeffs"), deg)


def validate_asset(asset: Asset) -> None:
    """Raise ValueError when an invariant is broken (sc/asset.py:143-161)."""
    n = len(asset)
    expect = {"means": (n, 3), "log_scales": (n, 3), "rotations": (n, 4),
              "opacity_logits": (n,), "sh_coeffs": (n, (asset.sh_degree + 1) ** 2, 3)}
    for name, shape in expect.items():
        arr = getattr(asset, name)
        if arr.shape != shape:
            raise ValueError(f"{name} has shape {arr.shape}, expected {shape}")
        if not np.isfinite(arr).all():
            raise ValueError(f"non-finite value in {name}")
    if n:
        qn = np.linalg.norm(asset.rotations.astype(np.float64), axis=1)
        if np.abs(qn - 1.0).max() > 1e-6:
            raise ValueError("rotation quaternions are not unit length")


def asset_hash(asset: Asset) -> int:
    """64-bit digest pairing models with assets (sc/asset.py:164-171)."""
    h = hashlib.sha256(np.int64(asset.sh_degree).tobytes())
    for arr in (asset.means, asset.log_scales, asset.rotations, asset.opacity_logits,
                asset.sh_coeffs):
        h.update(np.ascontiguousarray(arr, dtype=np.float32).tobytes())
    return int.from_bytes(h.digest()[:8], "little")


def prune(asset: Asset, threshold: float = DEFAULT_PRUNE_THRESHOLD) -> Asset:
    """Keep Gaussians with sigmoid(logit) >= threshold, order preserved."""
    if not (0.0 <= threshold < 1.0):
        raise ValueError(f"prune threshold must be in [0, 1), got {threshold}")
    keep = asset.opacities >= threshold
    return replace(asset, means=asset.means[keep], log_scales=asset.log_scales[keep],
                   rotations=asset.rotations[keep], opacity_logits=asset.opacity_logits[keep],
                   sh_coeffs=asset.sh_coeffs[keep], d_near=None, d_far=None)


def recenter(asset: Asset) -> Asset:
    """Move the bbox centre of the means to the origin; remember the shift."""
    if len(asset) == 0:
        raise ValueError("cannot recenter an empty asset")
    centre = (asset.bbox_min + asset.bbox_max) / 2.0
    shifted = (asset.means.astype(np.float64) - centre).astype(np.float32)
    return replace(asset, means=shifted,
                   center_offset=np.asarray(asset.center_offset, dtype=np.float64) + centre)


def compute_sampling_distances(asset: Asset, fov: float, p_near: float = 0.9,
                               p_far: float = 0.05) -> tuple[float, float]:
    """Eq. 1: d = r / (tan(fov/2) p) at p_near and p_far (fov = diagonal FoV)."""
    if not (0.0 < fov < math.pi):
        raise ValueError(f"fov must be in (0, pi), got {fov}")
    if not (0.0 < p_far < p_near <= 1.0):
        raise ValueError(f"need 0 < p_far < p_near <= 1, got p_near={p_near} p_far={p_far}")
    r = asset.bound_radius
    if r <= 0.0:
        raise ValueError("degenerate asset: bound radius is zero")
    half = math.tan(fov / 2.0)
    return r / (half * p_near), r / (half * p_far)


def prepare(asset: Asset, prune_threshold: float = DEFAULT_PRUNE_THRESHOLD,
            fov: float = math.radians(60.0), p_near: float = 0.9, p_far: float = 0.05) -> Asset:
    """prune -> recenter -> sampling distances (sc/asset.py:376-386)."""
    a = recenter(prune(asset, prune_threshold))
    d_near, d_far = compute_sampling_distances(a, fov, p_near, p_far)
    return replace(a, d_near=d_near, d_far=d_far)
