"""Pinhole camera (reference sc/raster.py:40-108).

Camera space is x-right, y-down, z-forward; ``rotation`` rows are
[right, down, forward] (world-to-camera).  Pixel centres sit on integer
coordinates with the principal point at ((W-1)/2, (H-1)/2).  ``far`` is kept
for API compatibility; the reference never uses it.

For the device the camera is flattened into the POD ``sc_camera`` of
``include/splatcull_b200.h`` by :meth:`Camera.pod_fields`; focal and the half
FoV tangents are computed here, on the host, with the same libm expressions
the reference uses, so device and oracle see bit-identical scalars.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(eq=False)
class Camera:
    position: np.ndarray
    rotation: np.ndarray
    fov_y: float
    width: int
    height: int
    near: float = 0.05
    far: float = 1e6

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64).reshape(3)
        self.rotation = np.asarray(self.rotation, dtype=np.float64).reshape(3, 3)
        ortho_err = float(np.abs(self.rotation @ self.rotation.T - np.eye(3)).max())
        if ortho_err > 1e-6:
            raise ValueError(f"camera rotation is not orthonormal (max error {ortho_err:.2e})")
        if not (0.0 < self.fov_y < math.pi):
            raise ValueError(f"fov_y must be in (0, pi), got {self.fov_y}")
        if self.focal <= 0.0:
            raise ValueError("camera focal must be positive")

    @property
    def focal(self) -> float:
        return self.height / (2.0 * math.tan(self.fov_y / 2.0))

    @property
    def forward(self) -> np.ndarray:
        return self.rotation[2].copy()

    @property
    def tan_half_fov(self) -> tuple[float, float]:
        t_y = math.tan(self.fov_y / 2.0)
        return t_y * self.width / self.height, t_y

    @classmethod
    def look_at(cls, position, target, fov_y, width, height, up=None, near=0.05,
                far=1e6) -> "Camera":
        eye = np.asarray(position, dtype=np.float64)
        fwd = np.asarray(target, dtype=np.float64) - eye
        length = np.linalg.norm(fwd)
        if length == 0.0:
            raise ValueError("camera position and target coincide")
        fwd = fwd / length
        if up is None:
            up = np.array([0.0, 0.0, 1.0])
            if abs(fwd @ up) > 0.999:
                up = np.array([1.0, 0.0, 0.0])
        right = np.cross(fwd, np.asarray(up, dtype=np.float64))
        right = right / np.linalg.norm(right)
        down = np.cross(fwd, right)
        return cls(position=eye, rotation=np.stack([right, down, fwd]), fov_y=float(fov_y),
                   width=int(width), height=int(height), near=near, far=far)


def diag_to_fov_y(fov_diag: float, width: int, height: int) -> float:
    """Vertical FoV of a camera whose full diagonal FoV is ``fov_diag``."""
    return 2.0 * math.atan(math.tan(fov_diag / 2.0) * height / math.hypot(width, height))


def fov_y_to_diag(fov_y: float, width: int, height: int) -> float:
    return 2.0 * math.atan(math.tan(fov_y / 2.0) * math.hypot(width, height) / height)


def train_focal(image_size: int = 256, fov_diag: float = math.radians(60.0)) -> float:
    """Focal of the visibility-extraction cameras, f_t of Eq. 2.

    Same value as the reference ``SamplingConfig().train_focal``
    (sc/sampling.py:57-63): square ``image_size`` images with a 60 degree
    diagonal FoV.
    """
    fy = diag_to_fov_y(fov_diag, image_size, image_size)
    return image_size / (2.0 * math.tan(fy / 2.0))
