"""Shared pytest configuration.

Markers: ``gpu`` tests need a B200 (they call libsplatcull_b200.so through its
C ABI and compare against the CPU oracle); everything else runs on CPU.
The oracle (oracle/) is imported here only as the checker.
"""

import math
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
GOLDEN_CASES = ["cloud3k_128", "shell4k_160x96", "slab_headon_96", "cloud_clip_112x80", "shell_sh3_144x112",
                "cloud_sh2_eval1_120x90", "cloud_bg_dil_100x70", "cloud_ts8_120x88", "shell_ts32_150x100",
                "cloud_ts12_100x76", "cloud_dil15_border_96x72"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: longer-running CPU test")


def load_golden(name):
    from paper_2511_19202_b200.asset import Asset
    from paper_2511_19202_b200.camera import Camera

    z = np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)
    asset = Asset(means=z["means"], log_scales=z["log_scales"], rotations=z["rotations"],
                  opacity_logits=z["opacity_logits"], sh_coeffs=z["sh_coeffs"], sh_degree=int(z["sh_degree"]))
    cam = Camera(position=z["cam_position"], rotation=z["cam_rotation"], fov_y=float(z["cam_fov_y"]),
                 width=int(z["cam_width"]), height=int(z["cam_height"]), near=float(z["cam_near"]))
    opts = eval(str(z["opts"]), {"__builtins__": {}})  # a literal dict written by gen_golden.py
    return asset, cam, opts, z


@pytest.fixture(params=GOLDEN_CASES)
def golden(request):
    return (request.param,) + load_golden(request.param)


def look_at(pos, target, fov_deg, w, h, up=None):
    from paper_2511_19202_b200.camera import Camera
    return Camera.look_at(pos, target, math.radians(fov_deg), w, h, up=up)
