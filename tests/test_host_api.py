"""Host-side API logic that needs no GPU: option validation mirroring the
reference's keywords (sc/raster.py:240-251), workspace keys, the oracle's
margin pad."""

import math

import numpy as np
import pytest


def _cam(w=320, h=240):
    from paper_2511_19202_b200.camera import Camera

    return Camera.look_at((0.0, -5.0, 1.0), (0.0, 0.0, 0.0), math.radians(50.0), w, h)


@pytest.mark.parametrize("ts", [1, 8, 12, 16, 32, 65535])
def test_tile_size_accepted(ts):
    from paper_2511_19202_b200.scene import RenderOptions

    assert RenderOptions(tile_size=ts).struct(_cam()).tile_size == ts


@pytest.mark.parametrize("ts", [0, -16, 65536, 8.5, True])
def test_tile_size_rejected(ts):
    from paper_2511_19202_b200.scene import RenderOptions

    with pytest.raises(ValueError):
        RenderOptions(tile_size=ts).struct(_cam())


def test_bands_need_tile_16():
    from paper_2511_19202_b200.scene import RenderOptions

    assert RenderOptions(band=(16, 64)).struct(_cam()).band_y1 == 64
    with pytest.raises(ValueError, match="tile_size 16"):
        RenderOptions(band=(16, 64), tile_size=8).struct(_cam())
    with pytest.raises(ValueError):
        RenderOptions(band=(8, 64)).struct(_cam())


def test_workspace_key_separates_tile_sizes_and_slots():
    from paper_2511_19202_b200.scene import Renderer

    cam = _cam()
    keys = {Renderer.ws_key(cam), Renderer.ws_key(cam, 1), Renderer.ws_key(cam, 0, 8)}
    assert len(keys) == 3


def test_margin_pad_kat():
    """pad = max(3, 3 sqrt(dilation) + 1 + 1e-6) px: 3 at the default dilation 0.3."""
    from oracle import raster_ref as rr

    L = rr.lib()
    assert L.orc_margin_pad(0.3) == 3.0
    assert L.orc_margin_pad(0.0) == 3.0
    assert L.orc_margin_pad(-1.0) == 3.0
    assert L.orc_margin_pad(1.5) == 3.0 * math.sqrt(1.5) + 1.0 + 1e-6
    assert L.orc_margin_pad(4.0) == 7.0 + 1e-6


def test_asset_fingerprint_tracks_buffers():
    import dataclasses

    from paper_2511_19202_b200 import raster, synth

    a = synth.make_random_cloud(100, seed=0)
    assert raster._asset_fingerprint(a) == raster._asset_fingerprint(a)
    b = dataclasses.replace(a, means=a.means.copy())
    assert raster._asset_fingerprint(a) != raster._asset_fingerprint(b)
    c = dataclasses.replace(a, sh_degree=a.sh_degree)
    assert raster._asset_fingerprint(a) == raster._asset_fingerprint(c)
    assert np.shares_memory(a.means, c.means)
