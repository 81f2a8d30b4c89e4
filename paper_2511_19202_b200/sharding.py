"""Multi-GPU work sharding of the render path: camera-path frames
or screen bands, one process per GPU, scene replicated on every GPU.

* Frames: frame k of a camera path is rendered by rank k mod G; no exchange.
* Bands: rank r renders tile rows [t_r, t_{r+1}) of every frame (the cull uses
  the band's sub-frustum, a conservative superset, so the band's pixels equal
  the whole-image render bit for bit); the bands are balanced by the previous
  frame's per-band cost and gathered into rank 0's frame by peer-to-peer
  copies over NVLink (CUDA IPC), with no NCCL collective on the render path.
  ``torch.distributed`` carries only control messages (IPC handles, band
  bounds, timings) -- gloo on CPU in the tests.
"""

from __future__ import annotations

import math

import numpy as np

TILE = 16


def frames_for_rank(n_frames: int, rank: int, world: int) -> list[int]:
    """Frames of a camera path rendered by ``rank`` (round robin)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return list(range(rank, n_frames, world))


def split_rows(n_rows: int, world: int, weights=None) -> list[int]:
    """Tile-row boundaries [0 = b_0 < b_1 < ... < b_world = n_rows] splitting the
    cumulative per-row weight evenly (equal rows when ``weights`` is None).
    Every band gets at least one row."""
    if world < 1 or n_rows < world:
        raise ValueError(f"cannot split {n_rows} tile rows into {world} bands")
    w = np.ones(n_rows) if weights is None else np.maximum(np.asarray(weights, np.float64), 1e-12)
    if w.shape != (n_rows,):
        raise ValueError("weights must have one entry per tile row")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    bounds = [0]
    for r in range(1, world):
        target = cum[-1] * r / world
        b = int(np.searchsorted(cum, target, side="left"))
        b = min(max(b, bounds[-1] + 1), n_rows - (world - r))
        bounds.append(b)
    bounds.append(n_rows)
    return bounds


def rebalance(bounds: list[int], band_ms: list[float]) -> list[int]:
    """New boundaries from the previous frame's per-band times: each band's cost
    is spread uniformly over its rows, then the rows are re-split evenly."""
    world = len(bounds) - 1
    if len(band_ms) != world:
        raise ValueError("one time per band")
    n_rows = bounds[-1]
    w = np.empty(n_rows)
    for r in range(world):
        rows = bounds[r + 1] - bounds[r]
        w[bounds[r]:bounds[r + 1]] = max(float(band_ms[r]), 1e-6) / rows
    return split_rows(n_rows, world, w)


def band_pixels(bounds: list[int], rank: int, height: int) -> tuple[int, int]:
    """Pixel rows [y0, y1) of ``rank``'s band."""
    return bounds[rank] * TILE, min(bounds[rank + 1] * TILE, height)


def tile_rows(height: int) -> int:
    return int(math.ceil(height / TILE))


class BandGather:
    """Assembles the bands of a frame in rank 0's image.

    On GPUs (``transport="p2p"``): rank 0 shares its full-frame image tensor by
    CUDA IPC once; every other rank writes its band rows straight into it with
    a device-to-device copy over NVLink, then signals completion with a
    control-plane barrier.  On CPU (``transport="gloo"``, tests): the band rows
    are sent to rank 0 with point-to-point messages.
    """

    def __init__(self, full_shape, rank: int, world: int, device=None, transport: str = "p2p", group=None):
        import torch
        import torch.distributed as dist

        self.rank, self.world, self.transport, self.group = rank, world, transport, group
        self.shape = tuple(full_shape)
        self.full = None
        if transport == "p2p":
            if rank == 0:
                self.full = torch.empty(self.shape, dtype=torch.float32, device=device)
                handle = [self.full.untyped_storage()._share_cuda_()]
            else:
                handle = [None]
            dist.broadcast_object_list(handle, src=0, group=group)
            if rank != 0:
                storage = torch.UntypedStorage._new_shared_cuda(*handle[0])
                self.full = torch.empty(0, dtype=torch.float32, device=device).set_(
                    storage, 0, self.shape, self._strides(self.shape))
        elif transport == "gloo":
            if rank == 0:
                self.full = torch.empty(self.shape, dtype=torch.float32)
        else:
            raise ValueError(f"unknown transport {transport}")

    @staticmethod
    def _strides(shape):
        st, acc = [], 1
        for d in reversed(shape):
            st.append(acc)
            acc *= d
        return tuple(reversed(st))

    def gather(self, band_image, bounds: list[int]):
        """``band_image``: this rank's rendered frame (full size, band rows valid).
        Returns the assembled frame on rank 0 (None elsewhere)."""
        import torch
        import torch.distributed as dist

        h = self.shape[0]
        y0, y1 = band_pixels(bounds, self.rank, h)
        if self.transport == "p2p":
            self.full[y0:y1].copy_(band_image[y0:y1], non_blocking=True)
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.group)
            return self.full if self.rank == 0 else None
        if self.rank == 0:
            self.full[y0:y1] = band_image[y0:y1]
            for r in range(1, self.world):
                ry0, ry1 = band_pixels(bounds, r, h)
                buf = torch.empty((ry1 - ry0,) + self.shape[1:], dtype=torch.float32)
                dist.recv(buf, src=r, group=self.group)
                self.full[ry0:ry1] = buf
            return self.full
        dist.send(band_image[y0:y1].contiguous().float(), dst=0, group=self.group)
        return None
