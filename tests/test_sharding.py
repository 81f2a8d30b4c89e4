"""Multi-GPU sharding host logic on CPU: band partition and
rebalancing, frame round robin, and the band gather with world_size 2 over
gloo (the GPU path moves the same rows by CUDA IPC peer copies)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_19202_b200 import sharding as sh


def test_split_rows_covers_and_balances():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 4, 8):
        for n in (world, 17, 68, 135):
            if n < world:
                continue
            w = rng.gamma(0.5, size=n) + 1e-3
            b = sh.split_rows(n, world, w)
            assert b[0] == 0 and b[-1] == n and len(b) == world + 1
            assert all(b1 > b0 for b0, b1 in zip(b, b[1:]))
            cost = [w[b[r]:b[r + 1]].sum() for r in range(world)]
            # a greedy prefix split is off the even share by at most one row's weight
            assert max(cost) <= w.sum() / world + w.max() + 1e-9
    with pytest.raises(ValueError):
        sh.split_rows(3, 4)


def test_rebalance_converges_on_a_skewed_frame():
    rng = np.random.default_rng(1)
    row_cost = np.concatenate([np.full(20, 0.1), rng.uniform(2.0, 6.0, 28), np.full(20, 0.2)])   # dense middle
    world = 4
    b = sh.split_rows(len(row_cost), world)
    spread0 = None
    for _ in range(6):
        t = [row_cost[b[r]:b[r + 1]].sum() for r in range(world)]
        spread = max(t) / (sum(t) / world)
        spread0 = spread0 or spread
        b = sh.rebalance(b, t)
    t = [row_cost[b[r]:b[r + 1]].sum() for r in range(world)]
    assert max(t) / (sum(t) / world) < 0.5 * spread0 + 0.5
    assert max(t) / (sum(t) / world) < 1.35


def test_frames_round_robin_partition():
    for world in (1, 2, 4, 8):
        got = sorted(f for r in range(world) for f in sh.frames_for_rank(120, r, world))
        assert got == list(range(120))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _frame(h, w, k):
    yy, xx = np.mgrid[0:h, 0:w]
    img = np.stack([np.sin(0.1 * xx + k), np.cos(0.07 * yy - k), (xx * yy % 7) / 7.0], -1)
    return torch.from_numpy(img.astype(np.float32))


def _worker(rank, world, port, h, w, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        bounds = sh.split_rows(sh.tile_rows(h), world)
        g = sh.BandGather((h, w, 3), rank, world, transport="gloo")
        ok = True
        for k in range(3):
            full = _frame(h, w, k)
            mine = torch.full_like(full, float("nan"))        # only the band rows are rendered
            y0, y1 = sh.band_pixels(bounds, rank, h)
            mine[y0:y1] = full[y0:y1]
            out = g.gather(mine, bounds)
            if rank == 0:
                ok &= bool(torch.equal(out, full))
            bounds = sh.rebalance(bounds, [1.0 + r for r in range(world)])
            obj = [bounds]
            dist.broadcast_object_list(obj, src=0)
            bounds = obj[0]
        frames = torch.tensor(sh.frames_for_rank(10, rank, world) + [-1] * 10)[:10]
        allf = [torch.empty_like(frames) for _ in range(world)]
        dist.all_gather(allf, frames)
        got = sorted(int(f) for t in allf for f in t if f >= 0)
        ok &= got == list(range(10))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_band_gather_world2_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 72, 40, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
