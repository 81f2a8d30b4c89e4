"""Screen-band sharding through its real transport: two ranks on
one GPU (gloo control plane only), each renders its band of a config-3 frame
with the library, the band rows land in rank 0's frame by CUDA-IPC peer copies
(BandGather, transport "p2p"), and the assembled frame equals the whole-image
render bit for bit, frame after frame with the bands rebalanced in between."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        from paper_2511_19202_b200 import sharding as sh
        from paper_2511_19202_b200.scene import RenderOptions, Renderer
        from paper_2511_19202_b200.workloads import config3

        wl = config3(n_per=4_000, n_instances=120, width=480, height=270)
        r = Renderer(wl.scene)
        h, w = int(wl.cameras[0].height), int(wl.cameras[0].width)
        g = sh.BandGather((h, w, 3), rank, world, device="cuda", transport="p2p")
        bounds = sh.split_rows(sh.tile_rows(h), world)
        ok = True
        for k, cam in enumerate(wl.cameras + wl.cameras[:1]):
            y0, y1 = sh.band_pixels(bounds, rank, h)
            band, st = r.render(cam, RenderOptions(band=(y0, y1)), to_host=False)
            out = g.gather(band.image, bounds)
            if rank == 0:
                full, _ = r.render(cam, RenderOptions(), to_host=False)
                torch.cuda.synchronize()
                ok &= bool(torch.equal(out, full.image))
            t = [torch.zeros(1) for _ in range(world)]
            dist.all_gather(t, torch.tensor([float(st.render_ms)]))
            bounds = sh.rebalance(bounds, [float(x) for x in t])
        q.put((rank, ok))
    except Exception as e:   # surface the failure in the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_band_gather_cuda_ipc_two_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}, res
