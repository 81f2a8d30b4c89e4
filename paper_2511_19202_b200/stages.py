"""Stage-level entry points (torch.ops.splatcull cull_mlp / project / bin_sort / blend).

Each reference stage can be driven on its own with explicit inputs, so parity
tests inject the oracle's survivor set, order or tile entries at any stage
boundary.  All functions enqueue on the current torch stream of
the scene's device; they return numpy arrays for the parity checks plus the
device splat records / windows for the next stage.
"""

from __future__ import annotations

import numpy as np

from . import _native as nat
from . import ops
from .scene import DeviceScene, RenderOptions, Workspace


def _survivor_tensor(surv_inst, surv_gid, device):
    import torch

    s = np.stack([np.asarray(surv_inst, np.int64), np.asarray(surv_gid, np.int64)], axis=1).astype(np.uint32)
    return torch.from_numpy(s.view(np.int32)).to(device)


def _u32(t, n):
    return t[:n].cpu().numpy().view(np.uint32).astype(np.int64)


def cull_mlp(dscene: DeviceScene, cam, opts: RenderOptions, cap: int | None = None):
    """Stages (a)+(b): -> (survivors (S, 2) int32 [inst, gid], stats dict)."""
    import torch

    nat.load()
    cap = int(cap if cap is not None else max(1, dscene.max_pairs))
    with torch.cuda.device(dscene.device):
        ws = Workspace(dscene, cam.width, cam.height, cap_s=1, cap_e=1, tile_size=opts.tile_size)
        cam_f, cam_i = ops.pack_camera(cam)
        opt_f, opt_i = ops.pack_opts(opts.struct(cam))
        surv, stats = ops.cull_mlp(dscene.op_scene, dscene.op_meta, cam_f, cam_i, opt_f, opt_i, ws.buf, ws.op_meta,
                                   cap)
    st = nat.stats_dict(stats.cpu().numpy())
    return surv[:min(cap, st["survivors"])], st


def project(dscene: DeviceScene, surv_inst, surv_gid, cam, opts: RenderOptions):
    """Stage (c) with f64 debug outputs: dict of numpy arrays + splat records."""
    import torch

    nat.load()
    with torch.cuda.device(dscene.device):
        sv = _survivor_tensor(surv_inst, surv_gid, dscene.device)
        n = int(sv.shape[0])
        cam_f, cam_i = ops.pack_camera(cam)
        opt_f, opt_i = ops.pack_opts(opts.struct(cam))
        splats, wins, dbg, rect, flags, stats = ops.project(dscene.op_scene, dscene.op_meta, sv, cam_f, cam_i, opt_f,
                                                            opt_i)
    d = dbg[:n].cpu().numpy()
    fl = flags[:n].cpu().numpy()
    return {"mean2d": d[:, 0:2], "conic": d[:, 2:5], "depth": d[:, 5], "radius": d[:, 6], "det": d[:, 7],
            "rect": rect[:n].cpu().numpy(), "valid": (fl & 1) > 0, "passed": (fl & 2) > 0,
            "splats": splats[:n], "windows": wins[:n], "stats": nat.stats_dict(stats.cpu().numpy())}


def bin_sort(dscene: DeviceScene, surv_inst, surv_gid, cam, opts: RenderOptions, cap_entries: int | None = None):
    """Stages (c)+(d): -> dict(order_idx, entry_idx, counts, splats, stats)."""
    import torch

    nat.load()
    with torch.cuda.device(dscene.device):
        sv = _survivor_tensor(surv_inst, surv_gid, dscene.device)
        n = int(sv.shape[0])
        cap_e = int(cap_entries if cap_entries is not None else max(1 << 16, 64 * n))
        ws = Workspace(dscene, cam.width, cam.height, cap_s=max(n, 1), cap_e=cap_e, tile_size=opts.tile_size)
        cam_f, cam_i = ops.pack_camera(cam)
        opt_f, opt_i = ops.pack_opts(opts.struct(cam))
        splats, wins, entries, offs, order, stats = ops.bin_sort(dscene.op_scene, dscene.op_meta, sv, cam_f, cam_i,
                                                                 opt_f, opt_i, ws.buf, ws.op_meta)
    st = nat.stats_dict(stats.cpu().numpy())
    if st["overflow"]:
        raise nat.NativeError(f"entry capacity {cap_e} too small for {st['entries']} entries")
    return {"order_idx": _u32(order, st["passed"]), "entry_idx": _u32(entries, st["entries"]),
            "counts": _u32(offs, offs.numel()), "splats": splats[:n], "windows": wins[:n], "stats": st}


def blend(splats, windows, entry_idx, counts, cam, opts: RenderOptions, n_splats: int | None = None):
    """Stage (e) on explicit entries: -> (image, trans[, contrib_sum, contrib_max]) numpy."""
    import torch

    nat.load()
    dev = splats.device
    n = int(n_splats if n_splats is not None else splats.shape[0])
    with torch.cuda.device(dev):
        ent = torch.from_numpy(np.asarray(entry_idx, np.int64).astype(np.uint32).view(np.int32)).to(dev)
        off = torch.from_numpy(np.asarray(counts, np.int64).astype(np.uint32).view(np.int32)).to(dev)
        cam_f, cam_i = ops.pack_camera(cam)
        opt_f, opt_i = ops.pack_opts(opts.struct(cam))
        image, trans, csum, cmax = ops.blend(splats, windows, ent, off, n, cam_f, cam_i, opt_f, opt_i)
    res = {"image": image.cpu().numpy(), "trans": trans.cpu().numpy()}
    if opts.record_contributions:
        res["contrib_sum"] = csum.cpu().numpy()
        res["contrib_max"] = cmax[:n].cpu().numpy()
    return res
