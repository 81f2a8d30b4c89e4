"""Stage-level entry points (sc_cull_mlp / sc_project / sc_bin_sort / sc_blend).

Each reference stage can be driven on its own with explicit inputs, so parity
tests inject the oracle's survivor set, order or tile entries at any stage
boundary.  All functions enqueue on the current torch stream and
return torch CUDA tensors.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .scene import DeviceScene, RenderOptions, Workspace


def _survivor_tensor(surv_inst, surv_gid, device):
    import torch

    s = np.stack([np.asarray(surv_inst, np.int64), np.asarray(surv_gid, np.int64)], axis=1).astype(np.uint32)
    return torch.from_numpy(s.view(np.int32)).to(device)


def cull_mlp(dscene: DeviceScene, cam, opts: RenderOptions, cap: int | None = None):
    """Stages (a)+(b): -> (survivors (S, 2) int32 [inst, gid], stats dict)."""
    import torch

    lib = nat.load()
    cap = int(cap if cap is not None else max(1, dscene.max_pairs))
    ws = Workspace(dscene, cam.width, cam.height, cap_s=1, cap_e=1, tile_size=opts.tile_size)
    surv = torch.empty((cap, 2), dtype=torch.int32, device=dscene.device)
    stats = torch.empty(nat.STATS_BYTES, dtype=torch.uint8, device=dscene.device)
    camc, optc = nat.camera_struct(cam), opts.struct(cam)
    nat.check(lib.sc_cull_mlp(ctypes.byref(dscene.struct), ctypes.byref(camc), ctypes.byref(optc),
                              ctypes.byref(ws.struct), nat.ptr(surv), cap, nat.ptr(stats), nat.stream_handle()),
              "sc_cull_mlp")
    st = nat.stats_dict(stats.cpu().numpy())
    return surv[:min(cap, st["survivors"])], st


def project(dscene: DeviceScene, surv_inst, surv_gid, cam, opts: RenderOptions):
    """Stage (c) with f64 debug outputs: dict of numpy arrays + splat records."""
    import torch

    lib = nat.load()
    dev = dscene.device
    sv = _survivor_tensor(surv_inst, surv_gid, dev)
    n = int(sv.shape[0])
    splats = torch.empty((max(n, 1), nat.SPLAT_BYTES), dtype=torch.uint8, device=dev)
    wins = torch.empty((max(n, 1), nat.WINDOW_BYTES), dtype=torch.uint8, device=dev)
    dbg = torch.empty((max(n, 1), 8), dtype=torch.float64, device=dev)
    rect = torch.empty((max(n, 1), 4), dtype=torch.int32, device=dev)
    flags = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    stats = torch.empty(nat.STATS_BYTES, dtype=torch.uint8, device=dev)
    camc, optc = nat.camera_struct(cam), opts.struct(cam)
    nat.check(lib.sc_project(ctypes.byref(dscene.struct), nat.ptr(sv), n, ctypes.byref(camc), ctypes.byref(optc),
                             nat.ptr(splats), nat.ptr(wins), nat.ptr(dbg), nat.ptr(rect), nat.ptr(flags),
                             nat.ptr(stats),
                             nat.stream_handle()), "sc_project")
    d = dbg[:n].cpu().numpy()
    return {"mean2d": d[:, 0:2], "conic": d[:, 2:5], "depth": d[:, 5], "radius": d[:, 6], "det": d[:, 7],
            "rect": rect[:n].cpu().numpy(), "valid": (flags[:n].cpu().numpy() & 1) > 0,
            "passed": (flags[:n].cpu().numpy() & 2) > 0, "splats": splats[:n], "windows": wins[:n],
            "stats": nat.stats_dict(stats.cpu().numpy())}


def bin_sort(dscene: DeviceScene, surv_inst, surv_gid, cam, opts: RenderOptions, cap_entries: int | None = None):
    """Stages (c)+(d): -> dict(order_idx, entry_idx, counts, splats, stats)."""
    import torch

    lib = nat.load()
    dev = dscene.device
    sv = _survivor_tensor(surv_inst, surv_gid, dev)
    n = int(sv.shape[0])
    cap_e = int(cap_entries if cap_entries is not None else max(1 << 16, 64 * n))
    ws = Workspace(dscene, cam.width, cam.height, cap_s=max(n, 1), cap_e=cap_e, tile_size=opts.tile_size)
    ts = int(opts.tile_size)
    n_tiles = ((cam.width + ts - 1) // ts) * ((cam.height + ts - 1) // ts)
    splats = torch.empty((max(n, 1), nat.SPLAT_BYTES), dtype=torch.uint8, device=dev)
    wins = torch.empty((max(n, 1), nat.WINDOW_BYTES), dtype=torch.uint8, device=dev)
    entries = torch.empty(max(cap_e, 1), dtype=torch.int32, device=dev)
    offs = torch.empty(n_tiles + 1, dtype=torch.int32, device=dev)
    order = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    stats = torch.empty(nat.STATS_BYTES, dtype=torch.uint8, device=dev)
    camc, optc = nat.camera_struct(cam), opts.struct(cam)
    nat.check(lib.sc_bin_sort(ctypes.byref(dscene.struct), nat.ptr(sv), n, ctypes.byref(camc), ctypes.byref(optc),
                              ctypes.byref(ws.struct), nat.ptr(splats), nat.ptr(wins), nat.ptr(entries), nat.ptr(offs),
                              nat.ptr(order), nat.ptr(stats), nat.stream_handle()), "sc_bin_sort")
    st = nat.stats_dict(stats.cpu().numpy())
    if st["overflow"]:
        raise nat.NativeError(f"entry capacity {cap_e} too small for {st['entries']} entries")
    return {"order_idx": order[:st["passed"]].cpu().numpy().view(np.uint32).astype(np.int64),
            "entry_idx": entries[:st["entries"]].cpu().numpy().view(np.uint32).astype(np.int64),
            "counts": offs.cpu().numpy().view(np.uint32).astype(np.int64), "splats": splats[:n],
            "windows": wins[:n], "stats": st}


def blend(splats, windows, entry_idx, counts, cam, opts: RenderOptions, n_splats: int | None = None):
    """Stage (e) on explicit entries: -> (image, trans[, contrib_sum, contrib_max]) numpy."""
    import torch

    lib = nat.load()
    dev = splats.device
    n = int(n_splats if n_splats is not None else splats.shape[0])
    h, w = int(cam.height), int(cam.width)
    ent = torch.from_numpy(np.asarray(entry_idx, np.int64).astype(np.uint32).view(np.int32)).to(dev)
    off = torch.from_numpy(np.asarray(counts, np.int64).astype(np.uint32).view(np.int32)).to(dev)
    image = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
    trans = torch.empty((h, w), dtype=torch.float32, device=dev)
    rec = opts.record_contributions
    csum = torch.empty((h, w), dtype=torch.float32, device=dev) if rec else None
    cmax = torch.empty(max(n, 1), dtype=torch.float32, device=dev) if rec else None
    fo = nat.ScFrameOut()
    fo.image, fo.trans = nat.ptr(image), nat.ptr(trans)
    fo.contrib_sum, fo.contrib_max = nat.ptr(csum), nat.ptr(cmax)
    camc, optc = nat.camera_struct(cam), opts.struct(cam)
    nat.check(lib.sc_blend(nat.ptr(splats), nat.ptr(windows), n, nat.ptr(ent) if ent.numel() else 0, nat.ptr(off),
                           ctypes.byref(camc), ctypes.byref(optc), ctypes.byref(fo), nat.stream_handle()),
              "sc_blend")
    res = {"image": image.cpu().numpy(), "trans": trans.cpu().numpy()}
    if rec:
        res["contrib_sum"] = csum.cpu().numpy()
        res["contrib_max"] = cmax[:n].cpu().numpy()
    return res
