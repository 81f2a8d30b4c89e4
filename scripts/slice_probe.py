"""Headroom of a two-slice frame (profiling only): blend the first R survivors of the
depth order, then emit / sort / blend the rest only into blocks that are not yet
saturated.  For each config-3 view and slice point R (fraction of the passed
survivors), reports the fraction of block entries the second slice could skip.

    python scripts/slice_probe.py      (builds the instrumented library)
"""
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2511_19202_b200", "csrc"), "debug", "-j8"], check=True)
os.environ["SPLATCULL_B200_DEBUG_LIB"] = "1"
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2511_19202_b200 import _native as nat
from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

wl = workloads.config3()
r = Renderer(wl.scene)
lib = nat.load()
fn = lib.sc_debug_blend_used
fn.restype = ctypes.c_int
fn.argtypes = [ctypes.c_void_p, ctypes.c_int64]
res = {}
for view, cam in enumerate(wl.cameras[:3]):
    _frame, st, dbg = r.render(cam, to_host=False, debug=True)
    torch.cuda.synchronize()
    nb = 8 * ((cam.width + 15) // 16) * ((cam.height + 15) // 16)
    buf = np.zeros((nb, 2), dtype=np.uint32)
    assert fn(buf.ctypes.data_as(ctypes.c_void_p), nb) == 0
    dev = "cuda"
    order = torch.from_numpy(dbg["order"]).to(dev)
    n_pass = order.numel()
    rank = torch.empty(int(order.max()) + 1, dtype=torch.int64, device=dev)
    rank[order] = torch.arange(n_pass, device=dev)
    off = torch.from_numpy(dbg["block_offsets"]).to(dev)
    ent = torch.from_numpy(dbg["block_entries"]).to(dev)
    er = rank[ent]                                    # depth rank of every block entry
    lens = (off[1:] - off[:-1])
    used = torch.minimum(torch.from_numpy(buf[:, 1].astype(np.int64)).to(dev), lens)
    sat = used < lens                                 # block saturated inside its list
    # depth rank at which the block saturates (rank of its last streamed entry), inf if never
    last = torch.clamp(off[:-1] + used - 1, min=0)
    r_sat = torch.where(sat & (used > 0), er[last], torch.full_like(last, 1 << 62))
    blk = torch.repeat_interleave(torch.arange(nb, device=dev), lens)
    rows = {}
    for f in (0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7):
        R = int(f * n_pass)
        rs = r_sat[blk]
        skip = ((rs < R) & (er >= R)).sum().item()
        slice1 = (er < R).sum().item()
        rows[f] = {"slice1_entries_frac": round(slice1 / ent.numel(), 4), "skippable_frac": round(skip / ent.numel(), 4)}
    res[("near", "mid", "far")[view]] = {"entries": int(ent.numel()), "passed": n_pass, "by_slice_point": rows}
    print(view, json.dumps(res[("near", "mid", "far")[view]]), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "slice_probe.json"), "w"), indent=1)
