"""Distribution of the frame path's (16x16 tile, 8x4 block) list lengths per
config-3 view (profiling only): which lists set the blend's tail.

    python scripts/blend_lists.py [view ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

views = [int(v) for v in sys.argv[1:]] or [0, 1, 2]
wl = workloads.config3()
r = Renderer(wl.scene)
for v in views:
    cam = wl.cameras[v]
    _, st, dbg = r.render(cam, to_host=False, debug=True)
    off = dbg["block_offsets"]
    ln = np.diff(off)
    nz = ln[ln > 0]
    tot = ln.sum()
    srt = np.sort(ln)[::-1]
    print(f"view {v}: lists {ln.size} nonempty {nz.size} entries {tot} mean {nz.mean():.0f} "
          f"p50 {np.percentile(nz, 50):.0f} p90 {np.percentile(nz, 90):.0f} p99 {np.percentile(nz, 99):.0f} "
          f"p99.9 {np.percentile(nz, 99.9):.0f} max {ln.max()}")
    print("   top 16:", srt[:16].tolist())
    for th in (2048, 4096, 8192, 16384):
        sel = ln >= th
        print(f"   >= {th}: {sel.sum()} lists, {ln[sel].sum() / tot:.3f} of entries")
    # per-tile: how unequal are the 8 lists of a tile
    t8 = ln[: (ln.size // 8) * 8].reshape(-1, 8)
    heavy = np.argsort(-t8.max(1))[:5]
    for t in heavy:
        print(f"   tile {t}: {t8[t].tolist()}")
