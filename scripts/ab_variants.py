"""A/B timing of library builds: per-view and per-stage ms on config 3 (L2 flushed before each frame).

    python scripts/ab_variants.py lib_a.so lib_b.so ...   (each variant in its own process)
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] != "--child":
    for lib in sys.argv[1:]:
        env = dict(os.environ, SPLATCULL_B200_VARIANT=lib)
        r = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(os.path.basename(lib), r.stdout.strip() or r.stderr[-2000:], flush=True)
    # images of every variant against the first one's (same survivors and lists: blend differences only)
    import numpy as np
    first = sys.argv[1]
    for lib in sys.argv[2:]:
        d = []
        for vi in range(3):
            try:
                a, b = np.load(first + f".v{vi}.npy"), np.load(lib + f".v{vi}.npy")
            except OSError:
                continue
            mse = float(np.mean((a.astype(np.float64) - b) ** 2))
            d.append((float(np.abs(a - b).max()), 10 * np.log10(1.0 / mse) if mse > 0 else float("inf")))
        print("images", os.path.basename(lib), "vs", os.path.basename(first), "(max-abs, PSNR dB) per view:", d)
    sys.exit(0)

sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2511_19202_b200 import _native as nat
from paper_2511_19202_b200 import workloads
from paper_2511_19202_b200.scene import Renderer

reps = int(os.environ.get("AB_REPS", "6"))
wl = workloads.config3()
r = Renderer(wl.scene)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = {}
for vi, cam in enumerate(wl.cameras):
    for _ in range(2):
        r.render(cam, to_host=False)
    frame = None
    per = []
    for _ in range(reps):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(nat.N_STAGE_EVENTS)]
        frame = r.render_device(cam, out=frame, stage_events=ev)
        torch.cuda.synchronize()
        per.append([ev[j].elapsed_time(ev[j + 1]) for j in range(nat.N_STAGE_EVENTS - 1)])
    per = np.median(np.array(per), axis=0)
    np.save(os.environ["SPLATCULL_B200_VARIANT"] + f".v{vi}.npy", frame.image.cpu().numpy())
    res[("near", "mid", "far")[vi]] = [round(float(x), 3) for x in per] + [round(float(per.sum()), 3)]
tot = np.mean([v[-1] for v in res.values()])
print(json.dumps({"views(cull,proj,sort,blend,total)": res, "mean_ms": round(float(tot), 3),
                  "fps": round(1000 / float(tot), 1)}))
