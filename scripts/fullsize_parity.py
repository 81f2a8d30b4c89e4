"""Full-size parity runs: config 2 orbit frames and config 3
near / mid / far at 1080p, GPU frame path vs the CPU oracle.

Per frame:
  * survivors: GPU cull + MLP vs the oracle's (frustum set equal; MLP flips all
    within the fp16 logit margin of the threshold);
  * order: the frame path's (depth, index) order of the GPU's own survivors vs the
    oracle's argsort(depth, kind="stable") over the same survivors (bit-exact);
  * image: GPU frame vs the oracle rendering the GPU's own survivors (max-abs,
    uncapped PSNR; contract 5e-3 / 80 dB) and vs the oracle's whole pipeline
    (PSNR >= 45 dB, SSIM >= 0.995).

    python scripts/fullsize_parity.py [cfg2|cfg3|all] > gpurun_out/fullsize_parity.json
"""

import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import raster_ref as rr  # noqa: E402
from oracle import scene_ref as sr  # noqa: E402
from paper_2511_19202_b200.scene import RenderOptions, Renderer  # noqa: E402
from paper_2511_19202_b200.workloads import config2, config3  # noqa: E402

LOGIT_MARGIN = 0.0025


def psnr(a, b):
    mse = float(((np.asarray(a, np.float64) - b) ** 2).mean())
    return math.inf if mse == 0 else -10 * math.log10(mse)


def frame(wl, cam, name):
    t0 = time.perf_counter()
    tabs = sr.SceneTables(wl.scene)
    r = Renderer(wl.scene)
    out, st, dbg = r.render(cam, RenderOptions(), return_survivors=True, debug=True)
    surv = out.survivors
    g_inst, g_gid = surv[:, 0], surv[:, 1]
    # oracle whole pipeline
    ref = sr.render_composed(wl.scene, cam, tables=tabs)
    c = ref.cull
    # survivor sets: compare as pair ids
    po = tabs.pair_offset
    g_pair = po[g_inst] + g_gid
    o_pair = po[c.surv_inst] + c.surv_gid
    only_gpu = np.setdiff1d(g_pair, o_pair, assume_unique=True)
    only_ora = np.setdiff1d(o_pair, g_pair, assume_unique=True)
    flips = np.concatenate([only_gpu, only_ora])
    flip_logit = np.abs(c.logit[flips]) if flips.size else np.zeros(0)
    not_queried = int(np.count_nonzero(~(c.flags[flips] & 2).astype(bool))) if flips.size else 0
    # oracle on the GPU's own survivors
    m, ls, q, op, sh, deg = sr.instantiate(tabs, cam, g_inst, g_gid)
    st_o = rr.Stages()
    same = rr.render_arrays(m, ls, q, op, sh, deg, cam, stages=st_o)
    order_equal = bool(np.array_equal(dbg["order"], st_o.order_idx))
    d_same = np.abs(out.image - same.image)
    rec = {
        "frame": name, "survivors_gpu": int(g_pair.size), "survivors_oracle": int(o_pair.size),
        "frustum_passed_gpu": st.frustum_passed, "frustum_passed_oracle": int(np.count_nonzero(c.flags & 1)),
        "mlp_flips": int(flips.size), "mlp_flips_max_abs_logit": float(flip_logit.max()) if flips.size else 0.0,
        "mlp_flips_not_queried": not_queried,
        "passed_gpu": st.passed, "passed_oracle_same_survivors": int(same.passed_count),
        "order_bit_exact": order_equal, "order_len": int(st_o.order_idx.size),
        "block_entries": st.block_entries, "reference_tile_entries": int(st_o.entry_idx.size),
        "same_survivors": {"max_abs": float(d_same.max()), "psnr_db": psnr(out.image, same.image),
                           "trans_max_abs": float(np.abs(out.final_transmittance - same.final_transmittance).max())},
        "whole_pipeline": {"psnr_db": psnr(out.image, ref.out.image), "ssim": float(rr.ssim(out.image, ref.out.image)),
                           "max_abs": float(np.abs(out.image - ref.out.image).max())},
        "wall_s": time.perf_counter() - t0,
    }
    rec["pass"] = bool(rec["frustum_passed_gpu"] == rec["frustum_passed_oracle"] and order_equal and
                       (flips.size == 0 or rec["mlp_flips_max_abs_logit"] < LOGIT_MARGIN) and not_queried == 0 and
                       rec["same_survivors"]["max_abs"] <= 5e-3 and rec["same_survivors"]["psnr_db"] >= 80 and
                       rec["whole_pipeline"]["psnr_db"] >= 45 and rec["whole_pipeline"]["ssim"] >= 0.995)
    print(json.dumps(rec), flush=True)
    del r
    torch.cuda.empty_cache()
    return rec


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    torch.cuda.set_device(0)
    recs = []
    if which in ("cfg2", "all"):
        wl = config2()
        for f in (0, 24, 48, 72, 96):
            recs.append(frame(wl, wl.cameras[f], f"cfg2 orbit frame {f}"))
        del wl
    if which in ("cfg3", "all"):
        wl = config3()
        for v, nm in enumerate(("near", "mid", "far")):
            recs.append(frame(wl, wl.cameras[v], f"cfg3 {nm}"))
    print(json.dumps({"summary": {"frames": len(recs), "all_pass": all(r["pass"] for r in recs),
                                  "cores": os.cpu_count()}}), flush=True)


if __name__ == "__main__":
    main()
