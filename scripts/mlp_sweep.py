"""Config 4: visibility-MLP batched query sweep (BASELINE configs[3]).

    python scripts/mlp_sweep.py [out.json]

Two modes:
  * materialised inputs: sc_vis_mlp_forward on Q rows of uniform [-1, 1]^16 f32
    (seed 0, generated on the device), Q in {1M, 4M, 16M, 64M, 200M};
    68 B per query (64 B f32 inputs + 4 B logit), 3,136 flop per query;
    decisions checked against the f64 host MLP on the first 1M rows;
  * fused-from-scene: the cull kernel of a config-3 frame (inputs built on
    chip, never in HBM): MLP queries per second of the cull + MLP stage.
CUDA-event timing on the current stream, 2 warm-up + 5 timed launches.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2511_19202_b200 import nn, synth, workloads
from paper_2511_19202_b200.asset import prepare

LOGIT_MARGIN = 0.01
torch.cuda.set_device(0)
a = prepare(synth.make_shell(500, seed=3))
model = workloads.calibrated_model(a, seed=3)
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}
rows = []
for q in (1 << 20, 4 << 20, 16 << 20, 64 << 20, 200_000_000):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.rand((q, 16), generator=g, device="cuda", dtype=torch.float32) * 2.0 - 1.0
    out = nn.forward(model, x)
    for _ in range(1):
        nn.forward(model, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        out = nn.forward(model, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    n_chk = min(q, 1 << 20)
    ref = model.vis_mlp.forward_host(x[:n_chk].cpu().numpy())[:, 0]
    got = out[:n_chk, 0].cpu().numpy()
    flips = (got >= 0) != (ref >= 0)
    worst = float(np.abs(ref[flips]).max()) if flips.any() else 0.0
    rows.append({"queries": q, "ms": ms, "queries_per_s": q / ms * 1e3, "gb_per_s": 68.0 * q / ms / 1e6,
                 "hbm_frac": 68.0 * q / ms / 1e6 / peaks["hbm_gbs"], "tflops": 3136.0 * q / ms / 1e9,
                 "tensor_frac": 3136.0 * q / ms / 1e9 / peaks["bf16_tflops"],
                 "checked_rows": n_chk, "decision_flips": int(flips.sum()), "max_abs_logit_at_flip": worst,
                 "max_abs_logit_diff": float(np.abs(got - ref).max()), "flips_within_margin": worst < LOGIT_MARGIN})
    print(json.dumps(rows[-1]), flush=True)
    del x, out
    torch.cuda.empty_cache()

# fused-from-scene: the cull + MLP stage of config-3 frames
from paper_2511_19202_b200.scene import Renderer

wl = workloads.config3()
r = Renderer(wl.scene)
fused = []
for ci, cam in enumerate(wl.cameras):
    r.render(cam, to_host=False)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    f = r.render_device(cam, stage_events=ev)
    torch.cuda.synchronize()
    from paper_2511_19202_b200 import _native as nat
    st = nat.stats_dict(f.stats_raw.cpu().numpy())
    ms = ev[0].elapsed_time(ev[1])
    fused.append({"view": ["near", "mid", "far"][ci], "pairs_tested": st["pairs_tested"],
                  "mlp_queried": st["mlp_queried"], "cull_mlp_ms": ms,
                  "queries_per_s": st["mlp_queried"] / ms * 1e3, "tflops": 3136.0 * st["mlp_queried"] / ms / 1e9})
    print(json.dumps(fused[-1]), flush=True)
res = {"config": "config 4: visibility-MLP batched query sweep (fp16 tensor cores, fp32 accumulate)",
       "materialised": rows, "fused_from_scene": fused, "device": torch.cuda.get_device_name(0),
       "flop_per_query": 3136, "bytes_per_query_materialised": 68}
out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "mlp_sweep.json")
json.dump(res, open(out_path, "w"), indent=1)
