"""Benchmark: 1080p FPS of the ~100M-Gaussian instanced scene (BASELINE config 3).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one frame of the composed-scene path (prep, cull + visibility MLP,
instanced projection, depth sort + tile binning, blend) over config 3:
~1,000 instances of 8 synthetic 100K-Gaussian assets (100M instantiated),
1920x1080, cycling the near / mid / far views.  Multi-GPU (torchrun): frames
are sharded across ranks (each rank renders its own K frames; weak scaling,
no collective on the render path — NCCL only for the barrier and the
max-over-ranks timing).

Timing: W untimed warm-up frames, then K frames each bracketed by CUDA events
on the rendering stream, L2 flushed (256 MiB write) before every frame and
excluded from the event time; max over ranks.  ``e2e`` repeats the frames
through the public API ``render_composed`` (camera in, image + transmittance
+ counters copied back to the host every frame), wall clock.

The CPU baseline (and ``--impl reference``) is the oracle port (oracle/: the
reference's numba kernels restated in C, OpenMP on every host core, plus the
restated scene / MLP stages) rendering whole config-3 frames: the reference
arm renders the same W + K frame near/mid/far cycle as this arm; the
``cpu_baseline`` of this arm is one full far-view frame (~20-40 s).
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "1080p FPS, ~100M-Gaussian instanced scene; peak VRAM GB; PSNR vs CPU oracle"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--config", choices=["cfg1", "cfg2", "cfg3", "cfg5"], default="cfg3")
    p.add_argument("--shard", choices=["frames", "bands"], default="frames",
                   help="multi-GPU: frames of the path per rank (weak scaling) or screen bands of every frame "
                        "(strong scaling, bands gathered to rank 0 by P2P copies)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=None)
    p.add_argument("--frames-in-flight", type=int, default=2,
                   help="frames rendered concurrently on separate streams (own workspaces); 1 = serial")
    p.add_argument("--e2e-frames-in-flight", type=int, default=3,
                   help="frames in flight for the end-to-end pass through render_path (one more than the device "
                        "pass: the host's wake-up after each frame's copy then never leaves the GPU one frame)")
    return p.parse_args()


def build_workload(name):
    from paper_2511_19202_b200 import workloads
    if name == "cfg1":
        return workloads.config1()
    if name == "cfg2":
        return workloads.config2(frames=3)
    if name == "cfg5":
        return workloads.config5(frames=8)
    return workloads.config3()


def describe(wl, args, n):
    cam = wl.cameras[0]
    return {"workload": {"cfg1": "config 1: 10K cloud x 1 instance, 256x256",
                         "cfg2": "config 2: 100K shell x 16 instances, 1080p orbit",
                         "cfg3": "config 3: ~1,000 instances of 8 synthetic 100K assets (~100M instantiated), "
                                 "1080p, near/mid/far views cycled",
                         "cfg5": "config 5: the config-3 scene on a 4K (3840x2160) orbit camera path"}[args.config],
            "width": int(cam.width), "height": int(cam.height), "instances": wl.scene.n_instances,
            "instantiated_gaussians": wl.scene.n_instantiated, "views": len(wl.cameras),
            "mlp": "random-init 16->32->32->1 per asset, output bias calibrated to keep ~65% of uniform queries",
            "l2": "flushed (256 MiB write) before every timed frame (on the frame's stream; inside the timed "
                  "region when frames are in flight, excluded from the serial pass's per-frame events)",
            "frames_in_flight": 1 if args.shard == "bands" and n > 1 else args.frames_in_flight,
            "parallelism": (f"screen bands x{n} (P2P gather to rank 0)" if args.shard == "bands" else f"frames x{n}")
            if n > 1 else "single GPU",
            "generators": {k: v for k, v in wl.meta.items() if k != "instantiated"}}


class ClockSampler:
    """NVML sampling of SM clocks and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz, self.ok = [], set(), None, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            pass
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        import statistics
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_oracle_frame(scene, cam, tables=None):
    from oracle import scene_ref as sr
    t0 = time.perf_counter()
    res = sr.render_composed(scene, cam, tables=tables)
    return time.perf_counter() - t0, res


def host_cpu():
    """(logical cores, CPU model) of this host."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return os.cpu_count(), model


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


def algorithmic_bytes(st, n_assets_gauss, n_inst, pixels):
    """SURVEY §8d per-stage algorithmic bytes / flops for one frame."""
    S, E, Q = st["survivors"], st["entries"], st["mlp_queried"]
    p = 6   # ceil((ceil(log2 n_tiles) + 32) / 8) at 1080p
    return {
        "cull_mlp": (n_assets_gauss * 24 + n_inst * 64 + 8 * S, 3136.0 * Q),
        "project": (8 * S + n_assets_gauss * 56 + 56 * S + 4 * S, 0.0),
        "sort_bin": ((4 * S + 24 * S + 12 * E) + 24 * E * p + 8 * E, 0.0),
        "blend": (4 * E + 36 * E + 12 * pixels, 0.0),
    }


def traffic_from_profiles():
    """DRAM bytes per k_blend launch from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "blend_dram_bytes.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def run_reference(args, rank):
    """The reference's CPU path (oracle port, all host cores) on this arm's workload:
    W warm-up frames, then K timed frames of the same (i + rank) % views cycle,
    each a whole config-3 frame (cull + MLP over every (instance, gaussian) pair,
    instancing, projection, sort / binning, blend).  Scene tables (the per-asset
    feature MLP, instance records) are built once, outside the timed frames, like
    the GPU arm's scene upload.  Under torchrun only rank 0 runs."""
    if rank != 0:
        return
    import numpy as np

    from oracle import scene_ref as sr
    wl = build_workload(args.config)
    cams = wl.cameras
    tabs = sr.SceneTables(wl.scene)
    for i in range(args.warmup):
        cpu_oracle_frame(wl.scene, cams[i % len(cams)], tabs)
    times, per_view = [], {}
    for i in range(args.steps):
        t, _ = cpu_oracle_frame(wl.scene, cams[i % len(cams)], tabs)
        times.append(t)
        per_view.setdefault(i % len(cams), []).append(t)
    tot = sum(times)
    value = args.steps / tot
    cores, model = host_cpu()
    names = ["near", "mid", "far"] if len(cams) == 3 else [str(k) for k in range(len(cams))]
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "FPS", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded reference generators, random-init visibility MLPs)",
            "config": describe(wl, args, 1),
            "per_view_s": {names[k]: float(np.mean(v)) for k, v in sorted(per_view.items())},
            "cpu_baseline": {"value": value, "unit": "FPS", "cores": cores, "cpu": model, "kind": "port",
                             "sample": f"the full workload: {args.warmup} warm-up + {args.steps} timed whole "
                                       f"config-3 frames ({wl.scene.n_instances} instances, "
                                       f"{wl.scene.n_instantiated} instantiated pairs per frame), views cycled "
                                       "as in the GPU arm; wall clock per frame, scene tables built once"},
            "e2e": {"value": value, "unit": "FPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import numpy as np
    import torch

    # SC_BENCH_SINGLE_DEVICE=1 (testing only): every rank on cuda:0, gloo control plane, so the
    # multi-process paths can be exercised on a one-GPU box (NCCL needs one GPU per rank)
    single = os.environ.get("SC_BENCH_SINGLE_DEVICE") == "1"
    if single:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if single:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2511_19202_b200 as pkg
    from paper_2511_19202_b200 import _native as nat
    from paper_2511_19202_b200.scene import Renderer, RenderOptions

    wl = build_workload(args.config)
    cams = wl.cameras
    ncam = len(cams)
    opts = RenderOptions()
    r = Renderer(wl.scene)
    lib = nat.load()
    torch.cuda.reset_peak_memory_stats()
    # warm-up: sizes the workspace for every view (re-renders on overflow)
    for i in range(max(args.warmup, ncam)):
        r.render(cams[(i + rank) % ncam], opts, to_host=False)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    K = args.steps
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(K)]
    stage_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(nat.N_STAGE_EVENTS)] for _ in range(K)]
    frames = [None] * ncam
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    bands = args.shard == "bands" and world > 1
    if bands:   # every rank renders its screen band of every frame; bands go to rank 0 by P2P copies
        from paper_2511_19202_b200 import sharding
        h0 = int(cams[0].height)
        bounds = sharding.split_rows(sharding.tile_rows(h0), world)
        gather = sharding.BandGather((h0, int(cams[0].width), 3), rank, world, device="cuda", transport="p2p")
        for i in range(ncam):   # size the band workspaces (every band is a subset of its frame)
            r.render(cams[i], opts, to_host=False)
        torch.cuda.synchronize()
        dist.barrier()
    F = max(1, args.frames_in_flight)
    streams = [torch.cuda.Stream() for _ in range(F)]
    pframes = [[None] * ncam for _ in range(F)]
    if F > 1:   # size the extra slots' workspaces, allocate every slot's outputs
        for j in range(F):
            for ci in range(ncam):
                pframes[j][ci] = r.render_device(cams[ci], opts, slot=j)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def pipelined_pass():
        """K frames, frame i on stream i % F with workspace slot i % F; one pair of events
        around the whole pass on the main stream (device time, max over ranks later)."""
        main_s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for st in streams:
            st.wait_stream(main_s)
        for i in range(K):
            ci = (i + rank) % ncam
            j = i % F
            with torch.cuda.stream(streams[j]):
                flush.fill_(i & 0xFF)
                pframes[j][ci] = r.render_device(cams[ci], opts, out=pframes[j][ci], slot=j)
        for st in streams:
            main_s.wait_stream(st)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    if F > 1 and not bands:   # untimed warm-up of the pipelined schedule itself
        K_t, K = K, max(args.warmup, F)
        pipelined_pass()
        K = K_t
    launches0 = lib.sc_kernel_launches()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        pipe_ms = pipelined_pass() if (F > 1 and not bands) else None
        pipe_launches = lib.sc_kernel_launches() - launches0
        # serial pass (one frame in flight): per-frame and per-stage events bracket the kernels alone
        for i in range(K):
            ci = i % ncam if bands else (i + rank) % ncam
            flush.fill_(i & 0xFF)
            if bands:
                y0, y1 = sharding.band_pixels(bounds, rank, h0)
                bopts = RenderOptions(band=(y0, y1))
                dist.barrier()
                ev_s[i].record()
                frames[ci] = r.render_device(cams[ci], bopts, out=frames[ci], stage_events=stage_ev[i])
                gather.full[y0:y1].copy_(frames[ci].image[y0:y1], non_blocking=True)   # NVLink P2P into rank 0
                ev_e[i].record()
                torch.cuda.synchronize()
                dist.barrier()   # rank 0's frame is complete
                t = torch.tensor([ev_s[i].elapsed_time(ev_e[i])], device="cuda")
                allt = [torch.empty_like(t) for _ in range(world)]
                dist.all_gather(allt, t)   # control plane: band times for the next frame's split
                bounds = sharding.rebalance(bounds, [float(x) for x in allt])
            else:
                ev_s[i].record()
                frames[ci] = r.render_device(cams[ci], opts, out=frames[ci], stage_events=stage_ev[i])
                ev_e[i].record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    launches = (pipe_launches if pipe_ms is not None else lib.sc_kernel_launches() - launches0)
    if dist:
        dist.barrier()
    dev_ms = [ev_s[i].elapsed_time(ev_e[i]) for i in range(K)]
    if bands:   # a frame takes as long as its slowest band (+ its copy into rank 0's frame)
        t = torch.tensor(dev_ms, device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = [float(x) for x in t]
    stage_ms = {name: [stage_ev[i][j].elapsed_time(stage_ev[i][j + 1]) for i in range(K)]
                for j, name in enumerate(nat.STAGE_NAMES)}
    total_ms = float(sum(dev_ms))   # serial pass
    peak_gb = torch.cuda.max_memory_allocated() / 1e9
    # per frame slot: its workspace (sized on the largest view) + its output frame; the scene is shared
    slot_ws = {k[2]: w.nbytes for k, w in r.workspaces.items() if k[3] == 16}
    frame_bytes = int(cams[0].width) * int(cams[0].height) * 16 + nat.STATS_BYTES
    vram = {"scene_gb": r.dscene.nbytes / 1e9,
            "per_frame_slot_gb": [round((slot_ws[j] + frame_bytes) / 1e9, 3) for j in sorted(slot_ws)],
            "frame_slots": len(slot_ws), "peak_allocated_gb": peak_gb,
            "note": "per slot = workspace (capacities from the largest view, +5 % headroom) + image/T/stats buffers"}
    stats = [nat.stats_dict(f.stats_raw.cpu().numpy()) if f is not None else None for f in frames]
    if any(s and s["overflow"] for s in stats):
        raise RuntimeError("workspace overflow inside the timed region")
    if dist:
        t = torch.tensor([total_ms, peak_gb, pipe_ms or 0.0], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, peak_gb = float(t[0]), float(t[1])
        pipe_ms = float(t[2]) if pipe_ms is not None else None
    frames_done = K if bands else world * K   # bands: all ranks render each of the K frames together

    # ---------------- e2e through the public API ----------------
    e2e = None
    if not args.no_e2e:
        ke = args.e2e_steps or max(K, 240)   # >= 240 frames (~2 s): a 50 ms host hiccup weighs ~2 %
        wl.scene._device = r            # the public API reuses this scene's uploaded copy
        pkg.render_composed(wl.scene, cams[rank % ncam])
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        seq = [cams[(i + rank) % ncam] for i in range(ke)]
        FE = max(1, args.e2e_frames_in_flight) if F > 1 else 1
        if FE > 1:   # warm the path API (its streams, output frames and pinned host buffers)
            for _ in pkg.render_path(wl.scene, seq[:2 * FE], frames_in_flight=FE):
                pass
            torch.cuda.synchronize()
        gc.collect()
        gc.disable()   # no cyclic-GC pause inside the timed host loop
        r.path_wait_s = 0.0
        t0 = time.perf_counter()
        if FE > 1:
            for out, fst in pkg.render_path(wl.scene, seq, frames_in_flight=FE):
                pass
        else:
            for cam in seq:
                out, fst = pkg.render_composed(wl.scene, cam)
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        gc.enable()
        host_busy = e2e_s - r.path_wait_s
        if dist:
            t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t[0])
        h, w = int(cams[0].height), int(cams[0].width)
        e2e = {"value": world * ke / e2e_s, "unit": "FPS",
               "h2d_bytes_per_step": 136 + 80,
               "d2h_bytes_per_step": h * w * 3 * 4 + h * w * 4 + nat.STATS_BYTES,
               "api": (f"paper_2511_19202_b200.render_path(scene, cams, frames_in_flight={FE}) -> RenderOutput per "
                       "frame (numpy image + transmittance)") if FE > 1 else
                      "paper_2511_19202_b200.render_composed -> RenderOutput (numpy image + transmittance)"}
        e2e["peak_vram_gb"] = torch.cuda.max_memory_allocated() / 1e9   # includes the e2e pass's frame slots
        if FE > 1:   # host time per frame not spent waiting on the GPU (render_path's own accounting)
            e2e["host_busy_ms_per_step"] = 1e3 * host_busy / ke
        if bands:
            e2e["sharding"] = "whole frames per rank (the banded path has no host-facing API of its own)"

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---------------- roofline of the dominant stage ----------------
    hbm, tflops, src = peaks()
    mean_stage = {k: float(np.mean(v)) for k, v in stage_ms.items()}
    per_view = {}
    for i in range(K):
        per_view.setdefault(i % ncam if bands else (i + rank) % ncam, []).append(dev_ms[i])
    n_gauss = sum(len(a.asset) for a in wl.scene.assets)
    pixels = int(cams[0].width) * int(cams[0].height)
    # views rendered in the serial pass (all of them unless K < the number of cameras)
    alg = [algorithmic_bytes(st_, n_gauss, wl.scene.n_instances, pixels) for st_ in stats if st_]
    def stage_roof(name):
        b = float(np.mean([a[name][0] for a in alg]))
        f = float(np.mean([a[name][1] for a in alg]))
        t = mean_stage[name] / 1e3
        r_ = {"bound": "hbm", "achieved": b / t / 1e9, "peak": hbm, "unit": "GB/s",
              "algorithmic_bytes": b, "ms": mean_stage[name]}
        if f > 0:
            r_["tensor_achieved_tflops"] = f / t / 1e12
            r_["tensor_frac"] = r_["tensor_achieved_tflops"] / tflops
        r_["frac"] = r_["achieved"] / r_["peak"]
        return r_

    roof_stages = {k: stage_roof(k) for k in mean_stage}
    # dominant single kernel: k_blend (the stage-3 -> stage-4 events bracket only
    # k_tile_order (~0.03 ms) and k_blend)
    roof = dict(roof_stages["blend"])
    roof["kernel"] = "k_blend"
    roof["peak_source"] = f"{src} (MEASURED_PEAKS.json hbm_gbs)" if src == "measured" else src
    roof["units"] = "SURVEY §8d: 4 E + 36 E + 12 P bytes per launch, E = reference tile entries, P = pixels"
    tr = traffic_from_profiles()
    roof["traffic"] = tr.get("per_launch_bytes") if tr and tr.get("kernel") == "k_blend" else None
    t_roof = float(np.mean([sum(b for b, _ in a.values()) / (hbm * 1e9) + sum(f for _, f in a.values()) /
                            (tflops * 1e12) for a in alg]))
    head_ms = pipe_ms if pipe_ms is not None else total_ms
    frame_roof = {"t_roof_ms": 1e3 * t_roof, "t_measured_ms": head_ms / K, "frac": 1e3 * t_roof / (head_ms / K)}

    # ---------------- CPU oracle beside it: baseline + PSNR ----------------
    cpu = None
    quality = None
    if not args.no_cpu_baseline:
        cam = cams[-1]
        t_cpu, ref = cpu_oracle_frame(wl.scene, cam)
        cores, model = host_cpu()
        cpu = {"value": 1.0 / t_cpu, "unit": "FPS", "cores": cores, "cpu": model, "kind": "port",
               "sample": f"one whole config-3 frame (the last view of the cycle, {ref.stats['instantiated']} "
                         f"instantiated of {wl.scene.n_instantiated} pairs), {t_cpu:.1f} s wall clock, "
                         "OpenMP on every host core"}
        gout, gst = pkg.render_composed(wl.scene, cam)
        from paper_2511_19202_b200.raster import psnr_uncapped, ssim
        quality = {"psnr_db": psnr_uncapped(gout.image, ref.out.image), "ssim": ssim(gout.image, ref.out.image),
                   "max_abs": float(np.abs(gout.image - ref.out.image).max()),
                   "frame": "full config-3 frame (last view), each side with its own cull/MLP survivors",
                   "survivors_gpu": gst.instantiated, "survivors_cpu": ref.stats["instantiated"]}
        del ref

    value = frames_done / (head_ms / 1e3)
    line = {
        "metric": METRIC, "value": value, "unit": "FPS", "n_gpus": world, "steps": K, "warmup": args.warmup,
        "ms_per_step": head_ms / K,
        "serial": {"value": frames_done / (total_ms / 1e3), "ms_per_step": total_ms / K,
                   "note": "one frame in flight; per_view_ms, stage_ms and the rooflines come from this pass"}, "higher_is_better": True, "scaling": "strong" if bands else "weak",
        "vs_baseline": None,
        "dtype": "f64 (cull, projection, keys) + fp16/f32 tensor-core MLP + fp32 blend",
        "data": "synthetic (seeded reference generators, random-init visibility MLPs)",
        "config": describe(wl, args, world),
        "peak_vram_gb": peak_gb, "vram": vram,
        "psnr_vs_cpu_oracle": quality,
        "per_view_ms": {["near", "mid", "far"][k] if ncam == 3 else str(k): float(np.mean(v))
                        for k, v in sorted(per_view.items())},
        "stage_ms": mean_stage,
        "frame_counts": [{k: s[k] for k in ("pairs_tested", "frustum_passed", "mlp_queried", "mlp_culled", "block_entries",
                                            "survivors", "passed", "entries")} for s in stats if s],
        "roofline": roof, "roofline_stages": roof_stages, "roofline_frame": frame_roof,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
