"""PyTorch custom ops (``torch.ops.splatcull.*``) over the C ABI of libsplatcull_b200.so.

Every GPU entry point of the package goes through these ops: the Python API
(``Renderer``, ``render``, ``render_composed``, ``stages``, ``nn.forward``,
``encode_features``, visibility extraction) packs its arguments into plain
tensors / int / float lists and calls ``torch.ops.splatcull.<op>``, whose
implementation builds the C structs of include/splatcull_b200.h and calls the
library on the current CUDA stream.  Each op has a fake (meta) kernel, so the
path traces under ``torch.compile`` / FakeTensorMode, and none synchronises
with the host, so frames can be captured in CUDA graphs.

Reference interfaces the ops replace:
  render_frame_ / render_frame   scene.render_composed, raster.render (sc/raster.py:240-339)
  cull_mlp                       render_composed steps (1)-(2)
  project                        project_kernel (sc/_kernels.py:13-134) + eval_sh_colors (sc/raster.py:198-226)
  bin_sort                       argsort(depth, stable) + bin_tiles (sc/raster.py:319, sc/_kernels.py:137-165)
  blend                          composite_tiles + finish (sc/_kernels.py:168-275, sc/raster.py:267-282)
  vis_mlp_forward                nn.forward
  encode_features                nn.encode_features
  visibility_labels_or_          sampling.visible_labels (sc/sampling.py:206-213)

Packed argument layouts (all plain lists, so the schemas stay simple):
  scene       [mean_opa, quat, scale_smax, sh, features, appear, assets, instances, vis_weights] tensors
  scene_meta  [n_gauss, sh_stride, n_assets, n_instances, n_models, n_pairs]
  cam_f       [pos x3, rot x9 (rows right, down, forward), focal, tan_x, tan_y, near]; cam_i [width, height]
  opt_f       [radius_clip, stop_transmittance, bg r, g, b, dilation, frustum_G]
  opt_i       [tile_size, sh_degree_eval, record_contributions, use_mlp, frustum_mode, exact_projection,
               band_y0, band_y1]
  ws_meta     [n_instances, max_pairs, cap_survivors, cap_entries] (workspace = uint8 device tensor)
"""

from __future__ import annotations

import ctypes

import torch
from torch.library import custom_op

from . import _native as nat

STATS_BYTES = nat.STATS_BYTES


# ---------------------------------------------------------------------------
# packing helpers (host)
# ---------------------------------------------------------------------------

def _scene_struct(scene: list[torch.Tensor], meta: list[int]) -> nat.ScScene:
    s = nat.ScScene()
    mean_opa, quat, scale_smax, sh, features, appear, assets, instances, weights = scene
    s.mean_opa, s.quat, s.scale_smax = nat.ptr(mean_opa), nat.ptr(quat), nat.ptr(scale_smax)
    s.sh, s.features, s.appear = nat.ptr(sh), nat.ptr(features), nat.ptr(appear)
    s.assets, s.instances, s.vis_weights = nat.ptr(assets), nat.ptr(instances), nat.ptr(weights)
    s.n_gauss, s.sh_stride, s.n_assets, s.n_instances, s.n_models, s.n_pairs = (int(v) for v in meta)
    return s


def _camera_struct(cam_f: list[float], cam_i: list[int]) -> nat.ScCamera:
    c = nat.ScCamera()
    c.pos[:] = [float(v) for v in cam_f[0:3]]
    c.rot[:] = [float(v) for v in cam_f[3:12]]
    c.focal, c.tan_x, c.tan_y, c.near_ = (float(v) for v in cam_f[12:16])
    c.width, c.height = int(cam_i[0]), int(cam_i[1])
    return c


def _opts_struct(opt_f: list[float], opt_i: list[int]) -> nat.ScOpts:
    o = nat.ScOpts()
    o.radius_clip, o.stop_transmittance = float(opt_f[0]), float(opt_f[1])
    o.background[:] = [float(v) for v in opt_f[2:5]]
    o.dilation, o.frustum_G = float(opt_f[5]), float(opt_f[6])
    (o.tile_size, o.sh_degree_eval, o.record_contributions, o.use_mlp, o.frustum_mode, o.exact_projection,
     o.band_y0, o.band_y1) = (int(v) for v in opt_i)
    return o


def _ws_struct(workspace: torch.Tensor, ws_meta: list[int]) -> nat.ScWorkspace:
    w = nat.ScWorkspace()
    w.base, w.bytes = nat.ptr(workspace), int(workspace.numel())
    w.n_instances, w.max_pairs, w.cap_survivors, w.cap_entries = (int(v) for v in ws_meta)
    return w


def _stream(t: torch.Tensor) -> int:
    return int(torch.cuda.current_stream(t.device).cuda_stream)


def pack_camera(cam) -> tuple[list[float], list[int]]:
    c = nat.camera_struct(cam)
    return list(c.pos) + list(c.rot) + [c.focal, c.tan_x, c.tan_y, c.near_], [int(c.width), int(c.height)]


def pack_opts(o: nat.ScOpts) -> tuple[list[float], list[int]]:
    return ([o.radius_clip, o.stop_transmittance] + list(o.background) + [o.dilation, o.frustum_G],
            [o.tile_size, o.sh_degree_eval, o.record_contributions, o.use_mlp, o.frustum_mode, o.exact_projection,
             o.band_y0, o.band_y1])


def n_tiles(cam_i: list[int], tile_size: int) -> int:
    return ((int(cam_i[0]) + tile_size - 1) // tile_size) * ((int(cam_i[1]) + tile_size - 1) // tile_size)


# ---------------------------------------------------------------------------
# whole frame (stages a-e, or c-e on injected survivors)
# ---------------------------------------------------------------------------

@custom_op("splatcull::render_frame_", mutates_args=("workspace", "image", "trans", "stats", "contrib_sum",
                                                      "contrib_max", "survivors_out", "debug"))
def render_frame_(scene: list[torch.Tensor], scene_meta: list[int], cam_f: list[float], cam_i: list[int],
                  opt_f: list[float], opt_i: list[int], workspace: torch.Tensor, ws_meta: list[int],
                  image: torch.Tensor, trans: torch.Tensor, stats: torch.Tensor, contrib_sum: torch.Tensor | None,
                  contrib_max: torch.Tensor | None, survivors_out: torch.Tensor | None,
                  survivors_in: torch.Tensor | None, stage_events: list[int], debug: list[torch.Tensor]) -> None:
    """sc_render_composed (survivors_in None) / sc_render_survivors into caller buffers.

    stage_events: 0 or 5 raw cudaEvent_t handles; debug: [] or [order, block_offsets,
    block_entries, block_codes] int32 device tensors (sc_frame_debug)."""
    lib = nat.load()
    sc = _scene_struct(scene, scene_meta)
    cam = _camera_struct(cam_f, cam_i)
    opts = _opts_struct(opt_f, opt_i)
    ws = _ws_struct(workspace, ws_meta)
    fo = nat.ScFrameOut()
    fo.image, fo.trans, fo.stats = nat.ptr(image), nat.ptr(trans), nat.ptr(stats)
    fo.contrib_sum, fo.contrib_max = nat.ptr(contrib_sum), nat.ptr(contrib_max)
    fo.survivors = nat.ptr(survivors_out)
    handles = None
    if stage_events:
        handles = (ctypes.c_void_p * nat.N_STAGE_EVENTS)(*[int(h) for h in stage_events[:nat.N_STAGE_EVENTS]])
        fo.stage_events = ctypes.cast(handles, ctypes.c_void_p)
        fo.n_stage_events = nat.N_STAGE_EVENTS
    dbg = None
    if debug:
        dbg = nat.ScFrameDebug()
        dbg.order, dbg.block_offsets, dbg.block_entries, dbg.block_codes = (nat.ptr(t) for t in debug)
        fo.debug = ctypes.addressof(dbg)
    st = _stream(image)
    if survivors_in is not None:
        nat.check(lib.sc_render_survivors(ctypes.byref(sc), nat.ptr(survivors_in), int(survivors_in.shape[0]),
                                          ctypes.byref(cam), ctypes.byref(opts), ctypes.byref(ws), ctypes.byref(fo),
                                          st), "sc_render_survivors")
    else:
        nat.check(lib.sc_render_composed(ctypes.byref(sc), ctypes.byref(cam), ctypes.byref(opts), ctypes.byref(ws),
                                         ctypes.byref(fo), st), "sc_render_composed")


@render_frame_.register_fake
def _render_frame_fake(scene, scene_meta, cam_f, cam_i, opt_f, opt_i, workspace, ws_meta, image, trans, stats,
                       contrib_sum, contrib_max, survivors_out, survivors_in, stage_events, debug):
    return None


@custom_op("splatcull::render_frame", mutates_args=("workspace",))
def render_frame(scene: list[torch.Tensor], scene_meta: list[int], cam_f: list[float], cam_i: list[int],
                 opt_f: list[float], opt_i: list[int], workspace: torch.Tensor,
                 ws_meta: list[int]) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
    """Functional whole frame -> (image (H, W, 3) f32, transmittance (H, W) f32, stats uint8[STATS_BYTES])."""
    if int(opt_i[2]):
        raise ValueError("render_frame: use render_frame_ with contribution buffers for record_contributions")
    dev = workspace.device
    h, w = int(cam_i[1]), int(cam_i[0])
    image = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
    trans = torch.empty((h, w), dtype=torch.float32, device=dev)
    stats = torch.empty(STATS_BYTES, dtype=torch.uint8, device=dev)
    render_frame_(scene, scene_meta, cam_f, cam_i, opt_f, opt_i, workspace, ws_meta, image, trans, stats, None,
                  None, None, None, [], [])
    return image, trans, stats


@render_frame.register_fake
def _render_frame_fake2(scene, scene_meta, cam_f, cam_i, opt_f, opt_i, workspace, ws_meta):
    h, w = int(cam_i[1]), int(cam_i[0])
    return (workspace.new_empty((h, w, 3), dtype=torch.float32), workspace.new_empty((h, w), dtype=torch.float32),
            workspace.new_empty((STATS_BYTES,), dtype=torch.uint8))


# ---------------------------------------------------------------------------
# stage-level ops (parity tests inject inputs at any stage boundary)
# ---------------------------------------------------------------------------

@custom_op("splatcull::cull_mlp", mutates_args=("workspace",))
def cull_mlp(scene: list[torch.Tensor], scene_meta: list[int], cam_f: list[float], cam_i: list[int],
             opt_f: list[float], opt_i: list[int], workspace: torch.Tensor, ws_meta: list[int],
             cap: int) -> tuple[torch.Tensor, torch.Tensor]:
    """Stages (a)+(b) -> (survivors (cap, 2) int32 [instance, gaussian] in flat order, stats)."""
    lib = nat.load()
    dev = workspace.device
    surv = torch.empty((max(cap, 1), 2), dtype=torch.int32, device=dev)
    stats = torch.empty(STATS_BYTES, dtype=torch.uint8, device=dev)
    sc, cam, opts, ws = (_scene_struct(scene, scene_meta), _camera_struct(cam_f, cam_i),
                         _opts_struct(opt_f, opt_i), _ws_struct(workspace, ws_meta))
    nat.check(lib.sc_cull_mlp(ctypes.byref(sc), ctypes.byref(cam), ctypes.byref(opts), ctypes.byref(ws),
                              nat.ptr(surv), int(cap), nat.ptr(stats), _stream(workspace)), "sc_cull_mlp")
    return surv, stats


@cull_mlp.register_fake
def _cull_fake(scene, scene_meta, cam_f, cam_i, opt_f, opt_i, workspace, ws_meta, cap):
    return (workspace.new_empty((max(cap, 1), 2), dtype=torch.int32),
            workspace.new_empty((STATS_BYTES,), dtype=torch.uint8))


@custom_op("splatcull::project", mutates_args=())
def project(scene: list[torch.Tensor], scene_meta: list[int], survivors: torch.Tensor, cam_f: list[float],
            cam_i: list[int], opt_f: list[float], opt_i: list[int]) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor,
                                                                            torch.Tensor, torch.Tensor, torch.Tensor]:
    """Stage (c) on explicit survivors -> (splats (n, 32) u8, windows (n, 8) u8, dbg (n, 8) f64
    [mx, my, conic a, b, c, depth, radius, det], rect (n, 4) i32, flags (n,) u8, stats)."""
    lib = nat.load()
    dev = survivors.device
    n = int(survivors.shape[0])
    m = max(n, 1)
    splats = torch.empty((m, nat.SPLAT_BYTES), dtype=torch.uint8, device=dev)
    wins = torch.empty((m, nat.WINDOW_BYTES), dtype=torch.uint8, device=dev)
    dbg = torch.empty((m, 8), dtype=torch.float64, device=dev)
    rect = torch.empty((m, 4), dtype=torch.int32, device=dev)
    flags = torch.empty(m, dtype=torch.uint8, device=dev)
    stats = torch.empty(STATS_BYTES, dtype=torch.uint8, device=dev)
    sc, cam, opts = _scene_struct(scene, scene_meta), _camera_struct(cam_f, cam_i), _opts_struct(opt_f, opt_i)
    nat.check(lib.sc_project(ctypes.byref(sc), nat.ptr(survivors), n, ctypes.byref(cam), ctypes.byref(opts),
                             nat.ptr(splats), nat.ptr(wins), nat.ptr(dbg), nat.ptr(rect), nat.ptr(flags),
                             nat.ptr(stats), _stream(survivors)), "sc_project")
    return splats, wins, dbg, rect, flags, stats


@project.register_fake
def _project_fake(scene, scene_meta, survivors, cam_f, cam_i, opt_f, opt_i):
    m = max(int(survivors.shape[0]), 1)
    e = survivors.new_empty
    return (e((m, nat.SPLAT_BYTES), dtype=torch.uint8), e((m, nat.WINDOW_BYTES), dtype=torch.uint8),
            e((m, 8), dtype=torch.float64), e((m, 4), dtype=torch.int32), e((m,), dtype=torch.uint8),
            e((STATS_BYTES,), dtype=torch.uint8))


@custom_op("splatcull::bin_sort", mutates_args=("workspace",))
def bin_sort(scene: list[torch.Tensor], scene_meta: list[int], survivors: torch.Tensor, cam_f: list[float],
             cam_i: list[int], opt_f: list[float], opt_i: list[int], workspace: torch.Tensor,
             ws_meta: list[int]) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor,
                                          torch.Tensor]:
    """Stages (c)+(d) -> (splats, windows, entry_idx (cap_entries,) i32, tile offsets (n_tiles + 1,)
    i32, order (n,) i32, stats): the reference's argsort + bin_tiles."""
    lib = nat.load()
    dev = survivors.device
    n = int(survivors.shape[0])
    m = max(n, 1)
    cap_e = int(ws_meta[3])
    splats = torch.empty((m, nat.SPLAT_BYTES), dtype=torch.uint8, device=dev)
    wins = torch.empty((m, nat.WINDOW_BYTES), dtype=torch.uint8, device=dev)
    entries = torch.empty(max(cap_e, 1), dtype=torch.int32, device=dev)
    offs = torch.empty(n_tiles(cam_i, int(opt_i[0])) + 1, dtype=torch.int32, device=dev)
    order = torch.empty(m, dtype=torch.int32, device=dev)
    stats = torch.empty(STATS_BYTES, dtype=torch.uint8, device=dev)
    sc, cam, opts, ws = (_scene_struct(scene, scene_meta), _camera_struct(cam_f, cam_i),
                         _opts_struct(opt_f, opt_i), _ws_struct(workspace, ws_meta))
    nat.check(lib.sc_bin_sort(ctypes.byref(sc), nat.ptr(survivors), n, ctypes.byref(cam), ctypes.byref(opts),
                              ctypes.byref(ws), nat.ptr(splats), nat.ptr(wins), nat.ptr(entries), nat.ptr(offs),
                              nat.ptr(order), nat.ptr(stats), _stream(survivors)), "sc_bin_sort")
    return splats, wins, entries, offs, order, stats


@bin_sort.register_fake
def _bin_sort_fake(scene, scene_meta, survivors, cam_f, cam_i, opt_f, opt_i, workspace, ws_meta):
    m = max(int(survivors.shape[0]), 1)
    e = survivors.new_empty
    return (e((m, nat.SPLAT_BYTES), dtype=torch.uint8), e((m, nat.WINDOW_BYTES), dtype=torch.uint8),
            e((max(int(ws_meta[3]), 1),), dtype=torch.int32), e((n_tiles(cam_i, int(opt_i[0])) + 1,), dtype=torch.int32),
            e((m,), dtype=torch.int32), e((STATS_BYTES,), dtype=torch.uint8))


@custom_op("splatcull::blend", mutates_args=())
def blend(splats: torch.Tensor, windows: torch.Tensor, entries: torch.Tensor, tile_offsets: torch.Tensor,
          n_splats: int, cam_f: list[float], cam_i: list[int], opt_f: list[float],
          opt_i: list[int]) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    """Stage (e) on explicit tile lists -> (image, trans, contrib_sum, contrib_max); the last two
    are empty unless record_contributions."""
    lib = nat.load()
    dev = splats.device
    h, w = int(cam_i[1]), int(cam_i[0])
    rec = bool(int(opt_i[2]))
    image = torch.empty((h, w, 3), dtype=torch.float32, device=dev)
    trans = torch.empty((h, w), dtype=torch.float32, device=dev)
    csum = torch.empty((h, w) if rec else (0,), dtype=torch.float32, device=dev)
    cmax = torch.empty((max(n_splats, 1),) if rec else (0,), dtype=torch.float32, device=dev)
    fo = nat.ScFrameOut()
    fo.image, fo.trans = nat.ptr(image), nat.ptr(trans)
    fo.contrib_sum, fo.contrib_max = (nat.ptr(csum), nat.ptr(cmax)) if rec else (0, 0)
    cam, opts = _camera_struct(cam_f, cam_i), _opts_struct(opt_f, opt_i)
    nat.check(lib.sc_blend(nat.ptr(splats), nat.ptr(windows), int(n_splats), nat.ptr(entries) if entries.numel() else 0,
                           nat.ptr(tile_offsets), ctypes.byref(cam), ctypes.byref(opts), ctypes.byref(fo),
                           _stream(splats)), "sc_blend")
    return image, trans, csum, cmax


@blend.register_fake
def _blend_fake(splats, windows, entries, tile_offsets, n_splats, cam_f, cam_i, opt_f, opt_i):
    h, w = int(cam_i[1]), int(cam_i[0])
    rec = bool(int(opt_i[2]))
    e = splats.new_empty
    return (e((h, w, 3), dtype=torch.float32), e((h, w), dtype=torch.float32),
            e((h, w) if rec else (0,), dtype=torch.float32), e((max(n_splats, 1),) if rec else (0,), dtype=torch.float32))


# ---------------------------------------------------------------------------
# MLPs and labels
# ---------------------------------------------------------------------------

@custom_op("splatcull::vis_mlp_forward", mutates_args=())
def vis_mlp_forward(weights: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """Visibility MLP 16->32->32->1 on materialised (n, 16) f32 rows -> (n,) f32 logits
    (weights: one sc_vis_weights record as a uint8 device tensor)."""
    lib = nat.load()
    if x.ndim != 2 or x.shape[1] != 16 or x.dtype != torch.float32 or not x.is_contiguous():
        raise ValueError(f"vis_mlp_forward expects contiguous (n, 16) float32 rows, got {tuple(x.shape)} {x.dtype}")
    out = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    nat.check(lib.sc_vis_mlp_forward(nat.ptr(weights), nat.ptr(x), int(x.shape[0]), nat.ptr(out), _stream(x)),
              "sc_vis_mlp_forward")
    return out


@vis_mlp_forward.register_fake
def _vis_fake(weights, x):
    return x.new_empty((x.shape[0],), dtype=torch.float32)


@custom_op("splatcull::encode_features", mutates_args=())
def encode_features(params: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """Feature MLP 14->32->32->6 on (n, 14) f32 -> (n, 8) fp16 (6 used)."""
    lib = nat.load()
    if x.ndim != 2 or x.shape[1] != 14 or x.dtype != torch.float32 or not x.is_contiguous():
        raise ValueError(f"encode_features expects contiguous (n, 14) float32 rows, got {tuple(x.shape)}")
    out = torch.empty((x.shape[0], 8), dtype=torch.float16, device=x.device)
    nat.check(lib.sc_encode_features(nat.ptr(params), nat.ptr(x), int(x.shape[0]), nat.ptr(out), _stream(x)),
              "sc_encode_features")
    return out


@encode_features.register_fake
def _feat_fake(params, x):
    return x.new_empty((x.shape[0], 8), dtype=torch.float16)


@custom_op("splatcull::visibility_labels_or_", mutates_args=("label_bits",))
def visibility_labels_or_(contrib_max: torch.Tensor, n: int, label_bits: torch.Tensor) -> None:
    """label_bits (int32 words) |= packbits(contrib_max[:n] > 0, little) (sc/sampling.py:206-213)."""
    lib = nat.load()
    nat.check(lib.sc_visibility_labels_or(nat.ptr(contrib_max), int(n), nat.ptr(label_bits), _stream(contrib_max)),
              "sc_visibility_labels_or")


@visibility_labels_or_.register_fake
def _labels_fake(contrib_max, n, label_bits):
    return None
