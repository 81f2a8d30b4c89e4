"""ctypes binding of ``libsplatcull_b200.so`` (include/splatcull_b200.h).

This is the only place the package touches the native library.  There is no
fallback: if the library is missing or no CUDA device is present, every
compute entry point raises.  Device buffers are torch CUDA tensors (torch is
the allocator and stream provider, nothing more); their raw pointers are
passed through the plain C ABI.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsplatcull_b200.so")
if os.environ.get("SPLATCULL_B200_DEBUG_LIB"):       # instrumented build (scripts/blend_stats.py only)
    LIB_PATH = os.path.join(_HERE, "libsplatcull_b200_dbg.so")
if os.environ.get("SPLATCULL_B200_VARIANT"):         # A/B builds of kernel variants (scripts/ab_variants.py only)
    LIB_PATH = os.path.abspath(os.environ["SPLATCULL_B200_VARIANT"])

SC_OK = 0
ABI_VERSION = 3   # include/splatcull_b200.h SC_ABI_VERSION
SC_FRUSTUM_MARGIN, SC_FRUSTUM_STRICT, SC_FRUSTUM_OFF = 0, 1, 2

c_f64, c_i32, c_i64, c_f32, c_u32, c_u16 = (ctypes.c_double, ctypes.c_int32, ctypes.c_int64,
                                            ctypes.c_float, ctypes.c_uint32, ctypes.c_uint16)
P = ctypes.c_void_p


class ScCamera(ctypes.Structure):
    _fields_ = [("pos", c_f64 * 3), ("rot", c_f64 * 9), ("focal", c_f64), ("tan_x", c_f64),
                ("tan_y", c_f64), ("near_", c_f64), ("width", c_i32), ("height", c_i32)]


class ScOpts(ctypes.Structure):
    _fields_ = [("tile_size", c_i32), ("sh_degree_eval", c_i32), ("record_contributions", c_i32),
                ("use_mlp", c_i32), ("frustum_mode", c_i32), ("exact_projection", c_i32),
                ("radius_clip", c_f64), ("stop_transmittance", c_f64), ("background", c_f64 * 3),
                ("dilation", c_f64), ("frustum_G", c_f64), ("band_y0", c_i32), ("band_y1", c_i32)]


class ScAssetRec(ctypes.Structure):
    _fields_ = [("offset", c_i64), ("count", c_i64), ("d_near", c_f64), ("d_far", c_f64),
                ("inv_mean_scale", c_f64), ("f_train", c_f64), ("bound_local", c_f64),
                ("sigma_max", c_f64), ("model", c_i32), ("sh_degree", c_i32),
                ("logit_threshold", c_f32), ("reserved0", c_i32)]


class ScInstanceRec(ctypes.Structure):
    _fields_ = [("R", c_f64 * 9), ("t", c_f64 * 3), ("q", c_f64 * 4), ("s", c_f64), ("ln_s", c_f64),
                ("asset", c_i32), ("reserved0", c_i32)]


class ScVisWeights(ctypes.Structure):
    _fields_ = [("w1", c_u16 * (32 * 16)), ("w2", c_u16 * (32 * 32)), ("b1", c_f32 * 32),
                ("b2", c_f32 * 32), ("w3", c_f32 * 32), ("b3", c_f32), ("reserved", c_f32 * 31)]


class ScScene(ctypes.Structure):
    _fields_ = [("mean_opa", P), ("quat", P), ("scale_smax", P), ("sh", P), ("features", P),
                ("n_gauss", c_i64), ("sh_stride", c_i32), ("n_assets", c_i32), ("assets", P),
                ("instances", P), ("n_instances", c_i64), ("vis_weights", P), ("n_models", c_i32),
                ("reserved0", c_i32), ("n_pairs", c_i64), ("appear", P)]


STATS_FIELDS = ("instances_visible", "pairs_tested", "frustum_passed", "mlp_queried", "mlp_culled",
                "survivors", "passed", "skipped", "entries", "used", "max_tie_run", "overflow", "block_entries",
                "exact_fallbacks")


class ScFrameStats(ctypes.Structure):
    _fields_ = [(n, c_i64) for n in STATS_FIELDS] + [("reserved", c_i64 * 2)]


class ScSurvivor(ctypes.Structure):
    _fields_ = [("inst", c_u32), ("gid", c_u32)]


class ScSplat(ctypes.Structure):
    _fields_ = [("mx", c_f32), ("my", c_f32), ("half_a", c_f32), ("b", c_f32), ("half_c", c_f32),
                ("p_min", c_f32), ("rgb", c_u16 * 3), ("reserved", c_u16)]


class ScWindow(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_int16), ("x1", ctypes.c_int16), ("y0", ctypes.c_int16), ("y1", ctypes.c_int16)]


class ScFrameDebug(ctypes.Structure):
    _fields_ = [("order", P), ("block_offsets", P), ("block_entries", P), ("block_codes", P)]


class ScFrameOut(ctypes.Structure):
    _fields_ = [("image", P), ("trans", P), ("contrib_sum", P), ("contrib_max", P), ("stats", P),
                ("survivors", P), ("stage_events", P), ("n_stage_events", c_i32), ("reserved0", c_i32),
                ("debug", P)]


N_STAGE_EVENTS = 5
STAGE_NAMES = ("cull_mlp", "project", "sort_bin", "blend")


class ScWorkspace(ctypes.Structure):
    _fields_ = [("base", P), ("bytes", ctypes.c_size_t), ("n_instances", c_i64), ("max_pairs", c_i64),
                ("cap_survivors", c_i64), ("cap_entries", c_i64)]


STATS_BYTES = ctypes.sizeof(ScFrameStats)
SPLAT_BYTES = ctypes.sizeof(ScSplat)
WINDOW_BYTES = ctypes.sizeof(ScWindow)
assert SPLAT_BYTES == 32 and WINDOW_BYTES == 8, (SPLAT_BYTES, WINDOW_BYTES)

# exported symbol -> (restype, argtypes); mirrors include/splatcull_b200.h
SIGNATURES = {
    "sc_abi_version": (c_i32, []),
    "sc_last_error": (ctypes.c_char_p, []),
    "sc_kernel_launches": (c_i64, []),
    "sc_workspace_bytes": (ctypes.c_size_t, [c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32]),
    "sc_render_composed": (c_i32, [P, P, P, P, P, P]),
    "sc_render_survivors": (c_i32, [P, P, c_i64, P, P, P, P, P]),
    "sc_cull_mlp": (c_i32, [P, P, P, P, P, c_i64, P, P]),
    "sc_project": (c_i32, [P, P, c_i64, P, P, P, P, P, P, P, P, P]),
    "sc_bin_sort": (c_i32, [P, P, c_i64, P, P, P, P, P, P, P, P, P, P]),
    "sc_blend": (c_i32, [P, P, c_i64, P, P, P, P, P, P]),
    "sc_vis_mlp_forward": (c_i32, [P, P, c_i64, P, P]),
    "sc_encode_features": (c_i32, [P, P, c_i64, P, P]),
    "sc_visibility_labels_or": (c_i32, [P, c_i64, P, P]),
}

_lib = None


class NativeError(RuntimeError):
    pass


def load(require_gpu: bool = True):
    """Load the library (raises if it was not built, or if no GPU when required)."""
    global _lib
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise NativeError("paper_2511_19202_b200 needs a CUDA device (sm_100a); none is visible")
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (or make -C paper_2511_19202_b200/csrc)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.sc_abi_version() != ABI_VERSION:
            raise NativeError("libsplatcull_b200.so ABI version mismatch")
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != SC_OK:
        msg = _lib.sc_last_error().decode(errors="replace") if _lib is not None else ""
        if rc == 1:
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what} failed (code {rc}): {msg}")


def stream_handle(stream=None) -> int:
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def ptr(t) -> int:
    return int(t.data_ptr()) if t is not None else 0


def struct_tensor(obj, device):
    """Copy a ctypes structure / array to a device uint8 tensor."""
    import torch
    buf = np.frombuffer(bytes(obj), dtype=np.uint8).copy()
    return torch.from_numpy(buf).to(device)


def camera_struct(cam) -> ScCamera:
    c = ScCamera()
    c.pos[:] = [float(v) for v in np.asarray(cam.position, dtype=np.float64).reshape(3)]
    c.rot[:] = [float(v) for v in np.asarray(cam.rotation, dtype=np.float64).reshape(9)]
    c.focal = float(cam.focal)
    tx, ty = cam.tan_half_fov
    c.tan_x, c.tan_y = float(tx), float(ty)
    c.near_ = float(cam.near)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def stats_dict(raw: np.ndarray) -> dict:
    vals = np.frombuffer(raw.tobytes(), dtype=np.int64)
    return {n: int(vals[i]) for i, n in enumerate(STATS_FIELDS)}
