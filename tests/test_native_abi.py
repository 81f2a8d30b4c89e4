"""The C-ABI library loads (no GPU needed), exports every symbol the header
declares, and the ctypes mirrors match the C compiler's struct layouts."""

import ctypes
import os
import re
import subprocess
import tempfile

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "splatcull_b200.h")


def _declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"SC_API\s+[\w\s\*]+?\b(sc_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2511_19202_b200 import _native

    lib = _native.load(require_gpu=False)
    declared = _declared_functions()
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(lib, name), name
        assert name in _native.SIGNATURES, f"{name} has no ctypes signature"
    assert lib.sc_abi_version() == _native.ABI_VERSION == 3


def test_workspace_bytes_is_host_computable():
    from paper_2511_19202_b200 import _native

    lib = _native.load(require_gpu=False)
    small = lib.sc_workspace_bytes(1, 10_000, 10_000, 40_000, 256, 256, 16)
    big = lib.sc_workspace_bytes(1000, 100_000_000, 60_000_000, 180_000_000, 1920, 1080, 16)
    assert 0 < small < big
    # any tile size in [1, 65535] (the reference's tile_size keyword); smaller tiles need more offsets
    assert lib.sc_workspace_bytes(1, 1, 1, 1, 256, 256, 8) > lib.sc_workspace_bytes(1, 1, 1, 1, 256, 256, 32) > 0
    assert lib.sc_workspace_bytes(1, 1, 1, 1, 256, 256, 0) == 0
    assert lib.sc_workspace_bytes(1, 1, 1, 1, 256, 256, 65536) == 0


STRUCTS = ["sc_camera", "sc_opts", "sc_asset_rec", "sc_instance_rec", "sc_vis_weights", "sc_scene",
           "sc_frame_stats", "sc_survivor", "sc_splat", "sc_window", "sc_frame_out", "sc_workspace",
           "sc_frame_debug"]


@pytest.mark.parametrize("name", STRUCTS)
def test_struct_layout_matches_c(name, tmp_path):
    from paper_2511_19202_b200 import _native as nat

    py = {"sc_camera": nat.ScCamera, "sc_opts": nat.ScOpts, "sc_asset_rec": nat.ScAssetRec,
          "sc_instance_rec": nat.ScInstanceRec, "sc_vis_weights": nat.ScVisWeights, "sc_scene": nat.ScScene,
          "sc_frame_stats": nat.ScFrameStats, "sc_survivor": nat.ScSurvivor, "sc_splat": nat.ScSplat, "sc_window": nat.ScWindow,
          "sc_frame_out": nat.ScFrameOut, "sc_workspace": nat.ScWorkspace, "sc_frame_debug": nat.ScFrameDebug}[name]
    lines = [f'printf("%zu\\n", sizeof({name}));']
    for fname, _t in py._fields_:
        lines.append(f'printf("%zu\\n", offsetof({name}, {fname}));')
    prog = ("#include <stdio.h>\n#include <stddef.h>\n#include \"splatcull_b200.h\"\nint main(void){\n"
            + "\n".join(lines) + "\nreturn 0;}\n")
    c = tmp_path / "layout.c"
    c.write_text(prog)
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(c), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got[0] == ctypes.sizeof(py)
    for (fname, _t), off in zip(py._fields_, got[1:]):
        assert getattr(py, fname).offset == off, fname


def test_compute_calls_fail_loudly_without_gpu(monkeypatch):
    import torch

    from paper_2511_19202_b200 import _native

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_native.NativeError):
        _native.load(require_gpu=True)
