"""Golden PLY fixtures made by running the reference's save_ply / load_ply
(sc/asset.py:218-321) in this container (test infrastructure only):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/gen_golden_ply.py
    -> tests/golden/ply_cases.npz  (NUMBA_CACHE_DIR keeps numba from writing into the read-only reference)
"""
import os
import sys
import tempfile

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")   # never write into /root/reference
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from splatcull.asset import Asset, load_ply, save_ply  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", "ply_cases.npz")


def asset(n, deg, seed):
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return Asset(means=rng.normal(size=(n, 3)).astype(np.float32),
                 log_scales=rng.uniform(-5, 0, (n, 3)).astype(np.float32), rotations=q.astype(np.float32),
                 opacity_logits=rng.normal(0, 2, n).astype(np.float32),
                 sh_coeffs=rng.normal(0, 0.5, (n, (deg + 1) ** 2, 3)).astype(np.float32), sh_degree=deg)


def main():
    out = {}
    with tempfile.TemporaryDirectory() as d:
        for deg in (0, 1, 3):
            a = asset(37, deg, seed=deg)
            p = os.path.join(d, f"a{deg}.ply")
            save_ply(a, p)
            out[f"saved_deg{deg}"] = np.frombuffer(open(p, "rb").read(), np.uint8)
            for k in ("means", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
                out[f"asset_deg{deg}_{k}"] = getattr(a, k)
        # a foreign file: double positions, extra uchar / int properties, unnormalised quaternions,
        # shuffled property order, a trailing face element
        rng = np.random.default_rng(9)
        n = 11
        props = [("rot_2", "f4"), ("x", "f8"), ("y", "f8"), ("z", "f8"), ("red", "u1"), ("f_dc_0", "f4"),
                 ("f_dc_1", "f4"), ("f_dc_2", "f4"), ("opacity", "f4"), ("id", "i4"), ("scale_0", "f4"),
                 ("scale_1", "f4"), ("scale_2", "f4"), ("rot_0", "f4"), ("rot_1", "f4"), ("rot_3", "f4")]
        tname = {"f4": "float", "f8": "double", "u1": "uchar", "i4": "int"}
        rec = np.zeros(n, dtype=[(p, "<" + t) for p, t in props])
        for p, t in props:
            rec[p] = rng.uniform(-2, 2, n).astype(t) if t != "u1" else rng.integers(0, 255, n)
        head = "ply\nformat binary_little_endian 1.0\ncomment foreign\nelement vertex %d\n" % n
        head += "".join(f"property {tname[t]} {p}\n" for p, t in props)
        head += "element face 0\nproperty list uchar int vertex_indices\nend_header\n"
        raw = head.encode() + rec.tobytes()
        p = os.path.join(d, "foreign.ply")
        open(p, "wb").write(raw)
        a = load_ply(p)
        out["foreign_raw"] = np.frombuffer(raw, np.uint8)
        for k in ("means", "log_scales", "rotations", "opacity_logits", "sh_coeffs"):
            out[f"foreign_{k}"] = getattr(a, k)
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
