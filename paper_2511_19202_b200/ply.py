"""Standard 3DGS PLY files (binary little-endian) <-> ``Asset``.

Same behaviour as the reference's ``load_ply`` / ``save_ply``
(sc/asset.py:178-321): the vertex element must come first and hold scalar
properties of the usual PLY numeric types; ``x y z f_dc_0..2 opacity
scale_0..2 rot_0..3`` are required; the SH degree follows from the number of
``f_rest_*`` properties, which are channel-major (all higher-order
coefficients of R, then G, then B); quaternions are renormalised only when
some norm is off by more than 1e-6 (valid files survive a load/save cycle bit
for bit); the writer emits float32 properties in the trainer's order with zero
normals.  Malformed input raises ``ValueError`` naming the file.
"""

from __future__ import annotations

import math
import re

import numpy as np

REQUIRED = ("x", "y", "z", "f_dc_0", "f_dc_1", "f_dc_2", "opacity", "scale_0", "scale_1", "scale_2",
            "rot_0", "rot_1", "rot_2", "rot_3")

# PLY scalar type names -> little-endian numpy codes
SCALAR_TYPES = {}
for _names, _code in ((("float", "float32"), "<f4"), (("double", "float64"), "<f8"), (("char", "int8"), "<i1"),
                      (("uchar", "uint8"), "<u1"), (("short", "int16"), "<i2"), (("ushort", "uint16"), "<u2"),
                      (("int", "int32"), "<i4"), (("uint", "uint32"), "<u4")):
    for _n in _names:
        SCALAR_TYPES[_n] = _code

_END = b"end_header\n"


def read_header(raw: bytes, path):
    """-> (vertex count, [(property, numpy code)], byte offset of the body)."""
    stop = raw.find(_END)
    if stop < 0 or not raw.startswith(b"ply"):
        raise ValueError(f"{path}: malformed PLY header")
    text = raw[:stop].decode("ascii", errors="replace")
    m = re.search(r"^format\s+(\S+)", text, re.M)
    if m is None or m.group(1) != "binary_little_endian":
        raise ValueError(f"{path}: expected binary_little_endian PLY")
    count, props, state = None, [], None   # state: None (before), "vertex", "other"
    for line in text.splitlines():
        tok = line.split()
        if not tok:
            continue
        if tok[0] == "element":
            if tok[1] == "vertex":
                if count is not None:
                    raise ValueError(f"{path}: duplicate vertex element")
                count, state = int(tok[2]), "vertex"
            else:
                if count is None:
                    raise ValueError(f"{path}: vertex must be the first element")
                state = "other"
        elif tok[0] == "property" and state == "vertex":
            if tok[1] == "list":
                raise ValueError(f"{path}: list properties are not supported")
            code = SCALAR_TYPES.get(tok[1])
            if code is None:
                raise ValueError(f"{path}: unsupported property type {tok[1]}")
            props.append((tok[2], code))
    if count is None:
        raise ValueError(f"{path}: missing vertex element")
    return count, props, stop + len(_END)


def load_ply(path):
    """Read a 3DGS PLY into an ``Asset`` (no recentering or pruning)."""
    from .asset import Asset

    with open(path, "rb") as fh:
        raw = fh.read()
    count, props, off = read_header(raw, path)
    names = [p for p, _ in props]
    for need in REQUIRED:
        if need not in names:
            raise ValueError(f"{path}: missing property {need}")
    rest = sorted((p for p in names if p.startswith("f_rest_")), key=lambda p: int(p.rsplit("_", 1)[1]))
    if len(rest) % 3:
        raise ValueError(f"{path}: f_rest property count {len(rest)} is not a multiple of 3")
    n_coef = len(rest) // 3 + 1
    deg = int(round(math.sqrt(n_coef))) - 1
    if deg > 3 or (deg + 1) ** 2 != n_coef:
        raise ValueError(f"{path}: f_rest count {len(rest)} does not correspond to a SH degree in 0..3")
    rec = np.dtype([(f"p{k}", code) for k, (_, code) in enumerate(props)])
    need_bytes = count * rec.itemsize
    if len(raw) - off < need_bytes:
        raise ValueError(f"{path}: truncated body, expected {count} vertices")
    table = np.frombuffer(raw, dtype=rec, count=count, offset=off)
    field = {p: table[f"p{k}"] for k, p in enumerate(names)}

    def cols(keys):
        return np.column_stack([np.asarray(field[k], dtype=np.float32) for k in keys]) if count else \
            np.zeros((0, len(keys)), np.float32)

    means = cols(("x", "y", "z"))
    log_scales = cols(("scale_0", "scale_1", "scale_2"))
    quats = cols(("rot_0", "rot_1", "rot_2", "rot_3"))
    opacity = np.asarray(field["opacity"], dtype=np.float32)
    sh = np.zeros((count, n_coef, 3), dtype=np.float32)
    higher = n_coef - 1
    for ch in range(3):
        sh[:, 0, ch] = field[f"f_dc_{ch}"]
        for j in range(higher):
            sh[:, 1 + j, ch] = field[rest[ch * higher + j]]
    for what, arr in (("position", means), ("scale", log_scales), ("rotation", quats), ("opacity", opacity),
                      ("sh", sh)):
        if not np.isfinite(arr).all():
            raise ValueError(f"{path}: non-finite value in {what} fields")
    if count:
        norm = np.linalg.norm(quats.astype(np.float64), axis=1)
        if (norm == 0.0).any():
            raise ValueError(f"{path}: zero-norm rotation quaternion")
        if np.abs(norm - 1.0).max() > 1e-6:
            quats = (quats.astype(np.float64) / norm[:, None]).astype(np.float32)
    return Asset(means=means, log_scales=log_scales, rotations=quats, opacity_logits=opacity, sh_coeffs=sh,
                 sh_degree=deg)


def save_ply(asset, path) -> None:
    """Write ``asset`` as a float32 3DGS PLY (trainer property order, zero normals)."""
    n, higher = len(asset), (asset.sh_degree + 1) ** 2 - 1
    order = (["x", "y", "z", "nx", "ny", "nz", "f_dc_0", "f_dc_1", "f_dc_2"]
             + [f"f_rest_{k}" for k in range(3 * higher)]
             + ["opacity", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3"])
    head = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    head += [f"property float {p}" for p in order]
    head.append("end_header")
    body = np.zeros((n, len(order)), dtype=np.float32)
    body[:, 0:3] = asset.means
    body[:, 6:9] = asset.sh_coeffs[:, 0, :]
    for ch in range(3):   # channel-major higher-order coefficients
        body[:, 9 + ch * higher:9 + (ch + 1) * higher] = asset.sh_coeffs[:, 1:, ch]
    k = 9 + 3 * higher
    body[:, k] = asset.opacity_logits
    body[:, k + 1:k + 4] = asset.log_scales
    body[:, k + 4:k + 8] = asset.rotations
    with open(path, "wb") as fh:
        fh.write(("\n".join(head) + "\n").encode("ascii"))
        fh.write(body.tobytes())
