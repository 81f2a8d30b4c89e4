"""Generate golden vectors from the REFERENCE implementation (run in the build
container only; /root/reference does not exist on the GPU box).

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python oracle/gen_golden.py [case names]   (no names: every case)

Writes tests/golden/*.npz: the inputs (asset arrays + camera) and the
reference's outputs of project_kernel, the (depth, index) order, bin_tiles
and render() (image, transmittance, contribution records).  tests/
test_oracle_golden.py pins the oracle to these; the GPU parity tests use them
as a second, reference-generated check.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF)
    import splatcull as ref
    from splatcull import raster, synth

    os.makedirs(OUT, exist_ok=True)
    cases = []
    a = ref.prepare(synth.make_random_cloud(3000, seed=1))
    cases.append(("cloud3k_128", a, ref.Camera.look_at([1.5 * a.d_near, 0.4, 0.3], [0, 0, 0], math.radians(50),
                                                        128, 128), dict(record_contributions=True)))
    b = ref.prepare(synth.make_shell(4000, seed=2))
    cases.append(("shell4k_160x96", b, ref.Camera.look_at([0.3, -2.2 * b.d_near, 0.5], [0.1, 0, 0],
                                                           math.radians(40), 160, 96),
                  dict(record_contributions=True)))
    c = ref.prepare(synth.make_slab_pair(1600, 900, seed=3))
    cases.append(("slab_headon_96", c, ref.Camera.look_at([0.0, 0.0, 2.0 * c.d_near], [0, 0, 0],
                                                          math.radians(45), 96, 96, up=[0, 1, 0]),
                  dict(record_contributions=True)))
    d = ref.prepare(synth.make_random_cloud(2500, seed=4, scale_range=(0.005, 0.3)))
    cases.append(("cloud_clip_112x80", d, ref.Camera.look_at([0.2, 1.2 * d.d_near, -0.4], [0, 0, 0],
                                                             math.radians(60), 112, 80),
                  dict(radius_clip=2.0, stop_transmittance=0.02)))
    # higher SH degrees (the synthetic generators emit degree 0): the same assets with seeded
    # degree-3 / degree-2 coefficients, rendered in full and with sh_degree_eval truncation
    import dataclasses
    rng = np.random.default_rng(11)
    e0 = ref.prepare(synth.make_shell(2500, seed=6))
    e = dataclasses.replace(e0, sh_degree=3, sh_coeffs=np.concatenate(
        [e0.sh_coeffs, rng.normal(0.0, 0.25, (len(e0), 15, 3)).astype(np.float32)], axis=1))
    cases.append(("shell_sh3_144x112", e, ref.Camera.look_at([0.6, -1.8 * e.d_near, 0.9], [0, 0, 0],
                                                             math.radians(50), 144, 112),
                  dict(record_contributions=True)))
    f0 = ref.prepare(synth.make_random_cloud(2000, seed=7))
    f = dataclasses.replace(f0, sh_degree=2, sh_coeffs=np.concatenate(
        [f0.sh_coeffs, rng.normal(0.0, 0.3, (len(f0), 8, 3)).astype(np.float32)], axis=1))
    cases.append(("cloud_sh2_eval1_120x90", f, ref.Camera.look_at([-1.4 * f.d_near, 0.5, 0.7], [0, 0, 0],
                                                                  math.radians(55), 120, 90),
                  dict(sh_degree_eval=1)))
    g = ref.prepare(synth.make_random_cloud(1800, seed=8))
    cases.append(("cloud_bg_dil_100x70", g, ref.Camera.look_at([0.9, -1.3 * g.d_near, -0.5], [0, 0, 0],
                                                               math.radians(48), 100, 70),
                  dict(background=(0.1, 0.2, 0.3), dilation=0.5)))
    # tile sizes other than 16 (the image depends on the tile size: the composite window
    # reaches one pixel past the tile rect, sc/_kernels.py:224-227), a non-power-of-two
    # size, and a large dilation with splats straddling the image border
    h = ref.prepare(synth.make_random_cloud(2200, seed=9))
    cases.append(("cloud_ts8_120x88", h, ref.Camera.look_at([1.3 * h.d_near, -0.6, 0.4], [0, 0, 0],
                                                            math.radians(52), 120, 88),
                  dict(tile_size=8, record_contributions=True)))
    k = ref.prepare(synth.make_shell(3000, seed=10))
    cases.append(("shell_ts32_150x100", k, ref.Camera.look_at([0.2, 1.9 * k.d_near, -0.7], [0, 0, 0],
                                                              math.radians(45), 150, 100),
                  dict(tile_size=32)))
    m = ref.prepare(synth.make_random_cloud(2000, seed=12))
    cases.append(("cloud_ts12_100x76", m, ref.Camera.look_at([-0.9, -1.2 * m.d_near, 0.6], [0, 0, 0],
                                                             math.radians(50), 100, 76),
                  dict(tile_size=12, stop_transmittance=0.01)))
    q = ref.prepare(synth.make_random_cloud(2400, seed=13))
    cases.append(("cloud_dil15_border_96x72", q, ref.Camera.look_at([0.7 * q.d_near, 0.3, -0.2], [0, 0, 0],
                                                                    math.radians(40), 96, 72),
                  dict(dilation=1.5)))
    only = set(sys.argv[1:])
    for name, asset, cam, kw in cases:
        if only and name not in only:
            continue
        out = ref.render(asset, cam, **kw)
        proj = raster.project_gaussians(asset, cam, kw.get("dilation", 0.3))
        valid = proj.valid.copy()
        if kw.get("radius_clip"):
            det = proj.cov2d[:, 0] * proj.cov2d[:, 2] - proj.cov2d[:, 1] ** 2
            valid &= ~(det < kw["radius_clip"])
        n = len(asset)
        idx = np.flatnonzero(valid)
        ts = kw.get("tile_size", 16)
        n_tx = (cam.width + ts - 1) // ts
        n_ty = (cam.height + ts - 1) // ts
        tx0 = np.zeros(n, np.int64); tx1 = np.zeros(n, np.int64)
        ty0 = np.zeros(n, np.int64); ty1 = np.zeros(n, np.int64)
        mx, my, r = proj.mean2d[idx, 0], proj.mean2d[idx, 1], proj.radius[idx]
        tx0[idx] = np.clip(np.floor((mx - r) / ts).astype(np.int64), 0, n_tx)
        tx1[idx] = np.clip(np.floor((mx + r) / ts).astype(np.int64) + 1, 0, n_tx)
        ty0[idx] = np.clip(np.floor((my - r) / ts).astype(np.int64), 0, n_ty)
        ty1[idx] = np.clip(np.floor((my + r) / ts).astype(np.int64) + 1, 0, n_ty)
        idx = idx[(tx1[idx] > tx0[idx]) & (ty1[idx] > ty0[idx])]
        order = idx[np.argsort(proj.depth[idx], kind="stable")]
        from splatcull._kernels import bin_tiles
        entry_idx, counts = bin_tiles(order, tx0, tx1, ty0, ty1, n_tx, n_tx * n_ty)
        np.savez_compressed(
            os.path.join(OUT, f"{name}.npz"),
            means=asset.means, log_scales=asset.log_scales, rotations=asset.rotations,
            opacity_logits=asset.opacity_logits, sh_coeffs=asset.sh_coeffs, sh_degree=asset.sh_degree,
            cam_position=cam.position, cam_rotation=cam.rotation, cam_fov_y=cam.fov_y,
            cam_width=cam.width, cam_height=cam.height, cam_near=cam.near,
            opts=np.array(repr(kw)),
            mean2d=proj.mean2d, conic=proj.conic, cov2d=proj.cov2d, depth=proj.depth, radius=proj.radius,
            valid=valid, n_skipped=proj.n_skipped, tx0=tx0, tx1=tx1, ty0=ty0, ty1=ty1, order_idx=order,
            entry_idx=entry_idx, counts=counts,
            image=out.image, final_transmittance=out.final_transmittance,
            contribution_max=(out.contribution_max if out.contribution_max is not None else np.zeros(0)),
            contribution_sum=(out.contribution_sum if out.contribution_sum is not None else np.zeros(0)),
            used_count=-1 if out.used_count is None else out.used_count,
            passed_count=out.passed_count, skipped_count=out.skipped_count,
            asset_hash=np.uint64(ref.asset_hash(asset)))
        print(name, n, "passed", out.passed_count, "entries", entry_idx.size)
    if only:
        return
    # generator hashes (tests/test_synth.py pins the product generators to them)
    gens = {
        "shell_1000_s0": ref.asset_hash(synth.make_shell(1000, seed=0)),
        "shell_100000_s0": ref.asset_hash(synth.make_shell(100000, seed=0)),
        "slab_500_400_s0": ref.asset_hash(synth.make_slab_pair(500, 400, seed=0)),
        "cloud_777_s0": ref.asset_hash(synth.make_random_cloud(777, seed=0)),
        "cloud_10000_s5": ref.asset_hash(synth.make_random_cloud(10000, seed=5)),
        "prepared_shell_2000_s7": ref.asset_hash(ref.prepare(synth.make_shell(2000, seed=7))),
    }
    np.savez(os.path.join(OUT, "generator_hashes.npz"), **{k: np.uint64(v) for k, v in gens.items()})
    print("generator hashes", gens)


if __name__ == "__main__":
    main()
