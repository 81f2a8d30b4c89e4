"""The scene / visibility-MLP restatement against the SPEC's own known answers
and invariants (acceptance criteria 2 and 7) — CPU only.

These pin oracle/scene_ref.py (the reference package ships no scene/nn code,
so there are no reference golden vectors for these stages) and the host
helpers of the product package that compute the same quantities.
"""

import math

import numpy as np

from oracle import raster_ref as rr
from oracle import scene_ref as sr
from paper_2511_19202_b200 import synth
from paper_2511_19202_b200.asset import Asset, prepare
from paper_2511_19202_b200.camera import Camera, train_focal
from paper_2511_19202_b200.scene import ComposedScene, InstanceTransform, instance_frame, local_inputs
from paper_2511_19202_b200.workloads import calibrated_model, random_unit_quats

from conftest import look_at


def _scene(with_model, n_inst=5, seed=3):
    rng = np.random.default_rng(seed)
    sc = ComposedScene()
    a0 = prepare(synth.make_shell(1500, seed=seed))
    a1 = prepare(synth.make_random_cloud(900, seed=seed + 1))
    sc.add_asset(a0, calibrated_model(a0, seed) if with_model else None)
    sc.add_asset(a1, calibrated_model(a1, seed + 1) if with_model else None)
    q = random_unit_quats(rng, n_inst)
    for k in range(n_inst):
        sc.add_instance(k % 2, InstanceTransform(rng.uniform(-4, 4, 3), q[k], float(rng.uniform(0.5, 2.0))))
    return sc


def test_zero_culling_equivalence_oracle():
    """SPEC.md:359 / acceptance 2: no models -> instanced render == flattened render, 0 bits."""
    sc = _scene(with_model=False)
    cam = look_at([0.0, -14.0, 5.0], [0, 0, 0], 45, 200, 160)
    res = sr.render_composed(sc, cam)
    tabs = sr.SceneTables(sc)
    counts = np.diff(tabs.pair_offset)
    inst = np.repeat(np.arange(len(counts)), counts)
    gid = np.arange(int(tabs.pair_offset[-1])) - np.repeat(tabs.pair_offset[:-1], counts)
    m, ls, q, op, sh, deg = sr.instantiate(tabs, cam, inst, gid)
    flat = rr.render_arrays(m, ls, q, op, sh, deg, cam)
    np.testing.assert_array_equal(res.out.image, flat.image)
    np.testing.assert_array_equal(res.out.final_transmittance, flat.final_transmittance)
    assert res.out.passed_count == flat.passed_count
    assert res.stats["mlp_culled"] == 0


def test_frustum_margin_is_superset_of_passed():
    """B3: every splat the rasterizer passes survives the frustum test (several cameras)."""
    sc = _scene(with_model=False, n_inst=6)
    tabs = sr.SceneTables(sc)
    counts = np.diff(tabs.pair_offset)
    inst = np.repeat(np.arange(len(counts)), counts)
    gid = np.arange(int(tabs.pair_offset[-1])) - np.repeat(tabs.pair_offset[:-1], counts)
    culled_any = False
    for pos, fov in (([0, -14, 5], 45), ([-3, -2, 0.5], 80), ([6, 1, 1], 30)):
        cam = look_at(pos, [0, 0, 0], fov, 160, 120)
        c = sr.cull(tabs, cam, frustum="margin", use_mlp=False)
        m, ls, q, op, sh, deg = sr.instantiate(tabs, cam, inst, gid)
        st = rr.Stages()
        rr.render_arrays(m, ls, q, op, sh, deg, cam, stages=st)
        passed = np.zeros(len(inst), bool)
        if st.passed_idx is not None:
            passed[st.passed_idx] = True
        assert np.all(c.keep[passed] == 1), "frustum culled a splat the rasterizer passes"
        culled_any |= bool(c.keep.sum() < len(inst))
    assert culled_any                          # ... and the test does cull something


def test_eq2_identity_and_scale():
    """f_t = f_r, s = 1 -> d_t = d_r; s = 2 -> d_t = d_r / 2."""
    a = prepare(synth.make_shell(400, seed=1))
    m = calibrated_model(a, 1)
    # camera with focal == f_train: 256x256 with the training fov_y
    from paper_2511_19202_b200.camera import diag_to_fov_y
    fy = diag_to_fov_y(math.radians(60.0), 256, 256)
    cam = Camera.look_at([0, -3.0 * a.d_near, 0.0], [0, 0, 0], fy, 256, 256)
    assert abs(cam.focal - m.f_train) < 1e-9
    for s in (1.0, 2.0):
        tr = InstanceTransform([0, 0, 0], [1, 0, 0, 0], s)
        x = local_inputs(0, a, tr, cam, m)
        mw = np.float32(s) * a.means[0].astype(np.float64)
        d_r = np.linalg.norm(mw - cam.position)
        d_t = d_r / s
        expect = min(1.0, max(-1.0, 2.0 * (d_t - m.d_near) / (m.d_far - m.d_near) - 1.0))
        assert abs(x[6] - expect) < 1e-6


def test_fov_invariance_of_inputs():
    """Acceptance 7a: inputs at (fov A, d) and (fov B, d f_B / f_A) match within 1e-6.

    Exact for a Gaussian at the asset centre (Eq. 2 corrects the camera distance
    of the asset; off-centre means see the usual parallax)."""
    base = prepare(synth.make_shell(300, seed=2))
    m = calibrated_model(base, 2)
    a = Asset(means=np.vstack([np.zeros((1, 3), np.float32), base.means]),
              log_scales=np.vstack([base.log_scales[:1], base.log_scales]),
              rotations=np.vstack([base.rotations[:1], base.rotations]),
              opacity_logits=np.concatenate([base.opacity_logits[:1], base.opacity_logits]),
              sh_coeffs=np.concatenate([base.sh_coeffs[:1], base.sh_coeffs]), sh_degree=0)
    rng = np.random.default_rng(0)
    for _ in range(200):
        direction = rng.normal(size=3)
        direction /= np.linalg.norm(direction)
        d = rng.uniform(1.1, 15.0) * m.d_near
        fa, fb = math.radians(rng.uniform(30, 80)), math.radians(rng.uniform(30, 80))
        ca = Camera.look_at(d * direction, [0, 0, 0], fa, 320, 240)
        ratio = (240 / (2 * math.tan(fb / 2))) / ca.focal
        cb = Camera.look_at(d * ratio * direction, [0, 0, 0], fb, 320, 240)
        tr = InstanceTransform()
        xa = local_inputs(0, a, tr, ca, m, features=np.zeros(6))
        xb = local_inputs(0, a, tr, cb, m, features=np.zeros(6))
        np.testing.assert_allclose(xa, xb, atol=1e-6)


def test_instance_equivariance():
    """instance rotated by R and camera orbited by the same R -> identical 16-vector."""
    a = prepare(synth.make_random_cloud(200, seed=4))
    m = calibrated_model(a, 4)
    rng = np.random.default_rng(1)
    for _ in range(10):
        q = random_unit_quats(rng, 1)[0]
        R = np.array(instance_frame(InstanceTransform([0, 0, 0], q, 1.0))[0]).reshape(3, 3)
        pos = np.array([0.3, -2.5 * m.d_near, 0.7])
        cam0 = Camera.look_at(pos, [0, 0, 0], math.radians(50), 256, 256)
        cam1 = Camera.look_at(R @ pos, [0, 0, 0], math.radians(50), 256, 256, up=R @ np.array([0.0, 0.0, 1.0]))
        g = int(rng.integers(0, len(a)))
        x0 = local_inputs(g, a, InstanceTransform(), cam0, m)
        x1 = local_inputs(g, a, InstanceTransform([0, 0, 0], q, 1.0), cam1, m)
        np.testing.assert_allclose(x0, x1, atol=2e-5)


def test_mlp_forward_kats():
    """zero weights -> logit 0; f64 vs f32 agree within 1e-4 relative."""
    a = prepare(synth.make_shell(100, seed=5))
    m = calibrated_model(a, 5)
    x = np.random.default_rng(0).uniform(-1, 1, (500, 16))
    ref = sr.mlp_forward(m.vis_mlp, x)[:, 0]
    host = m.vis_mlp.forward_host(x)[:, 0]
    np.testing.assert_allclose(ref, host, rtol=1e-9, atol=1e-9)
    zero = type(m.vis_mlp)([w * 0 for w in m.vis_mlp.weights], [b * 0 for b in m.vis_mlp.biases])
    assert np.all(sr.mlp_forward(zero, x) == 0.0)


def test_gate_below_d_near_keeps_all():
    """one identity instance, camera inside d_near -> mlp_culled = 0.

    "Inside" in corrected distance: a camera with the training focal (f_r = f_t)
    at half d_near, so every Gaussian is closer than d_near."""
    from paper_2511_19202_b200.camera import diag_to_fov_y

    a = prepare(synth.make_shell(800, seed=6))
    sc = ComposedScene()
    sc.add_asset(a, calibrated_model(a, 6, keep_target=0.1))
    sc.add_instance(0)
    cam = Camera.look_at([0, -0.5 * a.d_near, 0.1], [0, 0, 0], diag_to_fov_y(math.radians(60), 256, 256), 256, 256)
    c = sr.cull(sr.SceneTables(sc), cam)
    assert np.count_nonzero(c.flags & 2) == 0
    assert np.all(c.keep[(c.flags & 1) > 0] == 1)
