"""Visibility-MLP training and checkpoints (SPEC.md nn module).

CPU: schedule endpoints, gradient check, checkpoint round trip / truncation,
convergence on all-visible labels and on the labels the REFERENCE extracted
(tests/golden/sampling_labels.npz).  GPU: extract -> train -> render with the
trained model culling, image close to the unculled render.
"""

import os
import tempfile

import numpy as np
import pytest

from conftest import ROOT
from test_sampling import _asset, _dataset_with

from paper_2511_19202_b200 import nn, sampling, synth, training
from paper_2511_19202_b200.asset import prepare

GOLD = os.path.join(ROOT, "tests", "golden")


def test_lr_schedule_endpoints():
    cfg = training.TrainConfig(iterations=1000)
    assert training.lr_at(200, cfg) == pytest.approx(cfg.lr_init, rel=1e-12)
    assert training.lr_at(1000, cfg) == pytest.approx(cfg.lr_final, rel=1e-12)
    warm = [training.lr_at(t, cfg) for t in range(1, 201)]
    decay = [training.lr_at(t, cfg) for t in range(200, 1001)]
    assert 0.0 < warm[0] < 1e-5 and all(a < b for a, b in zip(warm, warm[1:]))
    assert all(a > b for a, b in zip(decay, decay[1:]))


def test_config_validation():
    for bad in (dict(lr_final=3e-3), dict(warmup_frac=0.0), dict(batch_size=0), dict(iterations=0)):
        with pytest.raises(ValueError):
            training.TrainConfig(**bad)


def test_grad_check():
    a = _asset()
    model = nn.make_model(a, seed=5, output_bias=0.3)
    rng = np.random.default_rng(0)
    geo = rng.normal(size=(6, 10))
    fin = nn.feature_inputs(a, model.mean_scale)[:6]
    y = np.array([1, 0, 1, 1, 0, 1], dtype=np.float64)
    assert training.grad_check(model, geo, fin, y) < 1e-4


def test_checkpoint_roundtrip_and_errors():
    a = _asset()
    model = nn.make_model(a, seed=2, f_train=221.7, threshold=0.4)
    model.meta["final_loss"] = 0.125
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "m.scvm")
        nn.save_model(model, path)
        raw = open(path, "rb").read()
        assert len(raw) < 32 * 1024
        back = nn.load_model(path)
        for m0, m1 in ((model.feature_mlp, back.feature_mlp), (model.vis_mlp, back.vis_mlp)):
            assert m0.widths == m1.widths
            for x, y in zip(m0.weights + m0.biases, m1.weights + m1.biases):
                np.testing.assert_array_equal(x, y)
        assert (back.mean_scale, back.d_near, back.d_far, back.f_train, back.threshold, back.asset_hash) == \
            (model.mean_scale, model.d_near, model.d_far, model.f_train, model.threshold, model.asset_hash)
        assert back.meta == {"final_loss": 0.125}
        model.asset_hash = None
        nn.save_model(model, path)
        assert nn.load_model(path).asset_hash is None
        for cut in (0, 10, 60, 200, len(raw) - 1):
            with open(path, "wb") as fh:
                fh.write(raw[:cut])
            with pytest.raises(ValueError):
                nn.load_model(path)
        with open(path, "wb") as fh:
            fh.write(b"XXXX" + raw[4:])
        with pytest.raises(ValueError, match="magic"):
            nn.load_model(path)


def test_all_visible_labels_learned():
    a = _asset()
    ones = _dataset_with(np.full((12, 250), 255, np.uint8))
    model = training.train(ones, a, training.TrainConfig(iterations=200, batch_size=1024), device="cpu")
    ev = training.evaluate(model, ones, a, device="cpu")
    assert ev["keep_rate"] == 1.0 and ev["recall"] == 1.0


def test_learns_reference_labels():
    """Labels extracted by the reference (12 views of a 2000-splat shell): the
    trained model keeps nearly every visible splat and culls most hidden ones."""
    z = np.load(os.path.join(GOLD, "sampling_labels.npz"))
    ds, a = _dataset_with(z["labels_packed"]), _asset()
    model = training.train(ds, a, training.TrainConfig(iterations=600, batch_size=4096), device="cpu")
    ev = training.evaluate(model, ds, a, device="cpu")
    assert ev["recall"] > 0.98 and ev["accuracy"] > 0.93, ev
    assert np.isfinite(model.meta["final_loss"]) and model.meta["iterations"] == 600


def test_train_rejects_mismatched_inputs():
    z = np.load(os.path.join(GOLD, "sampling_labels.npz"))
    ds = _dataset_with(z["labels_packed"])
    other = prepare(synth.make_shell(2000, seed=9))
    with pytest.raises(ValueError):
        training.train(ds, other, training.TrainConfig(iterations=1), device="cpu")


@pytest.mark.gpu
def test_trained_model_culls_without_visible_loss():
    """Extract labels on the GPU, train on the GPU, then render a composed scene
    with the trained model in the cull stage: a large share of splats is culled
    by the MLP while the image stays close to the unculled render."""
    import torch

    from paper_2511_19202_b200 import Camera
    from paper_2511_19202_b200.raster import psnr
    from paper_2511_19202_b200.scene import ComposedScene, InstanceTransform, RenderOptions, render_composed

    a = prepare(synth.make_shell(20000, seed=11))
    cfg = sampling.SamplingConfig(n_directions=96, n_distances=4, n_aux_views=2, image_size=128, seed=1)
    ds = sampling.extract_dataset(a, cfg)
    model = training.train(ds, a, training.TrainConfig(iterations=1500, batch_size=1 << 14, seed=3))
    held = sampling.extract_dataset(a, sampling.SamplingConfig(n_directions=16, n_distances=3, n_aux_views=2,
                                                               image_size=128, seed=7))
    ev = training.evaluate(model, held, a)
    assert ev["recall"] > 0.97 and ev["keep_rate"] < ev["visible_rate"] + 0.15, ev

    scene = ComposedScene()
    scene.add_asset(a, model)
    for k in range(4):
        scene.add_instance(0, InstanceTransform(translation=np.array([3.0 * a.bound_radius * k, 0.0, 0.0])))
    eye = np.array([4.5 * a.bound_radius, -2.0 * a.bound_radius, 6.0 * a.bound_radius])
    cam = Camera.look_at(eye, np.array([4.5 * a.bound_radius, 0.0, 0.0]), fov_y=np.radians(50.0), width=640,
                         height=480)
    on, st = render_composed(scene, cam, RenderOptions(use_mlp=True))
    off, _ = render_composed(scene, cam, RenderOptions(use_mlp=False))
    culled = st.mlp_culled / max(1, st.mlp_queried)
    assert culled > 0.2, st
    assert psnr(on.image, off.image) > 30.0
    torch.cuda.synchronize()
