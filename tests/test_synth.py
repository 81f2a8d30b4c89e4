"""The workload generators reproduce the reference generators bit for bit."""

import os

import numpy as np

from paper_2511_19202_b200 import synth
from paper_2511_19202_b200.asset import asset_hash, prepare

from conftest import GOLDEN


def test_generator_hashes():
    h = np.load(os.path.join(GOLDEN, "generator_hashes.npz"))
    assert asset_hash(synth.make_shell(1000, seed=0)) == int(h["shell_1000_s0"])
    assert asset_hash(synth.make_shell(100000, seed=0)) == int(h["shell_100000_s0"])
    assert asset_hash(synth.make_slab_pair(500, 400, seed=0)) == int(h["slab_500_400_s0"])
    assert asset_hash(synth.make_random_cloud(777, seed=0)) == int(h["cloud_777_s0"])
    assert asset_hash(synth.make_random_cloud(10000, seed=5)) == int(h["cloud_10000_s5"])
    assert asset_hash(prepare(synth.make_shell(2000, seed=7))) == int(h["prepared_shell_2000_s7"])


def test_fibonacci_kats():
    """SPEC.md:199-200."""
    assert abs(synth.fibonacci_directions(1)[0, 2]) < 1e-15
    np.testing.assert_allclose(synth.fibonacci_directions(2)[:, 2], [0.5, -0.5])


def test_sampling_distance_ratio():
    """d_far / d_near = 18 for p = 0.9 / 0.05."""
    a = prepare(synth.make_shell(500, seed=1))
    assert abs(a.d_far / a.d_near - 18.0) < 1e-12
