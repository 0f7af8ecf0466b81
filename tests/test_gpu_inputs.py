"""GPU input generation: convolve_valid / convolve_valid_2d
(pipeline.cpp:14-51) and add_noise (operators.cpp:332-358) on the device vs the
numpy restatements in workloads.py (pinned to the compiled reference at 1e-15
by tests/test_workloads.py) and, when it is built, the reference itself."""
import numpy as np
import pytest
import torch

import paper_0906_2704_b200 as P
from paper_0906_2704_b200 import workloads as W
from util import np_, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,taps", [(1, 1), (17, 5), (1024, 21), (4096, 29)])
def test_convolve_valid_1d(n, taps, rng):
    w = rng.random(taps)
    w /= w.sum()
    ext = rng.standard_normal((5, n + taps - 1))
    got = np_(P.convolve_valid(torch.from_numpy(ext).cuda(), w))
    assert got.shape == (5, n)
    assert rel(got, W.convolve_valid(ext, w)) < 1e-14


def test_convolve_valid_2d(rng):
    w = rng.random((7, 5))
    w /= w.sum()
    ext = rng.standard_normal((3, 40 + 6, 33 + 4))
    got = np_(P.convolve_valid_2d(torch.from_numpy(ext).cuda(), w))
    want = np.zeros((3, 40, 33))
    for j in range(7):
        for l in range(5):
            want += w[j, l] * ext[:, j:j + 40, l:l + 33]
    assert rel(got, want) < 1e-14


def test_convolve_valid_2d_against_reference(rng):
    import reflib as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    w = np.outer(W.gaussian_weights(3, 1.2), W.gaussian_weights(2, 0.9))
    ext = rng.standard_normal((24 + 6, 31 + 4))
    got = np_(P.convolve_valid_2d(torch.from_numpy(ext).cuda(), w))
    w = w / w.sum()
    got = np_(P.convolve_valid_2d(torch.from_numpy(ext).cuda(), w))
    assert rel(got, R.convolve_valid_2d(ext, w)) < 1e-13


@pytest.mark.parametrize("n", [1, 2, 7, 1024, 4097])
def test_add_noise_1d(n, rng):
    g = rng.standard_normal((6, n)) + 2.0
    seeds = W.item_key(1, np.arange(6))
    want = W.add_noise(g, 0.01, seeds)
    got = np_(P.add_noise(torch.from_numpy(g).cuda(), 0.01, seeds))
    assert rel(got, want) < 1e-13
    assert rel(got - g, want - g) < 1e-10  # the noise itself


def test_add_noise_2d_flat_and_edge_cases(rng):
    g = rng.random((2, 50, 37))
    seeds = np.array([123456789, 2 ** 63 + 5], dtype=np.uint64)
    want = np.stack([W.add_noise(g[i].reshape(-1), 0.05, seeds[i]).reshape(50, 37)
                     for i in range(2)])
    got = np_(P.add_noise(torch.from_numpy(g).cuda(), 0.05, seeds, item_dims=2))
    assert rel(got - g, want - g) < 1e-10
    same = np_(P.add_noise(torch.from_numpy(g).cuda(), 0.0, seeds, item_dims=2))
    assert np.array_equal(same, g)
    with pytest.raises(P.ValidationError):
        P.add_noise(torch.from_numpy(g).cuda(), -1.0, seeds, item_dims=2)


def test_device_generated_observation_matches_host_pipeline():
    """A config-2-like observation built entirely on the device (scene upload,
    blur, noise) equals workloads.image_2d's host pipeline, and restores to the
    same result."""
    cfg = W.config(2)
    n = 256
    m = (len(cfg.psf) - 1) // 2
    truth, g_host = W.image_2d(cfg, 3, n, n)
    key, ext = W._scene_2d(cfg, 3, n, n, m, m)
    gd = P.convolve_valid_2d(torch.from_numpy(ext).cuda(), cfg.psf2d())
    P.add_noise(gd, cfg.noise, key, item_dims=2)
    assert rel(np_(gd), g_host) < 1e-12
