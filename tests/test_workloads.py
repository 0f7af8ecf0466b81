"""Seeded input generators (host data preparation)."""
import json
import os

import numpy as np
import pytest

import fdoracle as O
import reflib as R
from paper_0906_2704_b200 import workloads as W
from util import rel

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_configs_match_baseline_shapes():
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert len(base["configs"]) == 5
    px = [W.config(i).pixels for i in range(5)]
    assert px == [1024, 65536 * 4096, 4096 * 4096, 512 * 1024 * 1024, 16384 * 16384]
    c1 = W.config(1)
    assert c1.count == 256 and (c1.mu_min, c1.mu_max) == (1e-8, 1.0) and c1.noise == 0.005
    assert len(c1.psf) == 29 and np.all(c1.psf[:14] == 0) and abs(c1.psf.sum() - 1) < 1e-15
    assert np.allclose(c1.psf[15:] / c1.psf[14:-1], np.exp(-1 / 5))
    c0 = W.config(0)
    assert len(c0.psf) == 21 and (c0.mu_min, c0.mu_max, c0.count) == (1e-6, 1.0, 64)
    assert len(W.config(2).psf) == 25 and len(W.config(4).psf) == 33
    assert len(W.config(3).psf) == 21 and np.all(W.config(3).psf[:10] == 0)


def test_items_are_independent_of_batching():
    c = W.config(1)
    t_a, g_a = W.signals_1d(c, 0, 8)
    t_b, g_b = W.signals_1d(c, 5, 3)
    assert np.array_equal(g_a[5:8], g_b) and np.array_equal(t_a[5:8], t_b)
    _, g_c = W.signals_1d(W.config(0), 5, 3)
    assert not np.array_equal(g_c[:, :100], g_b[:, :100])


def test_noise_matches_reference_add_noise():
    """operators.cpp:332-358 (SplitMix64 + Box-Muller, ||eta|| = level ||g||)."""
    rng = np.random.default_rng(3)
    for n in (1, 2, 7, 1024, 4097):
        g = rng.uniform(-1, 1, n)
        for seed in (0, 12345, 2 ** 63 + 11):
            a = W.add_noise(g, 0.01, seed)
            b = O.add_noise(g, 0.01, seed)
            assert rel(a, b) < 1e-15
            if R.available():
                assert rel(a, R.add_noise(g, 0.01, seed)) < 1e-15
            assert abs(np.linalg.norm(a - g) / np.linalg.norm(g) - 0.01) < 1e-12


def test_convolve_valid_matches_reference():
    rng = np.random.default_rng(4)
    e = rng.uniform(-1, 1, 300)
    for w in (W.gaussian_weights(10, 3.0), W.onesided_exp_weights(15, 0.2)):
        got = W.convolve_valid(e, w)
        assert rel(got, O.convolve_valid(e, O.make_psf(w))) < 1e-15
        if R.available():
            assert rel(got, R.convolve_valid(e, w)) < 1e-15


def test_2d_scene_is_clipped_and_seeded():
    c = W.config(2)
    t1, g1 = W.image_2d(c, 3, 64, 64)
    t2, g2 = W.image_2d(c, 3, 64, 64)
    assert np.array_equal(g1, g2)
    assert t1.min() >= 0.0 and t1.max() <= 1.0
    assert abs(np.linalg.norm(g1 - W.image_2d(W.Config(**{**c.__dict__, "noise": 0.0}), 3, 64,
                                                64)[1]) / np.linalg.norm(g1) - 0.01) < 1e-3


def test_image_2d_large_matches_serial():
    """Band-parallel generator (config 4 path) = image_2d up to the noise-norm
    summation order."""
    _, g = W.image_2d(W.config(4), 1, 600, 300)
    got = W.image_2d_large(4, 1, workers=3, n1=600, n2=300)
    assert np.max(np.abs(got - g)) < 1e-14 * np.max(np.abs(g))


def test_image_2d_rows_split():
    """Row bands of a split image equal the whole image (the noise norm summed
    over the bands' holders, as the ranks of a row-slab split do)."""
    whole = W.image_2d_large(4, 2, workers=2, n1=768, n2=200)
    parts = [W.image_2d_rows(4, 2, r0, r0 + 256, workers=2, n1=768, n2=200) for r0 in (0, 256, 512)]
    # without a reduction each part normalises alone; with it they match
    sums = []
    import numpy as np
    def collect(s):
        sums.append(s)
        return s
    for r0 in (0, 256, 512):
        W.image_2d_rows(4, 2, r0, r0 + 256, workers=2, n1=768, n2=200, reduce=collect)
    tot = sum(sums)
    got = np.concatenate([W.image_2d_rows(4, 2, r0, r0 + 256, workers=2, n1=768, n2=200,
                                          reduce=lambda s: tot) for r0 in (0, 256, 512)])
    assert np.max(np.abs(got - whole)) < 1e-14 * np.max(np.abs(whole))
    assert parts[0].shape == (256, 200)
