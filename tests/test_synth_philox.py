"""The counter-based reference generator (synth/philox.py) of the device data generator srmra_generate
(NEXT-4): Philox4x32-10 against its published known-answer vectors, and the draws against the
distributions they must follow (shift pmfs, standard normal noise, the forward model at sigma = 0)."""
import json
import os

import numpy as np

from synth import philox

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.json")


def test_philox_known_answers():
    for v in json.load(open(GOLD))["vectors"]:
        c = [int(w, 16) for w in v["ctr"]]
        k = [int(w, 16) for w in v["key"]]
        out = philox.philox4x32_10(*c, *k)
        assert [int(o) for o in out] == [int(w, 16) for w in v["out"]]


def test_shift_sampler_inverse_cdf():
    """Exact inverse CDF on the partial sums: boundaries, zero-mass entries never drawn, frequencies."""
    rho = np.array([0.25, 0.0, 0.5, 0.25, 0.0])
    C = np.cumsum(rho)
    # words just below / at the partial-sum boundaries
    u = np.array([0, int(0.25 * 2 ** 32) - 1, int(0.25 * 2 ** 32), int(0.75 * 2 ** 32), 2 ** 32 - 1], dtype=np.uint64)
    U = (u.astype(np.float64) + 0.5) * 2.0 ** -32
    s = philox.sample_shift(u, rho)
    for Ui, si in zip(U, s):
        assert rho[si] > 0 and (si == 3 or Ui < C[si]) and (si == 0 or Ui >= C[si - 1])
    x = np.zeros((10, 10), dtype=np.float32)
    r1 = np.random.default_rng(0).dirichlet(np.ones(10))
    r1[3] = 0.0
    r1 /= r1.sum()
    _, sh = philox.generate(x, r1, np.full(10, 0.1), 2, 0.0, 40000, seed=7)
    f = np.bincount(sh[:, 0], minlength=10) / 40000
    assert f[3] == 0.0
    assert np.abs(f - r1).max() <= 5 * np.sqrt(0.25 / 40000)


def test_noise_is_standard_normal_and_model_exact():
    rng = np.random.default_rng(1)
    x = rng.standard_normal((12, 12)).astype(np.float32)
    r = np.full(12, 1 / 12)
    y0, sh = philox.generate(x, r, r, 3, 0.0, 200, seed=11, first_index=5)
    for i in range(200):   # sigma = 0: y_i = P R_{s_i} x exactly
        np.testing.assert_array_equal(y0[i], np.roll(x, tuple(sh[i]), axis=(0, 1))[::3, ::3])
    y, sh2 = philox.generate(x, r, r, 3, 1.0, 5000, seed=11, first_index=5)
    assert np.array_equal(sh2[:200], sh)          # shifts do not depend on sigma
    z = (y - np.stack([np.roll(x, tuple(s), axis=(0, 1))[::3, ::3] for s in sh2])).ravel()
    assert abs(z.mean()) < 5 / np.sqrt(z.size) and abs(z.var() - 1) < 5 * np.sqrt(2 / z.size)
    # counter-based: a sub-range equals the slice of the full range
    ya, _ = philox.generate(x, r, r, 3, 1.0, 100, seed=11, first_index=105)
    np.testing.assert_array_equal(ya, y[100:200])
