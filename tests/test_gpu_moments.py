"""NEXT-2: the empirical moments of the projected method of moments (eq:empiric_MOM),
computed on the tensor cores through srmra_moments, against the oracle's float64 sums.

Tolerance (written here): the device forms y_i[a] y_i[b] as 3xTF32 products (relative
error <= 2^-21 each) accumulated in float32 in TMEM over chains of at most 4 k-tiles x 4 MMAs x 3 terms
= 48 accumulations (K sliced over the grid, 16 k-tiles per CTA, 4 TMEM split-K blocks), then in float64.
The tensor-core float32 accumulation can be biased (truncation), so the bound is the worst case
48 x 2^-23 ~ 6e-6 of the partial sums of |y_a y_b| (<= max_a M[a, a] by Cauchy-Schwarz) plus the product
error: |err| <= 1e-5 |M| + 1e-5 max|M| (the all-ones column gives M1 with the same arithmetic)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def srm():
    import paper_2204_04754_b200 as m
    return m


def _check(m1, m2, r1, r2, tag):
    s1 = np.abs(r1).max()
    s2 = np.abs(r2).max()
    e1 = np.abs(m1 - r1).max() / s1
    e2 = np.abs(m2 - r2).max() / s2
    print(f"{tag}: max rel-to-max error M1 {e1:.2e}, M2 {e2:.2e}")
    np.testing.assert_allclose(m1, r1, rtol=1e-5, atol=1e-5 * s1)
    np.testing.assert_allclose(m2, r2, rtol=1e-5, atol=1e-5 * s2)
    np.testing.assert_array_equal(m2, m2.T)


@pytest.mark.parametrize("name,N", [("c0", None), ("c1", None), ("c1", 777), ("c3", None), ("c2", 3001)])
def test_moments_match_oracle(srm, oracle_mod, name, N):
    """Several 128-row tiles and a ragged tail in both GEMM dimensions (L_low^2 + 1 rows with the
    all-ones row) and along the observations (N not a multiple of 8 or of the 32-wide K block)."""
    p = synth.make_config(name, N=N)
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
        m1, m2 = ctx.moments()
    r1, r2 = oracle_mod.empirical_moments(p.y)
    _check(m1, m2, r1, r2, f"{name} N={p.y.shape[0]}")


@pytest.mark.parametrize("L_low,K,N", [(3, 2, 1), (5, 3, 37), (7, 2, 513), (12, 3, 4099)])
def test_moments_odd_shapes(srm, oracle_mod, L_low, K, N):
    """Odd L_low (L_low^2 + 1 not 16-aligned), a single observation, N below one K block."""
    p = synth.make_random(L_low, K, N, 0.3, seed=L_low * 100 + N)
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
        m1, m2 = ctx.moments()
        # the moments do not depend on the EM state: unchanged after iterations
        ctx.em_iter(2)
        n1, n2 = ctx.moments()
    r1, r2 = oracle_mod.empirical_moments(p.y)
    _check(m1, m2, r1, r2, f"L_low={L_low} N={N}")
    np.testing.assert_array_equal(m1, n1)
    np.testing.assert_array_equal(m2, n2)


def test_moments_after_reload(srm, oracle_mod):
    """srmra_load replaces the observations: the moments follow the new set."""
    p = synth.make_config("c1", N=2000)
    q = synth.make_config("c1", N=2000, seed_offset=7)
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
        ctx.load(q.y, q.x0, q.rho1_0, q.rho2_0)
        m1, m2 = ctx.moments()
        with pytest.raises(ValueError):
            ctx.load(q.y[:1500], q.x0, q.rho1_0, q.rho2_0)
    r1, r2 = oracle_mod.empirical_moments(q.y)
    _check(m1, m2, r1, r2, "c1 reloaded")


def test_moments_approach_model_moments(srm, oracle_mod):
    """Law of large numbers: at c1's N = 1e4 the empirical moments are within a few
    standard errors of the analytic M1 = P C_x rho, M2 = P C_x D_rho C_x^T P^T + sigma^2 I of the
    generating (x, rho)."""
    p = synth.make_config("c1")
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
        m1, m2 = ctx.moments()
    a1, a2 = oracle_mod.analytic_moments(p.x_true, p.rho1_true, p.rho2_true, p.K, p.sigma)
    Y = p.y.reshape(p.y.shape[0], -1).astype(np.float64)
    N = Y.shape[0]
    # per-entry standard deviations: sd(y_a) <= sqrt(max_a E y_a^2), sd(y_a y_b) <= sqrt(max_a E y_a^4)
    # (Cauchy-Schwarz); 7 sd over the 1024^2 entries of the seeded draw
    sd1 = np.sqrt((Y ** 2).mean(0).max() / N)
    sd2 = np.sqrt((Y ** 4).mean(0).max() / N)
    print(f"c1 LLN: |M1 - E M1| {np.abs(m1 - a1).max() / sd1:.2f} sd, |M2 - E M2| {np.abs(m2 - a2).max() / sd2:.2f} sd")
    assert np.abs(m1 - a1).max() <= 7 * sd1
    assert np.abs(m2 - a2).max() <= 7 * sd2
