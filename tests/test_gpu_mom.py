"""NEXT-2: the moment objective eq:LS_SR and its gradient on the device (Fourier domain,
no C_x) against the oracle's spatial float64 form, and Algorithm 1 through srmra_mom_run.

Tolerances: both sides are float64; the device sums O(L^4) terms in a different order (DFTs, aliasing
sums) -> f within 1e-10 relative, gradients within 1e-9 of their max-norm."""
import ctypes

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def srm():
    import paper_2204_04754_b200 as m
    return m


def _theta(rng, L):
    x = rng.standard_normal((L, L))
    return x, rng.dirichlet(np.ones(L)), rng.dirichlet(np.ones(L))


def _cmp(dev, ref, tag):
    f, gx, g1, g2 = dev
    rf, rgx, rg1, rg2, _ = ref
    errs = [abs(f - rf) / abs(rf)] + [np.abs(a - b).max() / np.abs(b).max() for a, b in ((gx, rgx), (g1, rg1), (g2, rg2))]
    print(f"{tag}: f {f:.6e}  rel errors f {errs[0]:.1e} gx {errs[1]:.1e} g1 {errs[2]:.1e} g2 {errs[3]:.1e}")
    assert errs[0] <= 1e-10
    assert max(errs[1:]) <= 1e-9


@pytest.mark.parametrize("L_low,K,N,sigma", [(8, 2, 300, 0.3), (4, 3, 200, 0.5), (5, 2, 77, 0.25), (8, 4, 150, 0.2),
                                             (32, 2, 2000, 0.25)])
def test_objective_and_gradient_match_oracle(srm, oracle_mod, L_low, K, N, sigma):
    p = synth.make_random(L_low, K, N, sigma, seed=L_low * 7 + K)
    M1, M2 = oracle_mod.empirical_moments(p.y)
    rng = np.random.default_rng(L_low + 100 * K)
    L = p.L_high
    with srm.Context(p.y, L, L_low, K, sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
        ctx.mom_set_moments(M1, M2)
        for trial in range(2):
            x, r1, r2 = _theta(rng, L) if trial else (p.x0.astype(np.float64), p.rho1_0, p.rho2_0)
            dev = ctx.mom_objective(x, r1, r2)
            ref = oracle_mod.mom_objective(x, r1, r2, K, sigma, M1, M2)
            _cmp(dev, ref, f"L_low={L_low} K={K} trial {trial}")


def test_zero_at_truth_with_perfect_moments(srm, oracle_mod):
    """The paper's Fig. 2 MoM setting (perfect moments, N -> infinity): f = 0 and grad = 0 at the truth."""
    p = synth.make_random(8, 2, 64, 0.3, seed=5)
    A1, A2 = oracle_mod.analytic_moments(p.x_true, p.rho1_true, p.rho2_true, p.K, p.sigma)
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
        ctx.mom_set_moments(A1, A2)
        f, gx, g1, g2 = ctx.mom_objective(p.x_true, p.rho1_true, p.rho2_true)
        f0 = ctx.mom_objective(p.x0, p.rho1_0, p.rho2_0)[0]
    scale = np.abs(A2).max() ** 2
    assert abs(f) <= 1e-24 * scale * A2.size and f0 > 1e-6 * scale
    assert max(np.abs(gx).max(), np.abs(g1).max(), np.abs(g2).max()) <= 1e-12 * np.abs(A2).max()


def test_device_empirical_moments_feed_the_objective(srm, oracle_mod):
    """srmra_mom_set_moments(NULL, NULL): the tensor-core moments (float32-accurate, test_gpu_moments.py)
    give the oracle's objective within the bound their error implies: |df| <= 2 ||E|| ||d|| + ||d||^2,
    ||d||_F <= 2e-5 max|M2| L_low^2 (+ the lambda term likewise)."""
    p = synth.make_config("c1", N=3000)
    M1, M2 = oracle_mod.empirical_moments(p.y)
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
        ctx.mom_set_moments()
        f, gx, _, _ = ctx.mom_objective(p.x0, p.rho1_0, p.rho2_0)
    rf, rgx = oracle_mod.mom_objective(p.x0, p.rho1_0, p.rho2_0, p.K, p.sigma, M1, M2)[:2]
    d = 2e-5 * np.abs(M2).max() * M2.shape[0]
    bound = 2 * np.sqrt(rf) * d + d * d
    print(f"c1 N=3000: f {f:.6e} oracle {rf:.6e} |df| {abs(f - rf):.2e} bound {bound:.2e}")
    assert abs(f - rf) <= bound


def test_algorithm1_decreases_objective_and_sets_estimate(srm, oracle_mod):
    """Algorithm 1 with perfect moments from a perturbed truth: without projection (F = 0) L-BFGS drives
    the objective down by orders of magnitude; the reported f is the oracle's f at the returned estimate;
    the estimate stays on the simplex; EM iterations can follow."""
    p = synth.make_random(8, 2, 200, 0.3, seed=17)
    A1, A2 = oracle_mod.analytic_moments(p.x_true, p.rho1_true, p.rho2_true, p.K, p.sigma)
    rng = np.random.default_rng(3)
    x0 = (p.x_true + 0.3 * rng.standard_normal(p.x_true.shape)).astype(np.float32)
    r1 = 0.5 * p.rho1_true + 0.5 / p.L_high
    r2 = 0.5 * p.rho2_true + 0.5 / p.L_high
    f_init = oracle_mod.mom_objective(x0, r1, r2, p.K, p.sigma, A1, A2)[0]
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, x0, r1, r2) as ctx:
        ctx.mom_set_moments(A1, A2)
        f, steps = ctx.mom_run(300, F=0, gtol=0.0)
        x, q1, q2, _, _ = ctx.get_estimate()
        fr = oracle_mod.mom_objective(x, q1, q2, p.K, p.sigma, A1, A2)[0]
        print(f"Algorithm 1 (F = 0): f {f_init:.3e} -> {f:.3e} in {steps} steps (oracle at the float32 estimate {fr:.3e})")
        assert steps > 10 and f <= 1e-3 * f_init
        assert abs(fr - f) <= 1e-3 * f_init * 1e-3 + 1e-4 * abs(f)
        assert np.all(q1 >= 0) and abs(q1.sum() - 1) <= 1e-12 and abs(q2.sum() - 1) <= 1e-12
        ctx.em_iter(1)
        assert np.isfinite(ctx.get_estimate()[3])


def test_algorithm1_projection_schedule(srm, oracle_mod):
    """F = 5: the projection D (3x3 box + clamp) runs after every 5th step, so the estimate lies in [-1, 1]
    whenever the run ends on a projection; with a denoiser hook it receives sigma_j = 2^(-(j-1)/10)."""
    p = synth.make_random(8, 2, 200, 0.3, seed=19, image="blobs")
    A1, A2 = oracle_mod.analytic_moments(p.x_true, p.rho1_true, p.rho2_true, p.K, p.sigma)
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
        ctx.mom_set_moments(A1, A2)
        f, steps = ctx.mom_run(20, F=5)
        x = ctx.get_estimate()[0]
        assert steps == 20 and np.isfinite(f)
        assert np.abs(x).max() <= 1.0
        seen = []

        def hook(xdev, L, sig, stream):
            seen.append(sig)
            return 0
        ctx.set_denoiser(hook)
        ctx.mom_run(10, F=5)
        ctx.set_denoiser(None)
    assert len(seen) == 2 and seen[0] == 1.0 and abs(seen[1] - 2 ** -0.1) <= 1e-15


def test_mom_errors(srm, oracle_mod):
    p = synth.make_random(8, 2, 50, 0.3, seed=1)
    lib = srm._lib
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
        with pytest.raises(srm.SrmraError) as e:
            ctx.mom_objective(p.x0, p.rho1_0, p.rho2_0)
        assert e.value.code == srm.SRMRA_ERR_STATE
        with pytest.raises(srm.SrmraError) as e:
            ctx.mom_run(5)
        assert e.value.code == srm.SRMRA_ERR_STATE
        m1 = np.zeros(64)
        rc = lib.srmra_mom_set_moments(ctx.handle, m1.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), None)
        assert rc == srm.SRMRA_ERR_INVALID_ARG
        bad = np.full((64, 64), np.nan)
        with pytest.raises(srm.SrmraError) as e:
            ctx.mom_set_moments(m1, bad)
        assert e.value.code == srm.SRMRA_ERR_INVALID_ARG
        ctx.mom_set_moments()
        with pytest.raises(srm.SrmraError) as e:
            ctx.mom_run(-1)
        assert e.value.code == srm.SRMRA_ERR_INVALID_ARG
    q = synth.make_config("c4", N=4)
    with srm.Context(q.y, q.L_high, q.L_low, q.K, q.sigma, q.x0, q.rho1_0, q.rho2_0) as ctx:
        with pytest.raises(srm.SrmraError) as e:
            ctx.mom_set_moments()
        assert e.value.code == srm.SRMRA_ERR_UNSUPPORTED
