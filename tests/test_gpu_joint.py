"""NEXT-3: the joint (non-separable) shift prior — eq:rho_EM as written — on the GEMM
and direct paths against the oracle's joint iteration, element by element (tolerances of
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
         ("c1", 400, 0)]


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
    iters = 1 if name == "c1" else 3
    x, rho = p.x0.astype(np.float64), pr
    trace = []
    for _ in range(iters):
        r = oracle_mod.em_iter_joint(p.y, p.L_low, p.K, p.sigma, x, rho, project=True)
        trace.append(r.loglik)
        x, rho = r.x, r.rho
    for path in ("gemm", "direct"):
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


def test_joint_prior_rejected_on_fft_path_and_reset_by_load(srm):
    p = synth.make_config("c0")
    L = p.L_high
    with srm.Context(p.y, L, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path="fft") as ctx:
        with pytest.raises(srm.SrmraError) as ei:
            ctx.set_joint_rho(joint_prior(L, 1))
        assert ei.value.code == srm.SRMRA_ERR_UNSUPPORTED
    with srm.Context(p.y, L, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path="gemm") as ctx:
        ctx.set_joint_rho(joint_prior(L, 1))
        ctx.load(p.y, p.x0, p.rho1_0, p.rho2_0)
        with pytest.raises(srm.SrmraError) as ei:
            ctx.joint_rho()
        assert ei.value.code == srm.SRMRA_ERR_STATE


def test_product_joint_prior_equals_separable(srm):
    """rho = rho1 rho2^T through the joint machinery gives the separable iteration (GPU vs GPU) — for one
    iteration: the joint update of the next prior is no longer a product."""
    p = synth.make_config("c0")
    L = p.L_high
    outs = []
    for joint in (False, True):
        with srm.Context(p.y, L, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path="gemm") as ctx:
            if joint:
                ctx.set_joint_rho(np.outer(p.rho1_0, p.rho2_0))
            ctx.em_iter(1)
            outs.append(ctx.get_estimate())
    (xa, a1, a2, lla, _), (xb, b1, b2, llb, _) = outs
    np.testing.assert_allclose(xb, xa, atol=1e-5 * np.abs(xa).max())
    np.testing.assert_allclose(b1, a1, atol=1e-6)
    assert abs(llb - lla) <= 1e-7 * abs(lla)
