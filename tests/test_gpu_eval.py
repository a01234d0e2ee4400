"""NEXT-4: the paper's evaluation metric on the device — error(x_hat) = min_s ||R_s x_hat - x||_F / ||x||_F
 over all L_high^2 shifts — against the oracle's brute force, and at configs[4]'s
size against the closed form of a shifted, perturbed truth; SNR."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def srm():
    import paper_2204_04754_b200 as m
    return m


def test_error_after_em_matches_oracle(srm, oracle_mod):
    p = synth.make_config("c0")
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
        ctx.em_iter(5)
        err, s = ctx.relative_error(p.x_true.astype(np.float32))
        x, *_ = ctx.get_estimate()
    # the device evaluates the float64 state; the float32 estimate differs by < 1e-7 relative
    ref, rs = oracle_mod.relative_error(x, p.x_true.astype(np.float32))
    print(f"c0 after 5 iterations: error {err:.6f} at shift {s} (oracle {ref:.6f} at {rs})")
    assert s == rs and abs(err - ref) <= 1e-6


@pytest.mark.parametrize("name", ["c1", "c4"])
def test_error_of_a_shifted_truth(srm, name):
    """x_hat = R_u x + e loaded as the estimate: the minimiser is s = -u and the error is ||e|| / ||x||
    exactly (evaluated from the float32 values that were loaded)."""
    p = synth.make_config(name, N=8)
    rng = np.random.default_rng(11)
    L = p.L_high
    u = (L // 3, L - 5)
    x = p.x_true.astype(np.float32).astype(np.float64)
    xh = (np.roll(x, u, axis=(0, 1)) + 1e-4 * rng.standard_normal((L, L))).astype(np.float32)
    e = np.roll(xh.astype(np.float64), (-u[0], -u[1]), axis=(0, 1)) - x
    with srm.Context(p.y, L, p.L_low, p.K, p.sigma, xh, p.rho1_0, p.rho2_0) as ctx:
        err, s = ctx.relative_error(x.astype(np.float32))
    assert s == ((-u[0]) % L, (-u[1]) % L)
    np.testing.assert_allclose(err, np.linalg.norm(e) / np.linalg.norm(x), rtol=1e-9)
    assert abs(srm.snr(x, p.sigma) - (x * x).sum() / (L * L * p.sigma ** 2)) <= 1e-12 * srm.snr(x, p.sigma)
