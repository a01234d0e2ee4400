"""NEXT-4's device data generator srmra_generate against the counter-based reference synth/philox.py:
shifts bit-exact (integer decisions from the same float64 partial sums), y within the float32 error of
the device's Box-Muller (logf / sqrtf / sincospif, a few ulp of sigma |z|) plus one rounding of y; the
EM path then runs on the generated data exactly as on the same data loaded from the host."""
import numpy as np
import pytest

import synth
from synth import philox

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def srm():
    import paper_2204_04754_b200 as m
    return m


def _check(y, sh, yr, shr, sigma):
    np.testing.assert_array_equal(sh, shr)
    err = np.abs(y.astype(np.float64) - yr.astype(np.float64))
    tol = 2e-6 * sigma * 6 + 2.4e-7 * np.abs(yr)
    assert np.all(err <= tol), f"max err {err.max():.3e}"


@pytest.mark.parametrize("name,N,first", [("c0", 500, 0), ("c1", 3001, 12345), ("c3", 2000, 2 ** 33 + 7),
                                          ("c4", 64, 99)])
def test_generate_matches_reference(srm, name, N, first):
    p = synth.make_config(name, N=8)
    seed = 0xDEADBEEF12345 + N
    with srm.Context(None, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, n_local=N) as ctx:
        with pytest.raises(srm.SrmraError) as e:   # no observations yet
            ctx.em_iter(1)
        assert e.value.code == srm.SRMRA_ERR_STATE
        sh = ctx.generate(p.x_true.astype(np.float32), p.rho1_true, p.rho2_true, seed, p.x0, p.rho1_0, p.rho2_0,
                          first_index=first, want_shifts=True)
        y = ctx.observations()
    yr, shr = philox.generate(p.x_true.astype(np.float32), p.rho1_true, p.rho2_true, p.K, p.sigma, N, seed, first)
    _check(y, sh, yr, shr, p.sigma)


def test_generated_data_equals_loaded_data_for_em(srm, oracle_mod):
    """EM on device-generated observations == EM on the reference's observations loaded from the host
    (to the parity tolerance), and the generator's y matches the reference element-wise (read back through
    srmra_get_observations)."""
    p = synth.make_config("c1", N=8)
    N, seed = 4000, 20221019
    yr, shr = philox.generate(p.x_true.astype(np.float32), p.rho1_true, p.rho2_true, p.K, p.sigma, N, seed)
    with srm.Context(None, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, n_local=N) as a, \
            srm.Context(yr, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as b:
        a.generate(p.x_true.astype(np.float32), p.rho1_true, p.rho2_true, seed, p.x0, p.rho1_0, p.rho2_0)
        _check(a.observations(), shr, yr, shr, p.sigma)
        ma, Ma = a.moments()
        mb, Mb = b.moments()
        np.testing.assert_allclose(ma, mb, rtol=1e-6, atol=1e-6 * np.abs(mb).max())
        np.testing.assert_allclose(Ma, Mb, rtol=1e-5, atol=1e-6 * np.abs(Mb).max())
        a.em_iter(3)
        b.em_iter(3)
        xa, r1a, r2a, lla, _ = a.get_estimate()
        xb, r1b, r2b, llb, _ = b.get_estimate()
    assert abs(lla - llb) <= 1e-6 * abs(llb)
    assert np.abs(xa - xb).max() <= 1e-4 * np.abs(xb).max()
    assert np.abs(r1a - r1b).max() <= 1e-4 * r1b.max() and np.abs(r2a - r2b).max() <= 1e-4 * r2b.max()


def test_generate_shards_and_errors(srm):
    """Two ranks' shards (first_index offsets) reproduce the one-rank draw; invalid arguments."""
    p = synth.make_config("c0", N=8)
    seed = 5
    xt = p.x_true.astype(np.float32)
    with srm.Context(None, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, n_local=300) as ctx:
        full = ctx.generate(xt, p.rho1_true, p.rho2_true, seed, p.x0, p.rho1_0, p.rho2_0, want_shifts=True)
        m_full = ctx.moments()[0]
        with pytest.raises(srm.SrmraError) as e:
            ctx.generate(xt, p.rho1_true * 2, p.rho2_true, seed, p.x0, p.rho1_0, p.rho2_0)
        assert e.value.code == srm.SRMRA_ERR_INVALID_ARG
        with pytest.raises(srm.SrmraError) as e:
            ctx.generate(xt, p.rho1_true, p.rho2_true, seed, p.x0, p.rho1_0, p.rho2_0, first_index=-1)
        assert e.value.code == srm.SRMRA_ERR_INVALID_ARG
    parts = []
    for first, n in ((0, 120), (120, 180)):
        with srm.Context(None, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, n_local=n) as ctx:
            parts.append((ctx.generate(xt, p.rho1_true, p.rho2_true, seed, p.x0, p.rho1_0, p.rho2_0,
                                       first_index=first, want_shifts=True), ctx.moments()[0] * n))
    np.testing.assert_array_equal(np.concatenate([a for a, _ in parts]), full)
    np.testing.assert_allclose((parts[0][1] + parts[1][1]) / 300, m_full, rtol=1e-5, atol=1e-6)
