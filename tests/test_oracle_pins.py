"""Pins of the float64 oracle against things other than itself (CPU only).

Each test constructs its expectation independently of oracle/srmra_oracle.c:
dense P / R_s matrices written from the definitions, closed forms, the
paper's invariances, EM monotonicity, the sigma -> 0 limit,
textbook K = 1 MRA EM, and hand-enumerated index examples (tests/golden/).
"""
import json
import os

import numpy as np
import pytest

import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------- independent helpers
def R_matrix(L, s):
    """Dense 2-D circular translation, (R_s x)[n] = x[n - s] (PAPER.md:28 'R_s denotes a 2-D
    circular translation'), acting on row-major vec(x)."""
    M = np.zeros((L * L, L * L))
    for n1 in range(L):
        for n2 in range(L):
            M[n1 * L + n2, ((n1 - s[0]) % L) * L + (n2 - s[1]) % L] = 1.0
    return M


def P_matrix(L, K):
    """Dense down-sampling, (P x)[n] = x[n K] (PAPER.md:29 'collects L_low x L_low equally-spaced
    samples')."""
    Ll = L // K
    M = np.zeros((Ll * Ll, L * L))
    for n1 in range(Ll):
        for n2 in range(Ll):
            M[n1 * Ll + n2, (n1 * K) * L + n2 * K] = 1.0
    return M


def dense_em(y, K, sigma, x, rho1, rho2, prior=None):
    """EM iteration in the paper's matrix form (eq:likelihood_EM, eq:weights_EM, eq:x_EM with
    P^{-1} := P^T, eq:rho_EM marginals), dense and brute force.  `prior` [L][L]: a joint shift prior
    rho[s] in place of rho1[s1] rho2[s2] (NEXT-3)."""
    N, Ll, _ = y.shape
    L = Ll * K
    P = P_matrix(L, K)
    Rs = {(a, b): R_matrix(L, (a, b)) for a in range(L) for b in range(L)}
    xv = x.reshape(-1)
    A = np.zeros((L * L, L * L))
    bvec = np.zeros(L * L)
    colsum = np.zeros((L, L))
    LL = 0.0
    W = np.zeros((N, L, L))
    for i in range(N):
        yi = y[i].reshape(-1).astype(np.float64)
        ell = np.full((L, L), -np.inf)
        for (a, b), R in Rs.items():
            r = yi - P @ R @ xv
            with np.errstate(divide="ignore"):
                lp = np.log(prior[a, b]) if prior is not None else np.log(rho1[a]) + np.log(rho2[b])
                ell[a, b] = lp - r @ r / (2 * sigma ** 2)
        m = ell.max()
        lse = m + np.log(np.exp(ell - m).sum())
        LL += lse
        w = np.exp(ell - lse)
        W[i] = w
        colsum += w
        for (a, b), R in Rs.items():
            A += w[a, b] * R.T @ P.T @ P @ R
            bvec += w[a, b] * R.T @ P.T @ yi
    return dict(A=A, b=bvec, colsum=colsum, LL=LL, W=W,
                rho1=colsum.sum(1) / colsum.sum(), rho2=colsum.sum(0) / colsum.sum())


def box_clamp_dense(x):
    L = x.shape[0]
    out = np.zeros_like(x)
    for d1 in (-1, 0, 1):
        for d2 in (-1, 0, 1):
            out += np.roll(x, (-d1, -d2), axis=(0, 1))
    return np.clip(out / 9.0, -1.0, 1.0)


def tiny(L_low=2, K=2, N=5, sigma=0.7, seed=0, zeros=0):
    return synth.make_random(L_low, K, N, sigma, seed, rho_zeros=zeros)


# ----------------------------------------------------------------------- golden index examples
def test_golden_index_convention():
    g = json.load(open(os.path.join(GOLDEN, "index_convention.json")))
    for ex in g["shift_examples"] + g["downsample_examples"]:
        x = np.array(ex["x"], dtype=np.float64)
        K = ex["K"]
        y = synth.observe(x, np.array([ex["s"]]), K, 0.0, None)[0]
        np.testing.assert_array_equal(y, np.array(ex["out"], dtype=np.float32))
        # the dense operators used by the brute-force pin agree with the same examples
        L = x.shape[0]
        yd = (P_matrix(L, K) @ R_matrix(L, ex["s"]) @ x.reshape(-1)).reshape(L // K, L // K)
        np.testing.assert_array_equal(yd, np.array(ex["out"], dtype=np.float64))


# ----------------------------------------------------------------------- (1) brute force
@pytest.mark.parametrize("seed,zeros", [(0, 0), (1, 0), (2, 1)])
def test_bruteforce_dense_4x4(oracle_mod, seed, zeros):
    p = tiny(seed=seed, zeros=zeros)
    x = p.x0.astype(np.float64)
    d = dense_em(p.y, p.K, p.sigma, x, p.rho1_0, p.rho2_0)
    r = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0, project=False, tau=0.0)
    # A from the matrix form is diagonal (consequence of P^{-1} := P^T)
    A = d["A"]
    assert np.abs(A - np.diag(np.diag(A))).max() == 0.0
    np.testing.assert_allclose(r.A.reshape(-1), np.diag(A), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(r.b.reshape(-1), d["b"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(r.colsum, d["colsum"], rtol=1e-12, atol=1e-14)
    assert abs(r.loglik - d["LL"]) <= 1e-12 * abs(d["LL"])
    np.testing.assert_allclose(r.rho1, d["rho1"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(r.rho2, d["rho2"], rtol=1e-12, atol=1e-15)
    xs = np.linalg.solve(A, d["b"]).reshape(x.shape)       # A x = b (eq:x_EM)
    np.testing.assert_allclose(r.x, xs, rtol=1e-11, atol=1e-12)
    # per-observation posterior (eq:weights_EM)
    for i in range(p.N):
        w, lse = oracle_mod.posterior(p.y[i], p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0)
        np.testing.assert_allclose(w, d["W"][i], rtol=1e-11, atol=1e-15)
    # projection of the same iterate
    rp = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0, project=True, tau=0.0)
    np.testing.assert_allclose(rp.x, box_clamp_dense(xs), rtol=1e-11, atol=1e-12)


def test_bruteforce_dense_8x8_K4(oracle_mod):
    p = synth.make_random(2, 4, 3, 0.5, 5)
    x = p.x0.astype(np.float64)
    d = dense_em(p.y, p.K, p.sigma, x, p.rho1_0, p.rho2_0)
    r = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0, project=False, tau=0.0)
    np.testing.assert_allclose(r.A.reshape(-1), np.diag(d["A"]), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(r.b.reshape(-1), d["b"], rtol=1e-12, atol=1e-13)
    assert abs(r.loglik - d["LL"]) <= 1e-12 * abs(d["LL"])


# ----------------------------------------------------------------------- (2) normalisation
def test_posteriors_sum_to_one(oracle_mod):
    p = synth.make_random(4, 2, 40, 0.3, 3, rho_zeros=2)
    x = p.x0.astype(np.float64)
    for i in range(0, p.N, 7):
        w, _ = oracle_mod.posterior(p.y[i], p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0)
        assert abs(w.sum() - 1.0) < 1e-12
        assert np.all(np.isfinite(w)) and np.all(w >= 0)
    r = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0, project=False)
    assert abs(r.colsum.sum() - p.N) < 1e-10 * p.N
    assert abs(r.rho1.sum() - 1) < 1e-13 and abs(r.rho2.sum() - 1) < 1e-13
    # zero prior mass stays zero (log 0 = -inf contributes weight 0, never NaN)
    assert np.all(r.rho1[p.rho1_0 == 0] == 0) and np.all(r.rho2[p.rho2_0 == 0] == 0)
    # mass conservation (independent of x): sum_p b[p] = sum_{i,n} y_i[n]; sum_p A = N L_low^2
    assert abs(r.b.sum() - p.y.astype(np.float64).sum()) < 1e-9 * np.abs(p.y).sum()
    assert abs(r.A.sum() - p.N * p.L_low ** 2) < 1e-9 * p.N * p.L_low ** 2


# ----------------------------------------------------------------------- (3) EM monotone
def test_loglik_monotone_without_projection(oracle_mod):
    p = synth.make_random(4, 2, 60, 0.4, 11)
    _, _, _, trace = oracle_mod.run(p.y, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0,
                                    iters=20, proj_every=0)
    for a, b in zip(trace[:-1], trace[1:]):
        assert b >= a - 1e-9 * abs(a), (a, b)
    assert trace[-1] > trace[0]


# ----------------------------------------------------------------------- (4) sigma -> 0 recovery
def test_exact_recovery_sigma_to_zero(oracle_mod):
    L_low, K, N = 4, 2, 60
    L = L_low * K
    rng = np.random.default_rng(5)
    x_true = rng.standard_normal((L, L)).astype(np.float32).astype(np.float64)
    rho1 = rng.dirichlet(np.ones(L)); rho2 = rng.dirichlet(np.ones(L))
    shifts = np.stack([rng.choice(L, N, p=rho1), rng.choice(L, N, p=rho2)], 1)
    y = synth.observe(x_true, shifts, K, 0.0, None)        # noiseless
    sigma = 1e-3
    r = oracle_mod.em_iter(y, L_low, K, sigma, x_true, rho1, rho2, project=False)
    # posterior collapses on the true shift
    for i in range(0, N, 9):
        w, _ = oracle_mod.posterior(y[i], L_low, K, sigma, x_true, rho1, rho2)
        assert np.unravel_index(np.argmax(w), w.shape) == tuple(shifts[i])
        assert w.max() > 1 - 1e-12
    np.testing.assert_allclose(r.x, x_true, rtol=0, atol=1e-12)
    h1 = np.bincount(shifts[:, 0], minlength=L) / N
    h2 = np.bincount(shifts[:, 1], minlength=L) / N
    np.testing.assert_allclose(r.rho1, h1, atol=1e-12)
    np.testing.assert_allclose(r.rho2, h2, atol=1e-12)


# ----------------------------------------------------------------------- closed forms / limits
def test_constant_image_closed_form(oracle_mod):
    p = synth.make_random(4, 2, 30, 0.5, 7)
    c = 0.3
    x = np.full((p.L_high, p.L_high), c)
    r = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0, project=False)
    yy = p.y.astype(np.float64)
    ll = -(((yy - c) ** 2).sum(axis=(1, 2))) / (2 * p.sigma ** 2)
    np.testing.assert_allclose(r.ll_obs, ll, rtol=1e-12)
    w, _ = oracle_mod.posterior(p.y[0], p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0)
    np.testing.assert_allclose(w, np.outer(p.rho1_0, p.rho2_0), rtol=1e-11)
    # posterior = prior for every i  =>  rho' = rho (up to rounding)
    np.testing.assert_allclose(r.rho1, p.rho1_0, rtol=1e-11)


def test_large_sigma_posterior_is_prior(oracle_mod):
    p = synth.make_random(4, 2, 4, 0.5, 8)
    x = p.x0.astype(np.float64)
    w, _ = oracle_mod.posterior(p.y[1], p.L_low, p.K, 1e6, x, p.rho1_0, p.rho2_0)
    assert np.abs(w - np.outer(p.rho1_0, p.rho2_0)).max() < 1e-6


def test_point_mass_rho_stays_point_mass(oracle_mod):
    p = synth.make_random(4, 2, 20, 0.5, 9)
    L = p.L_high
    r1 = np.zeros(L); r1[3] = 1.0
    r2 = np.zeros(L); r2[5] = 1.0
    r = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, p.x0, r1, r2, project=False)
    np.testing.assert_array_equal(r.rho1, r1)
    np.testing.assert_array_equal(r.rho2, r2)


# ----------------------------------------------------------------------- invariances
def test_global_shift_invariance(oracle_mod):
    p = synth.make_random(4, 2, 25, 0.4, 12)
    x = p.x0.astype(np.float64)
    base = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0, project=False)
    u = (3, 6)
    xu = np.roll(x, u, axis=(0, 1))                       # R_u x
    r1u = np.roll(p.rho1_0, -u[0]); r2u = np.roll(p.rho2_0, -u[1])   # rho'(k) = rho(k + u)
    sh = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, xu, r1u, r2u, project=False)
    assert abs(sh.loglik - base.loglik) <= 1e-11 * abs(base.loglik)


def test_theorem1_separable_invariance(oracle_mod):
    """permuting sub-images and shifting each one on the low-res grid leaves
    the likelihood unchanged.  Separable version (per-axis class permutation pi_k and per-class
    shift tau_k) so that the product prior stays a product."""
    rng = np.random.default_rng(21)
    L_low, K = 4, 2
    L = L_low * K
    p = synth.make_random(L_low, K, 30, 0.4, 13)
    x = p.x0.astype(np.float64)
    base = oracle_mod.em_iter(p.y, L_low, K, p.sigma, x, p.rho1_0, p.rho2_0, project=False)
    for _ in range(5):
        pi = [rng.permutation(K), rng.permutation(K)]
        tau = [rng.integers(0, L_low, K), rng.integers(0, L_low, K)]
        xn = np.zeros_like(x)
        for r1 in range(K):
            for r2 in range(K):
                # x_r[m] = x[(K m - r) mod L];  x'_{pi(r)}[m] = x_r[m - tau(r)]
                for m1 in range(L_low):
                    for m2 in range(L_low):
                        src = x[(K * ((m1 - tau[0][r1]) % L_low) - r1) % L,
                                (K * ((m2 - tau[1][r2]) % L_low) - r2) % L]
                        xn[(K * m1 - pi[0][r1]) % L, (K * m2 - pi[1][r2]) % L] = src
        rn = []
        for k, rho in enumerate((p.rho1_0, p.rho2_0)):
            out = np.zeros(L)
            for r in range(K):
                for t in range(L_low):
                    out[pi[k][r] + K * ((t - tau[k][r]) % L_low)] = rho[r + K * t]
            rn.append(out)
        got = oracle_mod.em_iter(p.y, L_low, K, p.sigma, xn, rn[0], rn[1], project=False)
        assert abs(got.loglik - base.loglik) <= 1e-11 * abs(base.loglik)


def test_observation_permutation_invariance(oracle_mod):
    p = synth.make_random(4, 2, 33, 0.4, 14)
    x = p.x0.astype(np.float64)
    a = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0)
    perm = np.random.default_rng(0).permutation(p.N)
    b = oracle_mod.em_iter(p.y[perm], p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0)
    np.testing.assert_allclose(b.x, a.x, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(b.rho1, a.rho1, rtol=1e-12, atol=1e-15)
    assert abs(a.loglik - b.loglik) <= 1e-12 * abs(a.loglik)
    np.testing.assert_allclose(b.ll_obs, a.ll_obs[perm], rtol=1e-13)


# ----------------------------------------------------------------------- M-step = argmax Q
def test_mstep_maximises_Q(oracle_mod):
    p = synth.make_random(4, 2, 20, 0.5, 15)
    x = p.x0.astype(np.float64)
    L, K = p.L_high, p.K
    r = oracle_mod.em_iter(p.y, p.L_low, K, p.sigma, x, p.rho1_0, p.rho2_0, project=False)
    W = np.stack([oracle_mod.posterior(p.y[i], p.L_low, K, p.sigma, x, p.rho1_0, p.rho2_0)[0]
                  for i in range(p.N)])
    P = P_matrix(L, K)
    Rs = [[R_matrix(L, (a, b)) for b in range(L)] for a in range(L)]

    def Q(xc, r1, r2):   # eq:Q
        tot = 0.0
        for i in range(p.N):
            yi = p.y[i].reshape(-1).astype(np.float64)
            for a in range(L):
                for b in range(L):
                    w = W[i, a, b]
                    if w == 0:
                        continue
                    res = yi - P @ Rs[a][b] @ xc.reshape(-1)
                    tot += w * (np.log(r1[a]) + np.log(r2[b]) - res @ res / (2 * p.sigma ** 2))
        return tot

    q0 = Q(r.x, r.rho1, r.rho2)
    rng = np.random.default_rng(1)
    for _ in range(6):
        d = 1e-3 * rng.standard_normal(r.x.shape)
        assert Q(r.x + d, r.rho1, r.rho2) < q0
        e1 = rng.dirichlet(np.ones(L)); e2 = rng.dirichlet(np.ones(L))
        assert Q(r.x, 0.9 * r.rho1 + 0.1 * e1, 0.9 * r.rho2 + 0.1 * e2) < q0
    assert q0 >= Q(x, p.rho1_0, p.rho2_0)     # ascent from theta_t


# ----------------------------------------------------------------------- K = 1: textbook MRA EM
def test_K1_reduces_to_textbook_mra(oracle_mod):
    L, N, sigma = 6, 15, 0.6
    rng = np.random.default_rng(3)
    x = rng.standard_normal((L, L))
    r1 = rng.dirichlet(np.ones(L)); r2 = rng.dirichlet(np.ones(L))
    y = (rng.standard_normal((N, L, L))).astype(np.float32)
    yy = y.astype(np.float64)
    xn = np.zeros((L, L)); LL = 0.0; cs = np.zeros((L, L))
    for i in range(N):
        ell = np.zeros((L, L))
        for a in range(L):
            for b in range(L):
                ell[a, b] = (np.log(r1[a]) + np.log(r2[b])
                             - ((yy[i] - np.roll(x, (a, b), axis=(0, 1))) ** 2).sum() / (2 * sigma ** 2))
        m = ell.max(); lse = m + np.log(np.exp(ell - m).sum()); LL += lse
        w = np.exp(ell - lse); cs += w
        for a in range(L):
            for b in range(L):
                xn += w[a, b] * np.roll(yy[i], (-a, -b), axis=(0, 1))   # R_{-s} y_i
    xn /= N
    r = oracle_mod.em_iter(y, L, 1, sigma, x, r1, r2, project=False)
    np.testing.assert_allclose(r.x, xn, rtol=1e-11, atol=1e-13)
    assert abs(r.loglik - LL) <= 1e-12 * abs(LL)
    np.testing.assert_allclose(r.rho1, cs.sum(1) / N, rtol=1e-11)


# ----------------------------------------------------------------------- projection
def test_projection_stand_in(oracle_mod):
    L = 8
    np.testing.assert_allclose(oracle_mod.project(np.full((L, L), 0.25)), 0.25, rtol=1e-15)
    np.testing.assert_array_equal(oracle_mod.project(np.full((L, L), 2.0)), 1.0)
    np.testing.assert_array_equal(oracle_mod.project(np.full((L, L), -3.0)), -1.0)
    imp = np.zeros((L, L)); imp[0, 0] = 0.9
    out = oracle_mod.project(imp)
    exp = np.zeros((L, L))
    for d1 in (-1, 0, 1):
        for d2 in (-1, 0, 1):
            exp[d1 % L, d2 % L] = 0.1
    np.testing.assert_allclose(out, exp, atol=1e-16)
    z = np.random.default_rng(0).standard_normal((L, L))
    np.testing.assert_allclose(oracle_mod.project(z), box_clamp_dense(z), atol=1e-15)


def test_unobserved_class_keeps_previous_value(oracle_mod):
    """Reading R6: A[p] <= tau keeps x_t[p].  rho concentrated on even shifts leaves odd classes
    of pixels unobserved (pixel p is sampled under s iff s = -p mod K)."""
    p = synth.make_random(4, 2, 10, 0.5, 16)
    L = p.L_high
    r1 = np.zeros(L); r1[::2] = 1.0; r1 /= r1.sum()
    r2 = np.zeros(L); r2[::2] = 1.0; r2 /= r2.sum()
    x = p.x0.astype(np.float64)
    r = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, x, r1, r2, project=False)
    odd = np.ones((L, L), bool); odd[::2, ::2] = False
    assert np.all(r.A[odd] == 0)
    np.testing.assert_array_equal(r.x[odd], x[odd])
    assert np.all(r.A[::2, ::2] > 0)


# ---------------------------------------------------------------- NEXT-1: Algorithm 2 driver
def test_sigma_schedule_closed_form(oracle_mod):
    """eq:decaying_function: sigma_1 = 1, sigma_j = 2^(-1/10) sigma_{j-1}, i.e. the
    closed form 2^(-(j-1)/10); sigma halves every 10 projections."""
    for j in range(1, 40):
        assert abs(oracle_mod.sigma_schedule(j) - 2.0 ** (-(j - 1) / 10.0)) <= 1e-14
    assert abs(oracle_mod.sigma_schedule(11) - 0.5) <= 1e-14


def test_alg2_stopping_rule_and_identity_denoiser(oracle_mod):
    import synth
    p = synth.make_random(4, 2, 23, 0.5, 5)
    args = (p.y, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0)
    # a huge tolerance stops after the first checkable iteration (t = 1): two LL values recorded
    *_, tr, _ = oracle_mod.run_alg2(*args, 10, proj_every=1, rel_tol=1e30)
    assert len(tr) == 2
    # no tolerance: max_iters iterations, identical to run()
    x, r1, r2, tr, sig = oracle_mod.run_alg2(*args, 5, proj_every=2)
    xr, rr1, rr2, trr = oracle_mod.run(*args, 5, proj_every=2)
    np.testing.assert_array_equal(x, xr)
    np.testing.assert_array_equal(tr, trr)
    assert len(sig) == 2
    # the identity denoiser makes Algorithm 2 plain EM (PAPER.md:226-268 without the projection step)
    xi, *_, tri, sigi = oracle_mod.run_alg2(*args, 5, proj_every=2, denoiser=lambda v, s: v)
    x0, *_, tr0 = oracle_mod.run(*args, 5, proj_every=0)
    np.testing.assert_array_equal(xi, x0)
    np.testing.assert_array_equal(tri, tr0)
    assert sigi == [1.0, 2.0 ** -0.1]
    # the stopping point: the first t >= 1 with |LL_t - LL_{t-1}| <= tol |LL_t|
    *_, full, _ = oracle_mod.run_alg2(*args, 12, proj_every=0)
    d = [abs(full[t] - full[t - 1]) / abs(full[t]) for t in range(1, len(full))]
    tol = sorted(d)[len(d) // 2]
    t_star = 1 + next(k for k, v in enumerate(d) if v <= tol)
    *_, trs, _ = oracle_mod.run_alg2(*args, 12, proj_every=0, rel_tol=tol)
    assert len(trs) == t_star + 1


# ---------------------------------------------------------------- NEXT-4: evaluation
def test_relative_error_closed_forms(oracle_mod):
    """error(x_hat) = min_s ||R_s x_hat - x||_F / ||x||_F: zero for any circular shift
    of x, attained at the inverse shift; 1 for x_hat = 0 and for x_hat = 2x (Cauchy-Schwarz:
    <R_s x, x> <= ||x||^2, so ||R_s 2x - x||^2 = 5||x||^2 - 4<R_s x, x> >= ||x||^2, equality at s = 0)."""
    rng = np.random.default_rng(3)
    L = 12
    x = rng.standard_normal((L, L))
    for u in [(0, 0), (3, 5), (11, 1)]:
        err, s = oracle_mod.relative_error(np.roll(x, u, axis=(0, 1)), x)
        assert err <= 1e-14 and s == ((-u[0]) % L, (-u[1]) % L)
    assert abs(oracle_mod.relative_error(np.zeros((L, L)), x)[0] - 1.0) <= 1e-14
    err, s = oracle_mod.relative_error(2 * x, x)
    assert abs(err - 1.0) <= 1e-13 and s == (0, 0)
    # a perturbed shift: the distance is exactly the perturbation's norm while it stays the minimiser
    e = 1e-3 * rng.standard_normal((L, L))
    err, s = oracle_mod.relative_error(np.roll(x, (4, 7), axis=(0, 1)) + e, x)
    assert s == (L - 4, L - 7) and abs(err - np.linalg.norm(e) / np.linalg.norm(x)) <= 1e-12


# ---------------------------------------------------------------- NEXT-3: joint (non-separable) prior
def _joint_prior(L, seed, zeros=0):
    rng = np.random.default_rng(seed)
    pr = rng.uniform(0.05, 1.0, (L, L)) ** 3          # far from a product of marginals
    if zeros:
        idx = rng.choice(L * L, size=zeros, replace=False)
        pr.reshape(-1)[idx] = 0.0
    return pr / pr.sum()


@pytest.mark.parametrize("seed,zeros", [(0, 0), (1, 3)])
def test_joint_bruteforce_dense_4x4(oracle_mod, seed, zeros):
    """eq:rho_EM as written: rho'[s] = sum_i w^{i,s} / sum_i sum_s' w^{i,s'}, with the
    joint prior in eq:weights_EM, against the dense matrix form."""
    p = tiny(seed=seed)
    L = p.L_high
    x = p.x0.astype(np.float64)
    pr = _joint_prior(L, seed, zeros)
    d = dense_em(p.y, p.K, p.sigma, x, None, None, prior=pr)
    r = oracle_mod.em_iter_joint(p.y, p.L_low, p.K, p.sigma, x, pr, project=False, tau=0.0)
    assert abs(r.loglik - d["LL"]) <= 1e-12 * abs(d["LL"])
    np.testing.assert_allclose(r.colsum, d["colsum"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(r.rho, d["colsum"] / d["colsum"].sum(), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(r.rho1, r.rho.sum(1), rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(r.b.reshape(-1), d["b"], rtol=1e-12, atol=1e-13)
    xs = np.linalg.solve(d["A"], d["b"]).reshape(x.shape)
    np.testing.assert_allclose(r.x, xs, rtol=1e-11, atol=1e-12)
    assert np.all(r.rho.reshape(-1)[pr.reshape(-1) == 0] == 0.0)   # zero prior mass stays zero


def test_joint_with_product_prior_is_the_separable_iteration(oracle_mod):
    """With rho = rho1 rho2^T the joint iteration is the separable one, and the marginals of the joint
    update are the separable update (the latter is the marginal form of eq:rho_EM, reading R2)."""
    p = synth.make_random(4, 2, 31, 0.45, 4, rho_zeros=1)
    x = p.x0.astype(np.float64)
    sep = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0, project=True)
    jnt = oracle_mod.em_iter_joint(p.y, p.L_low, p.K, p.sigma, x, np.outer(p.rho1_0, p.rho2_0), project=True)
    assert abs(jnt.loglik - sep.loglik) <= 1e-12 * abs(sep.loglik)
    np.testing.assert_allclose(jnt.x, sep.x, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(jnt.rho1, sep.rho1, rtol=1e-12, atol=1e-16)
    np.testing.assert_allclose(jnt.rho2, sep.rho2, rtol=1e-12, atol=1e-16)


def test_joint_em_monotone(oracle_mod):
    """EM ascent with the joint prior update, projection off."""
    p = synth.make_random(4, 2, 40, 0.4, 6)
    x = p.x0.astype(np.float64)
    rho = _joint_prior(p.L_high, 9, zeros=2)
    lls = []
    for _ in range(15):
        r = oracle_mod.em_iter_joint(p.y, p.L_low, p.K, p.sigma, x, rho, project=False)
        lls.append(r.loglik)
        x, rho = r.x, r.rho
    assert np.all(np.diff(lls) >= -1e-9 * np.abs(lls[:-1])), lls


# ---------------------------------------------------------------- NEXT-2: moments
def test_empirical_moments_closed_forms(oracle_mod):
    rng = np.random.default_rng(5)
    y = rng.standard_normal((37, 4, 4)).astype(np.float32)
    M1, M2 = oracle_mod.empirical_moments(y)
    Y = y.reshape(37, -1).astype(np.float64)
    np.testing.assert_allclose(M1, Y.mean(0), rtol=1e-14)
    np.testing.assert_allclose(M2, M2.T, rtol=0, atol=0)                       # symmetric
    assert np.linalg.eigvalsh(M2 - np.outer(M1, M1)).min() >= -1e-12           # covariance is PSD
    assert abs(np.trace(M2) - (Y * Y).sum(1).mean()) <= 1e-12 * np.trace(M2)   # trace = mean ||y||^2
    one = np.repeat(y[:1], 5, axis=0)                                           # identical observations
    m1, m2 = oracle_mod.empirical_moments(one)
    np.testing.assert_allclose(m2, np.outer(m1, m1), rtol=1e-14)


def test_analytic_moments_definition_and_invariances(oracle_mod):
    """M1 = P C_x rho from the BCCB columns (dense construction of PAPER.md:201-212), M2 symmetric PSD +
    sigma^2 I; a point-mass prior gives M2 = v v^T + sigma^2 I with v = P R_s x."""
    L, K, sigma = 8, 2, 0.3
    rng = np.random.default_rng(2)
    x = rng.standard_normal((L, L))
    r1 = rng.dirichlet(np.ones(L)); r2 = rng.dirichlet(np.ones(L))
    M1, M2 = oracle_mod.analytic_moments(x, r1, r2, K, sigma)
    C = np.stack([R_matrix(L, (a, b)) @ x.reshape(-1) for a in range(L) for b in range(L)], axis=1)  # C_x
    P = P_matrix(L, K)
    rho = np.outer(r1, r2).reshape(-1)
    np.testing.assert_allclose(M1, P @ C @ rho, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(M2, P @ C @ np.diag(rho) @ C.T @ P.T + sigma ** 2 * P @ P.T, rtol=1e-12, atol=1e-13)
    e1 = np.zeros(L); e1[3] = 1.0
    e2 = np.zeros(L); e2[5] = 1.0
    m1, m2 = oracle_mod.analytic_moments(x, e1, e2, K, sigma)
    v = np.roll(x, (3, 5), axis=(0, 1))[::K, ::K].reshape(-1)
    np.testing.assert_allclose(m2, np.outer(v, v) + sigma ** 2 * np.eye(v.size), rtol=1e-13)
    np.testing.assert_allclose(m1, v, rtol=1e-13)


def test_moments_law_of_large_numbers(oracle_mod):
    """eq:moments_convergence: the empirical moments of data drawn from the model with
    known (x, rho, sigma) approach the analytic ones at the 1/sqrt(N) rate."""
    errs = []
    for N in (400, 6400):
        p = synth.make_random(4, 2, N, 0.5, 21)
        M1, M2 = oracle_mod.empirical_moments(p.y)
        A1, A2 = oracle_mod.analytic_moments(p.x_true, p.rho1_true, p.rho2_true, p.K, p.sigma)
        errs.append(np.abs(M2 - A2).max())
        assert np.abs(M1 - A1).max() <= 6.0 / np.sqrt(N)
    assert errs[1] < errs[0] / 2.0   # 16x the observations: ~4x smaller


# ---------------------------------------------------------------- NEXT-2: the moment objective eq:LS_SR
@pytest.mark.parametrize("L,K", [(8, 2), (6, 3)])
def test_mom_gradient_matches_finite_differences(oracle_mod, L, K):
    """The oracle's gradient of eq:LS_SR (derived, not printed in the paper) against central differences of
    its objective in every coordinate of x, rho1, rho2 (the objective is a polynomial: h = 1e-5 leaves
    O(h^2) truncation)."""
    rng = np.random.default_rng(L * 10 + K)
    Ll, sigma, h = L // K, 0.4, 1e-5
    x = rng.standard_normal((L, L))
    r1, r2 = rng.dirichlet(np.ones(L)), rng.dirichlet(np.ones(L))
    Y = rng.standard_normal((40, Ll * Ll))
    M1, M2 = Y.mean(0), Y.T @ Y / 40
    f, gx, g1, g2, _ = oracle_mod.mom_objective(x, r1, r2, K, sigma, M1, M2)

    def fd(fun, a):
        out = np.zeros_like(a)
        for idx in np.ndindex(a.shape):
            ap, am = a.copy(), a.copy()
            ap[idx] += h
            am[idx] -= h
            out[idx] = (fun(ap) - fun(am)) / (2 * h)
        return out
    nx = fd(lambda a: oracle_mod.mom_objective(a, r1, r2, K, sigma, M1, M2)[0], x)
    n1 = fd(lambda a: oracle_mod.mom_objective(x, a, r2, K, sigma, M1, M2)[0], r1)
    n2 = fd(lambda a: oracle_mod.mom_objective(x, r1, a, K, sigma, M1, M2)[0], r2)
    for g, n in ((gx, nx), (g1, n1), (g2, n2)):
        np.testing.assert_allclose(g, n, rtol=1e-6, atol=1e-6 * np.abs(n).max())


def test_mom_objective_definition_zero_and_invariance(oracle_mod):
    """f is the squared distance of PAPER.md:215-218 with lambda = 1/(L^2(1+sigma^2)): it
    equals the dense-matrix value, vanishes with zero gradient at the truth given the perfect moments
    (N -> infinity, as in the paper's Fig. 2 experiment), and is invariant under x -> R_u x,
    rho -> R_{-u} rho (the translation symmetry of the model)."""
    L, K, sigma = 8, 2, 0.25
    rng = np.random.default_rng(9)
    x = rng.standard_normal((L, L))
    r1, r2 = rng.dirichlet(np.ones(L)), rng.dirichlet(np.ones(L))
    assert oracle_mod.mom_lambda(64, 0.5) == 1.0 / (64 * 64 * 1.25)
    A1, A2 = oracle_mod.analytic_moments(x, r1, r2, K, sigma)
    f, gx, g1, g2, grho = oracle_mod.mom_objective(x, r1, r2, K, sigma, A1, A2)
    assert abs(f) <= 1e-24 and np.abs(gx).max() <= 1e-12 and np.abs(grho).max() <= 1e-12
    Y = rng.standard_normal((30, 16))
    M1, M2 = Y.mean(0), Y.T @ Y / 30
    C = np.stack([R_matrix(L, (a, b)) @ x.reshape(-1) for a in range(L) for b in range(L)], axis=1)
    P = P_matrix(L, K)
    rho = np.outer(r1, r2).reshape(-1)
    dense = (np.linalg.norm(P @ C @ np.diag(rho) @ C.T @ P.T + sigma ** 2 * P @ P.T - M2) ** 2
             + np.linalg.norm(P @ C @ rho - M1) ** 2 / (L * L * (1 + sigma ** 2)))
    f = oracle_mod.mom_objective(x, r1, r2, K, sigma, M1, M2)[0]
    np.testing.assert_allclose(f, dense, rtol=1e-12)
    u = (3, 5)
    fs = oracle_mod.mom_objective(np.roll(x, u, axis=(0, 1)), np.roll(r1, -u[0]), np.roll(r2, -u[1]), K, sigma,
                                  M1, M2)[0]
    np.testing.assert_allclose(fs, f, rtol=1e-12)


# ----------------------------------------------------------------------- dense-contraction form
# oracle/dense.py evaluates the same iteration as S = Y T(x)^T, Z = W^T Y through float64 BLAS (used for
# the configs[4] golden, where the brute-force loop would take ~30 h).  Pinned to the dense matrix form
# above (P and R_s built from their definitions) and to the brute-force loop on shapes with K = 2, 3, 4,
# odd L_low, zeros in rho and ragged chunking.
@pytest.mark.parametrize("Ll,K,N,sigma,seed,zeros", [(2, 2, 5, 0.7, 0, 0), (2, 2, 7, 0.5, 2, 1), (2, 3, 4, 0.6, 3, 1)])
def test_dense_form_equals_matrix_form(Ll, K, N, sigma, seed, zeros):
    from oracle.dense import em_iter_dense
    p = synth.make_random(Ll, K, N, sigma, seed, rho_zeros=zeros)
    x = p.x0.astype(np.float64)
    d = dense_em(p.y, p.K, p.sigma, x, p.rho1_0, p.rho2_0)
    r = em_iter_dense(p.y, p.L_low, p.K, p.sigma, x, p.rho1_0, p.rho2_0, project=False, tau=0.0, chunk=3)
    np.testing.assert_allclose(r.A.reshape(-1), np.diag(d["A"]), rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(r.b.reshape(-1), d["b"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(r.colsum, d["colsum"], rtol=1e-11, atol=1e-14)
    assert abs(r.loglik - d["LL"]) <= 1e-12 * abs(d["LL"])
    np.testing.assert_allclose(r.rho1, d["rho1"], rtol=1e-11, atol=1e-15)
    np.testing.assert_allclose(r.x, np.linalg.solve(d["A"], d["b"]).reshape(x.shape), rtol=1e-11, atol=1e-12)


@pytest.mark.parametrize("Ll,K,N,sigma,seed,zeros", [
    (4, 2, 37, 0.3, 1, 0), (4, 3, 21, 0.5, 2, 2), (3, 3, 17, 0.4, 6, 0), (8, 4, 9, 0.4, 3, 1),
    (16, 2, 50, 0.25, 4, 3), (5, 3, 13, 0.6, 5, 0)])
def test_dense_form_equals_bruteforce(oracle_mod, Ll, K, N, sigma, seed, zeros):
    from oracle.dense import em_iter_dense
    p = synth.make_random(Ll, K, N, sigma, seed, rho_zeros=zeros)
    a = oracle_mod.em_iter(p.y, Ll, K, sigma, p.x0, p.rho1_0, p.rho2_0, project=True)
    b = em_iter_dense(p.y, Ll, K, sigma, p.x0, p.rho1_0, p.rho2_0, project=True, chunk=7)
    for f in ("x", "b", "A", "colsum", "ll_obs", "rho1", "rho2"):
        u, v = getattr(a, f), getattr(b, f)
        assert np.abs(u - v).max() <= 1e-12 * np.abs(u).max() + 1e-300, f
    assert abs(a.loglik - b.loglik) <= 1e-13 * abs(a.loglik)
    assert np.all(b.rho1[p.rho1_0 == 0] == 0) and np.all(b.rho2[p.rho2_0 == 0] == 0)


def test_dense_form_reproduces_c1_golden():
    """configs[1]'s committed golden (10 projected iterations of the brute-force loop) from the dense form."""
    from oracle.dense import em_iter_dense
    g = np.load(os.path.join(GOLDEN, "c1_oracle.npz"))
    p = synth.make_config("c1")
    x, r1, r2, tr = p.x0, p.rho1_0, p.rho2_0, []
    for _ in range(int(g["iters"])):
        r = em_iter_dense(p.y, p.L_low, p.K, p.sigma, x, r1, r2, project=True, chunk=4096)
        x, r1, r2 = r.x, r.rho1, r.rho2
        tr.append(r.loglik)
    assert np.abs(x - g["x"]).max() <= 1e-12
    assert np.abs(r1 - g["rho1"]).max() <= 1e-13 and np.abs(r2 - g["rho2"]).max() <= 1e-13
    np.testing.assert_allclose(tr, g["trace"], rtol=1e-13)


# ----------------------------------------------------------------------- indexed log-likelihood
@pytest.mark.parametrize("Ll,K,N,sigma,seed", [(4, 2, 23, 0.4, 1), (3, 3, 11, 0.5, 2), (8, 4, 7, 0.3, 3),
                                               (128, 2, 3, 0.5, 4)])
def test_loglik_obs_equals_em_iter_terms(oracle_mod, Ll, K, N, sigma, seed):
    """oracle.loglik_obs (the per-observation checker of the full-size configs[4] test) equals the
    per-observation terms of em_iter at any index set, order and repetition (an index-offset mistake
    would pick another observation's term)."""
    p = synth.make_random(Ll, K, N, sigma, seed, rho_zeros=1, image="blobs" if Ll >= 64 else "noise")
    r = oracle_mod.em_iter(p.y, Ll, K, sigma, p.x0, p.rho1_0, p.rho2_0, project=False)
    idx = np.array([N - 1, 0, N // 2, 0, 1 % N])
    got = oracle_mod.loglik_obs(p.y, idx, Ll, K, sigma, p.x0, p.rho1_0, p.rho2_0)
    np.testing.assert_allclose(got, r.ll_obs[idx], rtol=1e-14)
    # and each term is the log normaliser of that observation's own posterior (eq:weights_EM)
    for i in {0, N - 1}:
        _, lse = oracle_mod.posterior(p.y[i], Ll, K, sigma, p.x0, p.rho1_0, p.rho2_0)
        assert abs(lse - r.ll_obs[i]) <= 1e-14 * abs(lse)
