"""ctypes wrapper of the float64 CPU oracle (oracle/srmra_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs, never by the product package.  See the header of
srmra_oracle.c for the passages of PAPER.md each step follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "srmra_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_ip = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O3 -march=x86-64-v3 -fopenmp; no -ffast-math; portable to the GPU hosts)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v3", "-fopenmp", "-fPIC", "-shared",
                               "-std=c11", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_em_iter.restype = ctypes.c_int
        lib.oracle_em_iter.argtypes = [_fp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_double, _dp, _dp, _dp, ctypes.c_int, ctypes.c_double,
                                       _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.oracle_em_iter_joint.restype = ctypes.c_int
        lib.oracle_em_iter_joint.argtypes = [_fp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_double, _dp, _dp, ctypes.c_int, ctypes.c_double,
                                             _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp]
        lib.oracle_posterior.restype = ctypes.c_double
        lib.oracle_posterior.argtypes = [_fp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                         _dp, _dp, _dp, _dp]
        lib.oracle_loglik_obs.restype = ctypes.c_int
        lib.oracle_loglik_obs.argtypes = [_fp, _ip, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_int, ctypes.c_double, _dp, _dp, _dp, _dp]
        lib.oracle_project.restype = None
        lib.oracle_project.argtypes = [_dp, ctypes.c_int, _dp]
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t):
    return None if a is None else a.ctypes.data_as(t)


@dataclass
class IterResult:
    x: np.ndarray        # float64 [L][L]   (after projection if requested)
    rho1: np.ndarray     # float64 [L]
    rho2: np.ndarray
    loglik: float        # LL at the input theta
    b: np.ndarray        # float64 [L][L]   numerator of eq:x_EM
    A: np.ndarray        # float64 [L][L]   diagonal of A in eq:x_EM
    colsum: np.ndarray   # float64 [L][L]   sum_i w^{i,s}
    ll_obs: np.ndarray   # float64 [N]


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def em_iter(y, L_low, K, sigma, x, rho1, rho2, project=True, tau=None) -> IterResult:
    """One EM iteration (eq:weights_EM, eq:x_EM, eq:rho_EM) + optional stand-in projection."""
    lib = _load()
    y = _f32(y)
    N = y.shape[0]
    L = L_low * K
    x = _f64(x).reshape(L, L)
    rho1 = _f64(rho1)
    rho2 = _f64(rho2)
    if tau is None:
        tau = 1e-12 * N
    xo = np.empty((L, L)); r1 = np.empty(L); r2 = np.empty(L); ll = np.empty(1)
    b = np.empty((L, L)); A = np.empty((L, L)); cs = np.empty((L, L)); llo = np.empty(N)
    rc = lib.oracle_em_iter(_p(y, _fp), N, L, L_low, K, float(sigma), _p(x, _dp), _p(rho1, _dp),
                            _p(rho2, _dp), int(bool(project)), float(tau), _p(xo, _dp), _p(r1, _dp),
                            _p(r2, _dp), _p(ll, _dp), _p(b, _dp), _p(A, _dp), _p(cs, _dp), _p(llo, _dp))
    if rc != 0:
        raise ValueError(f"oracle_em_iter failed rc={rc}")
    return IterResult(xo, r1, r2, float(ll[0]), b, A, cs, llo)


@dataclass
class JointResult:
    x: np.ndarray        # float64 [L][L]
    rho: np.ndarray      # float64 [L][L] joint prior rho'[s1, s2]
    rho1: np.ndarray     # its marginals
    rho2: np.ndarray
    loglik: float
    b: np.ndarray
    A: np.ndarray
    colsum: np.ndarray
    ll_obs: np.ndarray


def em_iter_joint(y, L_low, K, sigma, x, rho, project=True, tau=None) -> JointResult:
    """NEXT-3: one EM iteration with a joint shift prior rho [L][L] (eq:rho_EM as written)."""
    lib = _load()
    y = _f32(y)
    N = y.shape[0]
    L = L_low * K
    x = _f64(x).reshape(L, L)
    rho = _f64(rho).reshape(L, L)
    if tau is None:
        tau = 1e-12 * N
    xo = np.empty((L, L)); ro = np.empty((L, L)); r1 = np.empty(L); r2 = np.empty(L); ll = np.empty(1)
    b = np.empty((L, L)); A = np.empty((L, L)); cs = np.empty((L, L)); llo = np.empty(N)
    rc = lib.oracle_em_iter_joint(_p(y, _fp), N, L, L_low, K, float(sigma), _p(x, _dp), _p(rho, _dp),
                                  int(bool(project)), float(tau), _p(xo, _dp), _p(ro, _dp), _p(r1, _dp),
                                  _p(r2, _dp), _p(ll, _dp), _p(b, _dp), _p(A, _dp), _p(cs, _dp), _p(llo, _dp))
    if rc != 0:
        raise ValueError(f"oracle_em_iter_joint failed rc={rc}")
    return JointResult(xo, ro, r1, r2, float(ll[0]), b, A, cs, llo)


def run(y, L_low, K, sigma, x0, rho1_0, rho2_0, iters, proj_every=1, tau=None):
    """`iters` iterations of Algorithm 2 with the stand-in projection applied
    after iteration t when (t+1) % proj_every == 0 (proj_every=0: never).  Returns
    (x, rho1, rho2, [LL_0..LL_{iters-1}])."""
    x, r1, r2 = _f64(x0), _f64(rho1_0), _f64(rho2_0)
    trace = []
    for t in range(iters):
        proj = proj_every > 0 and (t + 1) % proj_every == 0
        r = em_iter(y, L_low, K, sigma, x, r1, r2, project=proj, tau=tau)
        x, r1, r2 = r.x, r.rho1, r.rho2
        trace.append(r.loglik)
    return x, r1, r2, trace


def sigma_schedule(j: int) -> float:
    """sigma^BM3D of the j-th projection (j = 1, 2, ...): sigma_1 = 1, sigma_j = 2^(-1/10) sigma_{j-1}
    (eq:decaying_function), evaluated by the recursion as written."""
    s = 1.0
    for _ in range(1, j):
        s *= 2.0 ** (-1.0 / 10.0)
    return s


def run_alg2(y, L_low, K, sigma, x0, rho1_0, rho2_0, max_iters, proj_every=1, rel_tol=0.0, denoiser=None,
             tau=None):
    """Algorithm 2 (projected EM): EM steps; after every F-th step (F = proj_every)
    x <- D(x, sigma_j) with the schedule sigma_j of eq:decaying_function; stop after the first iteration
    t >= 1 with |LL_t - LL_{t-1}| <= rel_tol |LL_t| (reading R12; rel_tol <= 0: never) or after
    max_iters.  D is the north_star stand-in (3x3 circular box, clamp) unless `denoiser(x, sigma_j)`
    is given.  Returns (x, rho1, rho2, [LL_0..], [sigma_1..] of the projections applied)."""
    x, r1, r2 = _f64(x0), _f64(rho1_0), _f64(rho2_0)
    trace, sigmas = [], []
    for t in range(max_iters):
        proj = proj_every > 0 and (t + 1) % proj_every == 0
        r = em_iter(y, L_low, K, sigma, x, r1, r2, project=proj and denoiser is None, tau=tau)
        x, r1, r2 = r.x, r.rho1, r.rho2
        trace.append(r.loglik)
        if proj:
            sigmas.append(sigma_schedule(len(sigmas) + 1))
            if denoiser is not None:
                x = _f64(denoiser(x, sigmas[-1]))
        if rel_tol > 0 and t >= 1 and abs(trace[t] - trace[t - 1]) <= rel_tol * abs(trace[t]):
            break
    return x, r1, r2, trace, sigmas


def relative_error(xhat, x):
    """error(x_hat) = min_s ||R_s x_hat - x||_F / ||x||_F, (R_s z)[p] = z[p - s]
    (Eq. (2) sign, np.roll), brute force over every shift; returns (error, (s1, s2)), ties: the
    smallest s1 L + s2."""
    xhat = _f64(xhat)
    x = _f64(x)
    L = x.shape[0]
    best, arg = np.inf, (0, 0)
    for s1 in range(L):
        for s2 in range(L):
            d = np.linalg.norm(np.roll(xhat, (s1, s2), axis=(0, 1)) - x)
            if d < best:
                best, arg = d, (s1, s2)
    return float(best / np.linalg.norm(x)), arg


# ---------------------------------------------------------------- NEXT-2: method of moments
def empirical_moments(y):
    """eq:empiric_MOM with D = 2: M1 = (1/N) sum_i y_i, M2 = (1/N) sum_i y_i y_i^T over
    vec(y_i) (row-major, L_low^2 entries), float64."""
    Y = _f32(y).reshape(y.shape[0], -1).astype(np.float64)
    N = Y.shape[0]
    return Y.sum(0) / N, (Y.T @ Y) / N


def analytic_moments(x, rho1, rho2, K, sigma, rho=None):
    """The first two moments of the model: M1 = P C_x rho, M2 = P C_x D_rho C_x^T P^T +
    sigma^2 P P^T, written as sums over the shifts s: (P C_x)[:, s] = vec(P R_s x), so
    M1 = sum_s rho[s] P R_s x and M2 = sum_s rho[s] (P R_s x)(P R_s x)^T + sigma^2 I (P P^T = I).
    rho[s] = rho1[s1] rho2[s2] (D_rho = diag vec(rho1 rho2^T)), or a joint `rho`."""
    x = _f64(x)
    L = x.shape[0]
    Ll = L // K
    pr = np.outer(rho1, rho2) if rho is None else _f64(rho).reshape(L, L)
    M1 = np.zeros(Ll * Ll)
    M2 = sigma ** 2 * np.eye(Ll * Ll)
    for s1 in range(L):
        for s2 in range(L):
            if pr[s1, s2] == 0.0:
                continue
            v = np.roll(x, (s1, s2), axis=(0, 1))[::K, ::K].reshape(-1)   # vec(P R_s x), Eq. (2)
            M1 += pr[s1, s2] * v
            M2 += pr[s1, s2] * np.outer(v, v)
    return M1, M2


def mom_lambda(L_high: int, sigma: float) -> float:
    """lambda = 1 / (L_high^2 (1 + sigma^2)) of eq:LS_SR."""
    return 1.0 / (L_high * L_high * (1.0 + sigma * sigma))


def shifted_templates(x, K):
    """V [L_high^2][L_low^2]: row s = s1 L_high + s2 is vec(P R_s x) (Eq. (2)), i.e. the
    columns of P C_x."""
    x = _f64(x)
    L = x.shape[0]
    V = np.empty((L * L, (L // K) ** 2))
    for s1 in range(L):
        for s2 in range(L):
            V[s1 * L + s2] = np.roll(x, (s1, s2), axis=(0, 1))[::K, ::K].reshape(-1)
    return V


def mom_objective(x, rho1, rho2, K, sigma, M1hat, M2hat):
    """The least-squares moment objective eq:LS_SR at theta = (x, rho1 rho2^T):
        f = || P C_x D_rho C_x^T P^T + sigma^2 I - M2hat ||_F^2 + lambda || P C_x rho - M1hat ||_2^2,
    lambda = mom_lambda(L_high, sigma), and its gradient (derived here, not printed in the paper; pinned by
    finite differences): with V = shifted_templates(x), E = M2(theta) - M2hat, e = M1(theta) - M1hat,
        df/drho[s] = 2 v_s^T E v_s + 2 lambda e^T v_s                      (joint rho, s = s1 L + s2)
        df/dx      = sum_s rho[s] R_s^T P^T (4 E v_s + 2 lambda e)         (E symmetric)
        df/drho1[s1] = sum_s2 df/drho[s1, s2] rho2[s2],  df/drho2[s2] = sum_s1 df/drho[s1, s2] rho1[s1].
    Returns (f, grad_x [L][L], grad_rho1 [L], grad_rho2 [L], grad_rho [L][L])."""
    x = _f64(x)
    L = x.shape[0]
    Ll = L // K
    rho = np.outer(_f64(rho1), _f64(rho2))
    r = rho.reshape(-1)
    V = shifted_templates(x, K)
    M1 = V.T @ r
    M2 = V.T @ (r[:, None] * V) + sigma ** 2 * np.eye(Ll * Ll)
    E = M2 - _f64(M2hat)
    e = M1 - _f64(M1hat).reshape(-1)
    lam = mom_lambda(L, sigma)
    f = float((E * E).sum() + lam * (e * e).sum())
    G = V @ E                                                   # row s: E v_s
    grho = (2.0 * (G * V).sum(1) + 2.0 * lam * (V @ e)).reshape(L, L)
    gx = np.zeros((L, L))
    for s1 in range(L):
        for s2 in range(L):
            z = r[s1 * L + s2] * (4.0 * G[s1 * L + s2] + 2.0 * lam * e)
            up = np.zeros((L, L))
            up[::K, ::K] = z.reshape(Ll, Ll)                    # P^T z
            gx += np.roll(up, (-s1, -s2), axis=(0, 1))           # R_s^T = R_{-s}
    return f, gx, grho @ _f64(rho2), grho.T @ _f64(rho1), grho


def posterior(yi, L_low, K, sigma, x, rho1, rho2):
    """(w [L][L], log-likelihood term) of one observation."""
    lib = _load()
    yi = _f32(yi)
    L = L_low * K
    w = np.empty((L, L))
    lse = lib.oracle_posterior(_p(yi, _fp), L, L_low, K, float(sigma), _p(_f64(x), _dp),
                               _p(_f64(rho1), _dp), _p(_f64(rho2), _dp), _p(w, _dp))
    return w, float(lse)


def loglik_obs(y, idx, L_low, K, sigma, x, rho1, rho2):
    """Per-observation log-likelihood terms for observation indices `idx`."""
    lib = _load()
    y = _f32(y)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    out = np.empty(idx.shape[0])
    rc = lib.oracle_loglik_obs(_p(y, _fp), _p(idx, _ip), idx.shape[0], L_low * K, L_low, K,
                               float(sigma), _p(_f64(x), _dp), _p(_f64(rho1), _dp),
                               _p(_f64(rho2), _dp), _p(out, _dp))
    if rc != 0:
        raise ValueError(f"oracle_loglik_obs rc={rc}")
    return out


def project(x):
    """3x3 circular box filter + clamp[-1,1] (north_star stand-in for the denoiser)."""
    lib = _load()
    x = _f64(x)
    L = x.shape[0]
    out = np.empty_like(x)
    lib.oracle_project(_p(x, _dp), L, _p(out, _dp))
    return out
