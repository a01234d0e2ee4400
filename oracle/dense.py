"""Float64 CPU oracle of one EM iteration in the paper's dense matrix form (numpy + BLAS).

TEST INFRASTRUCTURE ONLY: imported by tests/ and tests/golden/make_golden.py, never by the product
package.  It shares no code with the CUDA path.

Why a second form: the brute-force loop of srmra_oracle.c does N·L²·Ll² scalar residual terms
twice (E and M); at configs[4] (N = 10⁵, L = 256, Ll = 128) that is 2·10¹⁴ terms, ~30 h on this
host's 8 cores.  The same iteration written as the dense contraction the north_star names
(S = Y·T(x)ᵀ, Z = WᵀY) runs through float64 BLAS in ~30 min.  Every step is the plain definition:

  templates   T[s][n] = (P R_s x)[n] = x[(n1 K − s1) mod L, (n2 K − s2) mod L]   PAPER.md:37-38 (Eq. 2),
              the columns of P C_x, materialised by the index formula;
  E-step      ‖y_i − P R_s x‖² = ‖y_i‖² + ‖T[s]‖² − 2 (Y Tᵀ)[i, s]          (expansion of the norm),
              ℓ[i, s] = log ρ1[s1] + log ρ2[s2] − ‖·‖²/(2σ²),  lse_i = log Σ_s exp ℓ[i, s]
              (eq:likelihood_EM), w = exp(ℓ − lse)  (eq:weights_EM);
  M-step      Z = Wᵀ Y (Z[s][n] = Σ_i w^{i,s} y_i[n]); b[p] = Σ_{s,n: p = idx(s,n)} Z[s][n],
              A[p] = Σ_{s,n: p = idx(s,n)} Σ_i w^{i,s}  (eq:x_EM with P⁻¹ read as Pᵀ, reading R1,
              PAPER.md:255-263); x' = b/A where A > τ (reading R6);
              ρ1', ρ2' = marginals of Σ_i w^{i,s} / Σ_i Σ_s w  (eq:rho_EM, reading R2);
  projection  the stand-in D (3×3 circular box, clamp) of the brute-force oracle (reading R7).

Pinned (tests/test_oracle_pins.py): equal to the brute-force oracle em_iter (b, A, colsum, ll_obs, x,
ρ, LL) on random shapes with K = 2, 3, 4 and zeros in ρ, and to the committed brute-force golden of
configs[1] after its 10 iterations.  Observations are processed in chunks (memory only: every
per-observation quantity is independent of the chunking; the chunk sums are added in chunk order).
"""
from __future__ import annotations

import numpy as np

from . import IterResult, project as _project


def _rows(L: int, Ll: int, K: int) -> np.ndarray:
    """rows[s][n] = (n K − s) mod L, the sampled index of Eq. (2) along one axis."""
    return (np.arange(Ll)[None, :] * K - np.arange(L)[:, None]) % L


def templates(x: np.ndarray, K: int) -> np.ndarray:
    """T [L²][Ll²] float64, row s = s1 L + s2 is vec(P R_s x) (Eq. (2))."""
    L = x.shape[0]
    Ll = L // K
    rows = _rows(L, Ll, K)
    T = np.empty((L, L, Ll, Ll))
    for s1 in range(L):
        # T[s1, s2, n1, n2] = x[rows[s1, n1], rows[s2, n2]]
        T[s1] = x[rows[s1][None, :, None], rows[:, None, :]]
    return T.reshape(L * L, Ll * Ll)


def em_iter_dense(y, L_low, K, sigma, x, rho1, rho2, project=True, tau=None, chunk=1024,
                  verbose=False) -> IterResult:
    """One EM iteration in the dense form; same outputs as oracle.em_iter (ll_obs for every i)."""
    y = np.asarray(y, dtype=np.float32)
    N = y.shape[0]
    L = L_low * K
    Ll2 = L_low * L_low
    x = np.ascontiguousarray(x, dtype=np.float64).reshape(L, L)
    rho1 = np.asarray(rho1, dtype=np.float64)
    rho2 = np.asarray(rho2, dtype=np.float64)
    if tau is None:
        tau = 1e-12 * N
    with np.errstate(divide="ignore"):
        lprior = (np.log(rho1)[:, None] + np.log(rho2)[None, :]).reshape(-1)     # log ρ1[s1] + log ρ2[s2]
    T = templates(x, K)
    E = np.einsum("sn,sn->s", T, T)                                              # ‖P R_s x‖²
    inv2s2 = 1.0 / (2.0 * sigma * sigma)
    Z = np.zeros((L * L, Ll2))
    colsum = np.zeros(L * L)
    ll_obs = np.empty(N)
    for c0 in range(0, N, chunk):
        Yc = y[c0:c0 + chunk].reshape(-1, Ll2).astype(np.float64)
        S = Yc @ T.T                                                             # ⟨y_i, P R_s x⟩
        yn = np.einsum("in,in->i", Yc, Yc)
        ell = lprior[None, :] - (yn[:, None] + E[None, :] - 2.0 * S) * inv2s2
        m = ell.max(axis=1)
        lse = m + np.log(np.exp(ell - m[:, None]).sum(axis=1))
        W = np.exp(ell - lse[:, None])
        ll_obs[c0:c0 + chunk] = lse
        colsum += W.sum(axis=0)
        Z += W.T @ Yc
        if verbose:
            print(f"  dense em_iter: {min(c0 + chunk, N)}/{N}", flush=True)
    # fold: p = idx(s, n) = ((n1 K − s1) mod L) L + (n2 K − s2) mod L
    rows = _rows(L, L_low, K)
    b = np.zeros(L * L)
    A = np.zeros(L * L)
    Z = Z.reshape(L, L, L_low, L_low)
    cs = colsum.reshape(L, L)
    for s1 in range(L):
        p = rows[s1][None, :, None] * L + rows[:, None, :]                      # [s2][n1][n2]
        b += np.bincount(p.reshape(-1), weights=Z[s1].reshape(-1), minlength=L * L)
        A += np.bincount(p.reshape(-1), weights=np.broadcast_to(cs[s1][:, None, None], p.shape).reshape(-1),
                         minlength=L * L)
    tot = colsum.sum()
    r1 = cs.sum(axis=1) / tot if tot > 0 else rho1.copy()
    r2 = cs.sum(axis=0) / tot if tot > 0 else rho2.copy()
    xn = np.where(A > tau, b / np.where(A > 0, A, 1.0), x.reshape(-1)).reshape(L, L)
    xo = _project(xn) if project else xn
    return IterResult(xo, r1, r2, float(ll_obs.sum()), b.reshape(L, L), A.reshape(L, L),
                      colsum.reshape(L, L), ll_obs)
