"""Seeded synthetic SR-MRA workloads (shared input generator for the oracle and the CUDA path).

This module holds NO arithmetic of the EM method. It only draws the inputs the paper's
problem statement names (§I eq:model_1 and its explicit form):

    y_i[n1, n2] = x[(n1*K - s_i^1) mod L_high, (n2*K - s_i^2) mod L_high] + eps_i[n1, n2]

with s^1 ~ rho1, s^2 ~ rho2 i.i.d. and eps i.i.d. N(0, sigma^2), plus the
initial estimate (x0, rho0).  The recipes are BASELINE.json `configs[0..4]` as made concrete
in SURVEY.md §8(d) ("Synthetic inputs"); they stand in for the paper's images (CBSD-68, Lena,
an EMDB ribosome image), which are not available ("Input recipe").

All draws are made in float64 from numpy PCG64 streams spawned from
SeedSequence(20220411 + config_index): children (image, shifts, noise, init).  y is cast to
float32 and that float32 array is the shared input of both sides.
"""
from __future__ import annotations

import dataclasses
import numpy as np

__all__ = ["Problem", "CONFIGS", "make_config", "make_random", "observe"]


@dataclasses.dataclass
class Problem:
    """One SR-MRA workload.  Arrays are C-contiguous."""
    name: str
    L_high: int
    L_low: int
    K: int
    sigma: float
    y: np.ndarray          # float32 [N][L_low][L_low]
    x0: np.ndarray         # float32 [L_high][L_high]   initial estimate
    rho1_0: np.ndarray     # float64 [L_high]
    rho2_0: np.ndarray     # float64 [L_high]
    iters: int = 1         # EM iterations the config asks for
    x_true: np.ndarray | None = None      # float64 [L_high][L_high]
    shifts: np.ndarray | None = None      # int64 [N][2]  (diagnostics only)
    rho1_true: np.ndarray | None = None
    rho2_true: np.ndarray | None = None

    @property
    def N(self) -> int:
        return int(self.y.shape[0])


# ---------------------------------------------------------------- image / pmf recipes
def _circ_dist(L: int) -> np.ndarray:
    k = np.arange(L)
    return np.minimum(k, L - k).astype(np.float64)


def _blurred_noise(rng: np.random.Generator, L: int, sigma_b: float) -> np.ndarray:
    """N(0,1) field, circularly Gaussian-blurred (kernel ∝ exp(-d_circ^2/(2 sigma_b^2)), sum 1,
    applied by FFT), scaled so max|x| = 1 (BASELINE.json configs[0])."""
    z = rng.standard_normal((L, L))
    d = _circ_dist(L)
    ker = np.exp(-(d[:, None] ** 2 + d[None, :] ** 2) / (2.0 * sigma_b ** 2))
    ker /= ker.sum()
    x = np.real(np.fft.ifft2(np.fft.fft2(z) * np.fft.fft2(ker)))
    return x / np.max(np.abs(x))


def _blobs(rng: np.random.Generator, L: int, n_blobs: int) -> np.ndarray:
    """Sum of periodic isotropic Gaussian blobs: centres U[0,L)^2, std U[L/32, L/8],
    amplitude U[0.5, 1]; normalised to max 1 (BASELINE.json configs[2..4])."""
    c = rng.uniform(0.0, L, size=(n_blobs, 2))
    sd = rng.uniform(L / 32.0, L / 8.0, size=n_blobs)
    amp = rng.uniform(0.5, 1.0, size=n_blobs)
    k = np.arange(L, dtype=np.float64)
    x = np.zeros((L, L))
    for j in range(n_blobs):
        d1 = np.abs(k - c[j, 0]); d1 = np.minimum(d1, L - d1)
        d2 = np.abs(k - c[j, 1]); d2 = np.minimum(d2, L - d2)
        x += amp[j] * np.exp(-(d1[:, None] ** 2 + d2[None, :] ** 2) / (2.0 * sd[j] ** 2))
    return x / np.max(x)


def _discrete_gaussian(L: int, centre: float, std: float) -> np.ndarray:
    k = np.arange(L, dtype=np.float64)
    p = np.exp(-((k - centre) ** 2) / (2.0 * std ** 2))
    return p / p.sum()


# ---------------------------------------------------------------- forward model (eq:model_1)
def observe(x: np.ndarray, shifts: np.ndarray, K: int, sigma: float,
            rng: np.random.Generator | None, chunk: int = 8192) -> np.ndarray:
    """y_i = P R_{s_i} x + eps_i, PAPER.md:37-38 (explicit form of eq:model_1), float32 out.

    Drawn in float64 (noise too) and cast to float32 at the end, chunked over i."""
    L = x.shape[0]
    Ll = L // K
    N = shifts.shape[0]
    y = np.empty((N, Ll, Ll), dtype=np.float32)
    n = np.arange(Ll)
    for a in range(0, N, chunk):
        b = min(N, a + chunk)
        s1 = shifts[a:b, 0][:, None]
        s2 = shifts[a:b, 1][:, None]
        rows = (n[None, :] * K - s1) % L            # [B, Ll]
        cols = (n[None, :] * K - s2) % L            # [B, Ll]
        blk = x[rows[:, :, None], cols[:, None, :]]  # [B, Ll, Ll] float64
        if sigma > 0 and rng is not None:
            blk = blk + sigma * rng.standard_normal(blk.shape)
        y[a:b] = blk.astype(np.float32)
    return y


# ---------------------------------------------------------------- BASELINE.json configs
CONFIGS = {
    # name: (L_high, L_low, K, N, sigma, iters)
    "c0": (16, 8, 2, 500, 0.125, 1),
    "c1": (64, 32, 2, 10_000, 0.25, 10),
    "c2": (128, 64, 2, 20_000, 0.5, 1),
    "c3": (128, 32, 4, 100_000, 0.125, 1),
    "c4": (256, 128, 2, 100_000, 0.5, 1),
}


def make_config(name: str, N: int | None = None, seed_offset: int = 0) -> Problem:
    """BASELINE.json configs[c] with the recipe of SURVEY.md §8(d).  `N` overrides the
    observation count (first N observations of the same streams are NOT guaranteed to be a
    prefix of the full set; use it for reduced-size parity cases)."""
    L, Ll, K, N_cfg, sigma, iters = CONFIGS[name]
    c = int(name[1:])
    N = N_cfg if N is None else int(N)
    ss = np.random.SeedSequence(20220411 + c + seed_offset)
    r_img, r_sh, r_noise, r_init = [np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(4)]

    if c == 0:
        x = _blurred_noise(r_img, L, 1.5)
        rho1 = rho2 = _discrete_gaussian(L, L / 2, 2.0)
        x0 = _blurred_noise(r_init, L, 1.5)
    elif c == 1:
        x = _blurred_noise(r_img, L, 3.0)
        rho1 = rho2 = _discrete_gaussian(L, L / 2, L / 8)
        x0 = _blurred_noise(r_init, L, 3.0)
    elif c == 2:
        x = _blobs(r_img, L, 30)
        rho1 = rho2 = _discrete_gaussian(L, L / 2, 16.0)
        x0 = _blurred_noise(r_init, L, 3.0)
    elif c == 3:
        x = _blobs(r_img, L, 30)
        rho1 = r_sh.dirichlet(np.ones(L))
        rho2 = r_sh.dirichlet(np.ones(L))
        x0 = _blurred_noise(r_init, L, 3.0)
    elif c == 4:
        x = _blobs(r_img, L, 60)
        rho1 = rho2 = _discrete_gaussian(L, L / 2, 32.0)
        x0 = _blurred_noise(r_init, L, 3.0)
    else:
        raise ValueError(name)

    s1 = r_sh.choice(L, size=N, p=rho1)
    s2 = r_sh.choice(L, size=N, p=rho2)
    shifts = np.stack([s1, s2], axis=1).astype(np.int64)
    y = observe(x, shifts, K, sigma, r_noise)
    u = np.full(L, 1.0 / L)
    return Problem(name=name, L_high=L, L_low=Ll, K=K, sigma=sigma, y=y,
                   x0=np.ascontiguousarray(x0.astype(np.float32)),
                   rho1_0=u.copy(), rho2_0=u.copy(), iters=iters, x_true=x, shifts=shifts,
                   rho1_true=rho1, rho2_true=rho2)


def make_random(L_low: int, K: int, N: int, sigma: float, seed: int,
                rho_zeros: int = 0, rho_kind: str = "dirichlet", image: str = "noise") -> Problem:
    """Randomised small shapes (SURVEY.md §4 'randomised tiny shapes'): blurred-noise image
    (`image="noise"`) or the blob image of configs[2..4] (`image="blobs"`, 2 L / 8 blobs),
    Dirichlet shift pmfs (optionally with `rho_zeros` exact zeros in the *initial* rho),
    odd N allowed."""
    L = L_low * K
    ss = np.random.SeedSequence([777, L_low, K, N, seed])
    r_img, r_sh, r_noise, r_init = [np.random.Generator(np.random.PCG64(s)) for s in ss.spawn(4)]
    x = _blobs(r_img, L, max(1, L // 4)) if image == "blobs" else _blurred_noise(r_img, L, max(1.0, L / 16))
    if rho_kind == "dirichlet":
        rho1 = r_sh.dirichlet(np.ones(L))
        rho2 = r_sh.dirichlet(np.ones(L))
    else:
        rho1 = rho2 = np.full(L, 1.0 / L)
    s1 = r_sh.choice(L, size=N, p=rho1)
    s2 = r_sh.choice(L, size=N, p=rho2)
    shifts = np.stack([s1, s2], axis=1).astype(np.int64)
    y = observe(x, shifts, K, sigma, r_noise)
    x0 = _blurred_noise(r_init, L, max(1.0, L / 16))
    r10 = r_init.uniform(0.2, 1.0, L)
    r20 = r_init.uniform(0.2, 1.0, L)
    if rho_zeros:
        zi = r_init.choice(L, size=min(rho_zeros, L - 1), replace=False)
        r10[zi] = 0.0
        zj = r_init.choice(L, size=min(rho_zeros, L - 1), replace=False)
        r20[zj] = 0.0
    r10 /= r10.sum()
    r20 /= r20.sum()
    return Problem(name=f"rand_L{L_low}_K{K}_N{N}_s{seed}", L_high=L, L_low=L_low, K=K,
                   sigma=sigma, y=y, x0=np.ascontiguousarray(x0.astype(np.float32)),
                   rho1_0=r10, rho2_0=r20, iters=1, x_true=x, shifts=shifts,
                   rho1_true=rho1, rho2_true=rho2)
