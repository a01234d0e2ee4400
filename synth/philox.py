"""Counter-based synthetic observations (NEXT-4's "GPU data generator for large N"): the reference of the
device generator `srmra_generate`.  Input generation only (the forward model of PAPER.md:37-38), no EM
arithmetic; both sides implement the same counter-based generator, so the device draws can be checked
draw by draw.

Generator: Philox4x32-10 (Salmon et al., SC'11; constants M0 = 0xD2511F53, M1 = 0xCD9E8D57, key bumps
W0 = 0x9E3779B9, W1 = 0xBB67AE85), key = (seed mod 2^32, seed >> 32).  For global observation index j
(counter words c0 = j mod 2^32, c1 = j >> 32):
  * shifts: Philox((c0, c1, 0, 0)) -> (u0, u1, ., .); U = (u + 0.5) 2^-32 (float64);
    s^1 = min{k : U_0 < C1[k]}, C1 = cumsum(rho1) in float64 (sequential), s^2 likewise from U_1 and
    rho2; a draw at or above the last partial sum takes the last k with rho[k] > 0.
  * noise: for b = 0, 1, ...: Philox((c0, c1, 1 + b, 0)) -> (r0, r1, r2, r3); V = ((r >> 9) + 0.5) 2^-23
    (exact in float32); Box-Muller pairs (V0, V1), (V2, V3): z = sqrt(-2 ln V_a) (cos, sin)(2 pi V_b)
    give the noise of pixels 4b .. 4b + 3 of y_j (row-major, L_low^2 pixels).
  * y_j[n1, n2] = x[(n1 K - s^1) mod L, (n2 K - s^2) mod L] + sigma z   (float32).
"""
from __future__ import annotations

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 on uint64 arrays holding 32-bit words; returns four uint64 arrays."""
    c0, c1, c2, c3 = (np.asarray(v, dtype=np.uint64) & MASK for v in (c0, c1, c2, c3))
    k0 = np.uint64(k0 & MASK)
    k1 = np.uint64(k1 & MASK)
    for r in range(10):
        if r:
            k0 = np.uint64((int(k0) + W0) & MASK)
            k1 = np.uint64((int(k1) + W1) & MASK)
        p0 = np.uint64(M0) * c0
        p1 = np.uint64(M1) * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & np.uint64(MASK)
        hi1, lo1 = p1 >> np.uint64(32), p1 & np.uint64(MASK)
        c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return c0, c1, c2, c3


def _key(seed: int):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & MASK, seed >> 32


def sample_shift(u, rho):
    """Inverse-CDF draw on the float64 sequential partial sums of rho (see the module docstring)."""
    C = np.cumsum(np.asarray(rho, dtype=np.float64))
    U = (u.astype(np.float64) + 0.5) * 2.0 ** -32
    s = np.searchsorted(C, U, side="right")   # min k with U < C[k]
    last = int(np.nonzero(np.asarray(rho) > 0)[0][-1])
    return np.minimum(s, last)


def generate(x, rho1, rho2, K: int, sigma: float, n: int, seed: int, first_index: int = 0):
    """(y float32 [n][L_low][L_low], shifts int32 [n][2]) for global indices first_index .. + n - 1."""
    x = np.asarray(x, dtype=np.float32)
    L = x.shape[0]
    Ll = L // K
    k0, k1 = _key(seed)
    j = np.arange(first_index, first_index + n, dtype=np.uint64)
    jl, jh = j & np.uint64(MASK), j >> np.uint64(32)
    zero = np.zeros_like(j)
    u0, u1, _, _ = philox4x32_10(jl, jh, zero, zero, k0, k1)
    s1 = sample_shift(u0, rho1)
    s2 = sample_shift(u1, rho2)
    P = Ll * Ll
    nb = (P + 3) // 4
    z = np.empty((n, 4 * nb), dtype=np.float64)
    for b in range(nb):
        r0, r1, r2, r3 = philox4x32_10(jl, jh, zero + np.uint64(1 + b), zero, k0, k1)
        V = [((r >> np.uint64(9)).astype(np.float64) + 0.5) * 2.0 ** -23 for r in (r0, r1, r2, r3)]
        ra = np.sqrt(-2.0 * np.log(V[0]))
        rb = np.sqrt(-2.0 * np.log(V[2]))
        z[:, 4 * b] = ra * np.cos(2 * np.pi * V[1])
        z[:, 4 * b + 1] = ra * np.sin(2 * np.pi * V[1])
        z[:, 4 * b + 2] = rb * np.cos(2 * np.pi * V[3])
        z[:, 4 * b + 3] = rb * np.sin(2 * np.pi * V[3])
    nn = np.arange(Ll)
    rows = (nn[None, :] * K - s1[:, None]) % L
    cols = (nn[None, :] * K - s2[:, None]) % L
    clean = x.astype(np.float64)[rows[:, :, None], cols[:, None, :]]
    y = (clean + sigma * z[:, :P].reshape(n, Ll, Ll)).astype(np.float32)
    return y, np.stack([s1, s2], axis=1).astype(np.int32)
