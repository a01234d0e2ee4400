"""Parity margin at L_low = 128 vs N: one iteration from theta_0 and from the GPU's theta_1."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402

oracle.build()


def one(p, x0, r1, r2):
    ref = oracle.em_iter(p.y, p.L_low, p.K, p.sigma, x0, r1, r2, project=True)
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, x0, r1, r2, path="fft") as ctx:
        ctx.em_iter(1)
        x, q1, q2, ll, it = ctx.get_estimate()
        b, cm, m1, m2 = ctx.stats()
    xe = np.abs(x - ref.x).max() / np.abs(ref.x).max()
    re = max(np.abs(q1 - ref.rho1).max() / ref.rho1.max(), np.abs(q2 - ref.rho2).max() / ref.rho2.max())
    be = np.abs(b - ref.b).max() / np.abs(ref.b).max()
    le = abs(ll - ref.loglik) / abs(ref.loglik)
    return x, q1, q2, f"x={xe:.2e} rho={re:.2e} b={be:.2e} ll={le:.2e}"


for N in (24, 96):
    p = synth.make_config("c4", N=N)
    x1, q1, q2, msg = one(p, p.x0, p.rho1_0, p.rho2_0)
    print(f"c4 N={N} theta0: {msg}", flush=True)
    _, _, _, msg = one(p, x1.astype(np.float32), q1, q2)
    print(f"c4 N={N} theta1: {msg}", flush=True)
for (K, N, s, seed, z) in [(1, 16, 0.5, 11, 0), (2, 16, 0.5, 12, 2), (2, 16, 0.5, 14, 0), (1, 16, 0.5, 15, 3)]:
    p = synth.make_random(128, K, N, s, seed, rho_zeros=z, image="blobs")
    _, _, _, msg = one(p, p.x0, p.rho1_0, p.rho2_0)
    print(f"tiny blobs K={K} N={N} sigma={s} seed={seed}: {msg}", flush=True)
