"""Error of the FFT path (fp32 register FFTs) and the GEMM path (3xTF32) vs the float64 oracle on
randomised shapes, as a function of L_low and N (one iteration, projection on)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402

oracle.build()
cases = [(32, 2, 6), (64, 2, 6), (128, 2, 6), (128, 2, 24), (128, 2, 96), (64, 2, 96), (128, 1, 6), (128, 1, 96)]
for Ll, K, N in cases:
    for seed in (12, 13):
        p = synth.make_random(Ll, K, N, 0.35, seed, rho_zeros=2)
        ref = oracle.em_iter(p.y, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=True)
        for path in ("fft", "gemm"):
            try:
                with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path=path) as ctx:
                    ctx.em_iter(1)
                    x, r1, r2, ll, it = ctx.get_estimate()
            except srm.SrmraError as e:
                print(f"Ll={Ll} K={K} N={N} seed={seed} {path}: {e}")
                continue
            xe = np.abs(x - ref.x).max() / np.abs(ref.x).max()
            re = max(np.abs(r1 - ref.rho1).max() / ref.rho1.max(), np.abs(r2 - ref.rho2).max() / ref.rho2.max())
            le = abs(ll - ref.loglik) / abs(ref.loglik)
            print(f"Ll={Ll:3d} K={K} N={N:3d} seed={seed} {path:4s}: x_err={xe:.2e} rho_err={re:.2e} ll_err={le:.2e}",
                  flush=True)
