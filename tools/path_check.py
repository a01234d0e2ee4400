"""Parity of one path vs the oracle on small shapes and one config (quick GPU check)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else "gemm"
cases = [synth.make_random(4, 2, 37, 0.5, 1), synth.make_random(8, 2, 130, 0.3, 2),
         synth.make_random(8, 4, 45, 0.25, 3, rho_zeros=2), synth.make_random(16, 2, 300, 0.25, 4),
         synth.make_config("c0"), synth.make_config("c1", N=1000)]
for p in cases:
    ref = oracle.em_iter(p.y, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=True)
    t0 = time.time()
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path=path) as ctx:
        ctx.em_iter(1)
        x, r1, r2, ll, _ = ctx.get_estimate()
        b, cm, m1, m2 = ctx.stats()
    xe = np.abs(x - ref.x).max() / np.abs(ref.x).max()
    re = max(np.abs(r1 - ref.rho1).max() / ref.rho1.max(), np.abs(r2 - ref.rho2).max() / ref.rho2.max())
    be = np.abs(b - ref.b).max() / np.abs(ref.b).max()
    print(f"{p.name:24s} path={path} x_err={xe:.2e} rho_err={re:.2e} b_err={be:.2e} "
          f"ll_err={abs(ll - ref.loglik) / abs(ref.loglik):.2e} ({time.time() - t0:.2f}s)", flush=True)
