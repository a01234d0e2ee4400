"""Quick L_low = 128 check: tiny shapes and the c4 geometry at small N vs the oracle, then c4 timing."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402

oracle.build()


def err(p, g, ref):
    x, r1, r2, ll = g
    xe = np.abs(x - ref.x).max() / np.abs(ref.x).max()
    re = max(np.abs(r1 - ref.rho1).max() / ref.rho1.max(), np.abs(r2 - ref.rho2).max() / ref.rho2.max())
    le = abs(ll - ref.loglik) / abs(ref.loglik)
    return xe, re, le


cases = [("tinyK1", synth.make_random(128, 1, 5, 0.5, 11)), ("tinyK2", synth.make_random(128, 2, 6, 0.35, 12, rho_zeros=2)),
         ("c4/N=24", synth.make_config("c4", N=24))]
for name, p in cases:
    t0 = time.time()
    ref = oracle.em_iter(p.y, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=True)
    t1 = time.time()
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path="fft") as ctx:
        ctx.em_iter(1)
        x, r1, r2, ll, it = ctx.get_estimate()
        llo = ctx.obs_loglik()
    xe, re, le = err(p, (x, r1, r2, ll), ref)
    lloe = np.abs(llo - ref.ll_obs).max() / np.abs(ref.ll_obs).max()
    print(f"{name}: oracle {t1 - t0:.1f}s  x_err={xe:.2e} rho_err={re:.2e} ll_err={le:.2e} llobs_err={lloe:.2e}", flush=True)

p = synth.make_config("c4")
units = p.N * p.L_high ** 2
t0 = time.time()
with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path="fft") as ctx:
    ctx.em_iter(1)
    ctx.get_estimate()
    t1 = time.time()
    ctx.profile(True)
    ctx.em_iter(3)
    em, tot, n = ctx.profile_read()
    print(f"c4 fft: init+1 iter {t1 - t0:.2f}s  E/M {em / n:.3f} ms  iteration {tot / n:.3f} ms  "
          f"{units / (tot / n / 1e3):.3e} obs*shift/s", flush=True)
    llo = ctx.obs_loglik()
idx = np.array([0, 1, 12345, 54321, 77777, p.N - 1])
