"""Per-iteration LL error of a path vs the oracle when the GPU is fed the oracle's own theta_t."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else "gemm"
p = synth.make_config("c1", N=1000)
x, r1, r2 = p.x0.astype(np.float64), p.rho1_0, p.rho2_0
for t in range(3):
    ref = oracle.em_iter(p.y, p.L_low, p.K, p.sigma, x, r1, r2, project=True)
    # GPU from the fp32-rounded oracle state; oracle re-run from the same rounded state for a fair LL
    xf = x.astype(np.float32)
    ref_r = oracle.em_iter(p.y, p.L_low, p.K, p.sigma, xf.astype(np.float64), r1, r2, project=True)
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, xf, r1, r2, path=path) as ctx:
        ctx.em_iter(1)
        _, _, _, ll, _ = ctx.get_estimate()
        llo = ctx.obs_loglik()
    d = llo - ref_r.ll_obs
    print(f"t={t} {path}: LL_err(rounded theta)={abs(ll - ref_r.loglik) / abs(ref_r.loglik):.2e} "
          f"LL_err(vs fp64 theta)={abs(ll - ref.loglik) / abs(ref.loglik):.2e} obs max|d|={np.abs(d).max():.3e} "
          f"mean d={d.mean():.3e} rho0s={(r1 == 0).sum()},{(r2 == 0).sum()} minrho={min(r1[r1 > 0].min(), r2[r2 > 0].min()):.2e}")
    x, r1, r2 = ref.x, ref.rho1, ref.rho2
