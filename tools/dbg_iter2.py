"""Debug: c1 geometry N=601: one iteration from the oracle's theta_1 (fresh context) vs the oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle
import paper_2204_04754_b200 as srm

for N in (601, 1000):
    p = synth.make_config("c1", N=N)
    r1 = oracle.em_iter(p.y, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=True)
    x1 = r1.x.astype(np.float32)
    for path in ("fft", "direct", "gemm"):
        ref = oracle.em_iter(p.y, p.L_low, p.K, p.sigma, x1, r1.rho1, r1.rho2, project=True)
        with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, x1, r1.rho1, r1.rho2, path=path) as ctx:
            ctx.em_iter(1)
            x, ra, rb, ll, it = ctx.get_estimate()
            b, cm, m1, m2 = ctx.stats()
            llo = ctx.obs_loglik()
        K = p.K
        be = np.abs(b - ref.b) / np.abs(ref.b).max()
        cls = [[be[a::K, c::K].max() for c in range(K)] for a in range(K)]
        cm_ref = np.array([[ref.colsum[a::K, c::K].sum() for c in range(K)] for a in range(K)])
        print(N, path, f"x {np.abs(x - ref.x).max() / np.abs(ref.x).max():.2e} rho {np.abs(ra - ref.rho1).max() / ref.rho1.max():.2e}"
              f" ll {abs(ll - ref.loglik) / abs(ref.loglik):.2e} llobs {np.abs(llo - ref.ll_obs).max():.2e}"
              f" b per class {np.array(cls).round(6).tolist()} cm err {np.abs(cm - cm_ref).max():.2e}", flush=True)
        if path == "fft":
            worst = np.unravel_index(np.argmax(be), be.shape)
            print("  worst b pixel", worst, b[worst], ref.b[worst], "A", ref.A[worst], flush=True)
            e = np.abs(llo - ref.ll_obs)
            print("  worst obs", np.argsort(-e)[:5], e[np.argsort(-e)[:5]], flush=True)
