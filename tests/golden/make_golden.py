"""Write the oracle outputs used by the full-size GPU parity tests.

Calls only oracle/ (and the shared input generator synth/).  Output per config:
tests/golden/<cfg>_oracle.npz with x, rho1, rho2 after `iters` iterations (proj_every=1, the
north_star parity setting), the LL trace, and, for the first iteration, the per-observation
log-likelihood terms of a fixed sample of observations.

    python tests/golden/make_golden.py c1 c3 c2
    python tests/golden/make_golden.py --dense c4

--dense uses oracle.dense.em_iter_dense (the same iteration as the dense float64 contraction
S = Y T(x)^T, Z = W^T Y through BLAS; pinned to the brute-force oracle.em_iter in
tests/test_oracle_pins.py): the brute-force loop would take ~30 h at configs[4].
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sample_idx(N, k=64):
    return np.unique(np.linspace(0, N - 1, k).astype(np.int64))


def main(names, dense=False):
    if dense:
        from oracle.dense import em_iter_dense
    for name in names:
        p = synth.make_config(name)
        t0 = time.time()
        x, r1, r2 = p.x0.astype(np.float64), p.rho1_0, p.rho2_0
        trace = []
        ll_obs0 = None
        for t in range(p.iters):
            if dense:
                r = em_iter_dense(p.y, p.L_low, p.K, p.sigma, x, r1, r2, project=True, verbose=True)
            else:
                r = oracle.em_iter(p.y, p.L_low, p.K, p.sigma, x, r1, r2, project=True)
            if t == 0:
                ll_obs0 = r.ll_obs[sample_idx(p.N)]
            x, r1, r2 = r.x, r.rho1, r.rho2
            trace.append(r.loglik)
            print(f"{name} iter {t}: LL={r.loglik:.10e}  ({time.time() - t0:.1f}s)", flush=True)
        np.savez(os.path.join(OUT, f"{name}_oracle.npz"), x=x, rho1=r1, rho2=r2, trace=np.array(trace),
                 ll_obs0_idx=sample_idx(p.N), ll_obs0=ll_obs0, iters=p.iters,
                 threads=oracle.max_threads(), seconds=time.time() - t0,
                 form="dense" if dense else "brute_force")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if a != "--dense"]
    main(args or ["c1"], dense="--dense" in sys.argv[1:])
