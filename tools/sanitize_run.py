"""Small invocations of every E/M path for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
c0 (FFT, direct, GEMM), randomised tiny shapes (K = 1, 2, 3, 4), the c1 and c3 geometries (FFT with TMEM
accumulators, several observations per CTA), c4 geometry (L_low = 128 cluster kernel), the joint prior and
the Algorithm 2 driver.  Usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2204_04754_b200 as srm
import synth


def run(p, path, iters=2, **kw):
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path=path, **kw) as ctx:
        ctx.em_iter(iters)
        x, *_ = ctx.get_estimate()
        assert np.all(np.isfinite(x))
    print("ok", p.name, path, kw, flush=True)


cases = [synth.make_config("c0"), synth.make_random(4, 3, 13, 0.4, 1, rho_zeros=1), synth.make_random(8, 2, 9, 0.3, 2),
         synth.make_random(2, 4, 7, 0.5, 3), synth.make_random(8, 1, 5, 0.5, 4)]
for p in cases:
    for path in ("fft", "direct", "gemm"):
        try:
            run(p, path)
        except srm.SrmraError as e:
            if e.code != srm.SRMRA_ERR_UNSUPPORTED:
                raise
run(synth.make_config("c1", N=300), "fft", grid_cap=3)
run(synth.make_config("c3", N=40), "fft", grid_cap=2)
run(synth.make_config("c4", N=6), "fft", iters=1, grid_cap=2)
p = synth.make_config("c0")
L = p.L_high
pr = np.full((L, L), 1.0 / (L * L))
with srm.Context(p.y, L, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
    ctx.set_joint_rho(pr)
    ctx.em_iter(2)
    ctx.load(p.y, p.x0, p.rho1_0, p.rho2_0)
    ctx.run(10, 1e-9)
    ctx.get_estimate()
print("all ok")
