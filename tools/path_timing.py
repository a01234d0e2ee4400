"""E/M-kernel and iteration time per path and config (CUDA events inside libsrmra via srmra_profile)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402

names = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c0", "c1", "c2", "c3"]
paths = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fft", "gemm", "direct"]
for name in names:
    p = synth.make_config(name)
    units = p.N * p.L_high ** 2
    for path in paths:
        try:
            with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path=path) as ctx:
                ctx.em_iter(2)
                ctx.profile(True)
                n_it = 5 if units < 5e9 else 2
                ctx.em_iter(n_it)
                em, tot, n = ctx.profile_read()
                print(f"{name} {path:6s}: E/M {em / n:9.3f} ms  iteration {tot / n:9.3f} ms  "
                      f"{units / (tot / n / 1e3):.3e} obs*shift/s  launches/iter {ctx.launches_per_iter()}", flush=True)
        except srm.SrmraError as e:
            print(f"{name} {path:6s}: {e}", flush=True)
