"""Time the FFT E/M kernel for a config under different launch settings (env overrides read at
srmra_init): SRMRA_FFT_GROUPS (groups per CTA) and SRMRA_FFT_XS (Xhat in shared memory)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
p = synth.make_config(name)
settings = [(g, xs) for xs in ("0", "1") for g in ("1", "2", "3", "4", "5", "15")]
for g, xs in settings:
    os.environ["SRMRA_FFT_GROUPS"] = g
    os.environ["SRMRA_FFT_XS"] = xs
    try:
        with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
            ctx.em_iter(3)
            ctx.profile(True)
            ctx.em_iter(10)
            em, tot, n = ctx.profile_read()
            print(f"{name} groups<={g} xs={xs}: em {em / n * 1e3:8.1f} us  iter {tot / n * 1e3:8.1f} us  "
                  f"units/s {p.N * p.L_high**2 / (em / n / 1e3):.3e}", flush=True)
    except srm.SrmraError as e:
        print(name, g, xs, "error", e)
