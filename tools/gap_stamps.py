"""Device-clock gaps of one FFT iteration: E/M kernel (first-CTA start .. last-CTA end, from the profiling
stamps) and the tail kernel (earliest block start .. latest block end, SRMRA_TAIL_STAMPS)."""
import os
import sys

os.environ["SRMRA_TAIL_STAMPS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
p = synth.make_config(name)
with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
    ctx.em_iter(3)
    for _ in range(4):
        ctx.profile(True)
        ctx.em_iter(20)
        em20, it20, n = ctx.profile_read()
        srm.srmra_debug_timestamps(ctx.handle)  # re-arm the tail extremes
        ctx.em_iter(1)
        st = srm.srmra_debug_timestamps(ctx.handle).astype(np.int64)
        em, it = em20 / n, it20 / n
        print(f"{name}: iteration (E/M start spacing) {it * 1e3:.1f} us = E/M {em * 1e3:.1f} + tail span "
              f"{(st[7] - st[6]) / 1e3:.1f} + launch gaps {(it - em) * 1e3 - (st[7] - st[6]) / 1e3:.1f}")
        print(f"    tail span {(st[7] - st[6]) / 1e3:.1f} us "
              f"(phases: reduce {(st[1] - st[0]) / 1e3:.1f}, fold+update {(st[4] - st[1]) / 1e3:.1f}, "
              f"prep {(st[5] - st[4]) / 1e3:.1f})")
        for k, nm in ((2, "fold"), (3, "prep")):
            print(f"    slowest {nm} block: {(int(st[k]) >> 12) / 1e3:.1f} us of item work (last item {int(st[k]) & 0xfff})")
