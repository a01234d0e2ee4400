"""Print the FFT tail-kernel phase durations (SRMRA_TAIL_STAMPS debug hook) for a config."""
import os
import sys
import time

os.environ["SRMRA_TAIL_STAMPS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
p = synth.make_config(name)
with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
    for it in range(5):
        srm.srmra_debug_timestamps(ctx.handle)  # re-arms the cross-block extremes
        ctx.em_iter(1)
        st = srm.srmra_debug_timestamps(ctx.handle).astype(np.int64)
        names = ["reduce", "fold+update", "project+prep"]
        bounds = [(0, 1), (1, 4), (4, 5)]
        d = [(st[b] - st[a_]) / 1e3 if st[b] and st[a_] else 0.0 for a_, b in bounds]
        print(name, "tail phases (us):", ", ".join(f"{n}={v:.1f}" for n, v in zip(names, d)),
              f"total={(st[5] - st[0]) / 1e3:.1f}", f"first-block-start..block0 {(st[0] - st[6]) / 1e3:.1f}",
              f"block0-end..last-block-end {(st[7] - st[5]) / 1e3:.1f}")
    em, tot, n = 0, 0, 0
    ctx.profile(True)
    ctx.em_iter(20)
    em, tot, n = ctx.profile_read()
    print(name, f"em kernel {em / n * 1e3:.1f} us, iteration {tot / n * 1e3:.1f} us")
