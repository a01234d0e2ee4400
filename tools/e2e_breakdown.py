"""Where the end-to-end job time goes (bench.py's e2e step): load (H2D + init kernels), iterations,
estimate read-back; host timers with a device sync after each part."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
p = synth.make_config(name)
y_pin = torch.from_numpy(p.y).pin_memory().numpy()
with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
    ctx.em_iter(p.iters)
    ctx.get_estimate()
    for rep in range(3):
        t0 = time.perf_counter()
        ctx.load(y_pin, p.x0, p.rho1_0, p.rho2_0)  # synchronises
        t1 = time.perf_counter()
        ctx.em_iter(p.iters)
        ctx.get_estimate()
        t2 = time.perf_counter()
        print(f"{name}: load {1e3 * (t1 - t0):.3f} ms, {p.iters} iterations + estimate {1e3 * (t2 - t1):.3f} ms, "
              f"job {1e3 * (t2 - t0):.3f} ms, y {p.y.nbytes / 1e6:.1f} MB -> {p.y.nbytes / (t1 - t0) / 1e9:.1f} GB/s load")
