"""NEXT-2 timing: srmra_moments (tensor-core empirical moments), srmra_mom_set_moments (Fourier transform of
the data moments), one objective + gradient evaluation, and Algorithm 1 steps, at the configs' shapes.
Wall-clock around synchronising C-ABI calls (each call synchronises), median of repeats.
Usage: python tools/mom_timing.py [c1 c2 c3]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_04754_b200 as srm  # noqa: E402
import synth  # noqa: E402


def med(fn, reps):
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return float(np.median(ts)) * 1e3


def main(names):
    out = {}
    for name in names:
        p = synth.make_config(name)
        N = p.y.shape[0]
        with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
            ctx.moments()  # warm-up (tensor maps, attributes)
            t_mom = med(ctx.moments, 5)
            ctx.mom_set_moments()
            t_set = med(ctx.mom_set_moments, 3)
            x = p.x0.astype(np.float64)
            ctx.mom_objective(x, p.rho1_0, p.rho2_0)
            t_obj = med(lambda: ctx.mom_objective(x, p.rho1_0, p.rho2_0), 10)
            t = time.perf_counter()
            f, steps = ctx.mom_run(50, F=5)
            t_run = (time.perf_counter() - t) * 1e3
        Ll2 = p.L_low ** 2
        gemm_flop = 2.0 * 3 * (Ll2 + 16) ** 2 * N / 2  # symmetric: upper tiles, 3 tf32 MMAs per product
        out[name] = {"L_high": p.L_high, "L_low": p.L_low, "K": p.K, "N": N,
                     "moments_ms": t_mom, "moments_tflops_effective": gemm_flop / (t_mom * 1e-3) / 1e12,
                     "set_moments_ms": t_set, "objective_ms": t_obj,
                     "alg1_50_steps_ms": t_run, "alg1_steps": steps, "alg1_f": f}
        print(name, json.dumps(out[name]), flush=True)
    return out


if __name__ == "__main__":
    res = main(sys.argv[1:] or ["c1", "c2", "c3"])
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/mom_timing.json", "w") as fh:
        json.dump(res, fh, indent=1)
