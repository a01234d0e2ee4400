import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, synth
from synth import philox
import paper_2204_04754_b200 as srm
p = synth.make_config("c1", N=8); N=3001; first=12345; seed=0xDEADBEEF12345 + N
with srm.Context(None, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, n_local=N) as ctx:
    sh = ctx.generate(p.x_true.astype(np.float32), p.rho1_true, p.rho2_true, seed, p.x0, p.rho1_0, p.rho2_0, first_index=first, want_shifts=True)
    y = ctx.observations()
yr, shr = philox.generate(p.x_true.astype(np.float32), p.rho1_true, p.rho2_true, p.K, p.sigma, N, seed, first)
err = np.abs(y.astype(np.float64)-yr)
idx = np.unravel_index(np.argmax(err), err.shape)
print("max", err.max(), idx, y[idx], yr[idx])
i, n1, n2 = idx; pix = n1*32+n2; b = pix//4; e = pix%4
j = np.uint64(first+i)
r = philox.philox4x32_10(j & np.uint64(0xffffffff), j >> np.uint64(32), np.uint64(1+b), np.uint64(0), seed & 0xffffffff, seed >> 32)
V = [((int(v) >> 9) + 0.5) * 2.0**-23 for v in r]
print("e", e, "V", V)
zs = sorted(err.ravel())[-10:]; print(zs)
print("frac over 1e-6:", (err > 1e-6).mean())
