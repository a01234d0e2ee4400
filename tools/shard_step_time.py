"""Per-rank compute time of a strong-scaled iteration, measured on ONE GPU: for G in 1, 2, 4, 8 the first shard of
shard.shard_bounds(N, G) runs alone as a world-1 context (E/M kernel + full tail from the kernels' own globaltimer
stamps, srmra_profile).  The exchange (one float64 all-reduce of the statistics, NCCL) and the split of the tail
around it are NOT in these numbers: T_1 / (G T_G) from this table is the compute-side UPPER bound of the strong-
scaling efficiency, not a measured scaling curve (that needs a multi-GPU node: bench.py --gpus N).
Usage: python tools/shard_step_time.py c3 c4"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2204_04754_b200 as srm  # noqa: E402
from paper_2204_04754_b200 import shard  # noqa: E402
import synth  # noqa: E402

for name in sys.argv[1:] or ["c3"]:
    p = synth.make_config(name)
    t1 = None
    for G in (1, 2, 4, 8):
        lo, hi = shard.shard_bounds(p.N, G, 0)
        with srm.Context(p.y[lo:hi], p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0) as ctx:
            ctx.em_iter(3)
            ctx.profile(True)
            ctx.em_iter(20)
            em, tot, n = ctx.profile_read()
        em, tot = em / n * 1e3, tot / n * 1e3
        t1 = t1 or tot
        print(f"{name} G={G} n_local={hi - lo}: E/M {em:9.1f} us  iteration {tot:9.1f} us  "
              f"compute-side efficiency bound T1/(G T_G) = {t1 / (G * tot):.3f}", flush=True)
