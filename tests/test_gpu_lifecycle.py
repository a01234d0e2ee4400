"""Context lifecycle: repeated create / use / free of contexts exercising every subsystem (EM on all
paths, the joint prior, moments, the moment objective, the generator, profiling) leaves the device's
free memory where the first round left it (no leaked buffers; the stream-ordered pool is warmed by the
first round)."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def srm():
    import paper_2204_04754_b200 as m
    return m


def _round(srm, p, pr):
    for path in ("fft", "gemm", "direct"):
        with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path=path) as ctx:
            ctx.em_iter(2)
            ctx.set_joint_rho(pr)
            ctx.em_iter(1)
            ctx.moments()
            ctx.mom_set_moments()
            ctx.mom_objective(p.x0, p.rho1_0, p.rho2_0)
            ctx.mom_run(3, F=2)
            ctx.generate(p.x_true.astype(np.float32), p.rho1_true, p.rho2_true, 7, p.x0, p.rho1_0, p.rho2_0)
            ctx.profile(True)
            ctx.em_iter(2)
            ctx.profile_read()
            ctx.profile(False)
            ctx.relative_error(p.x_true.astype(np.float32))


def test_repeated_contexts_do_not_leak(srm):
    import torch
    p = synth.make_config("c0")
    pr = np.random.default_rng(3).dirichlet(np.ones(p.L_high ** 2)).reshape(p.L_high, p.L_high)
    _round(srm, p, pr)
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    for _ in range(8):
        _round(srm, p, pr)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    print(f"free memory after 1 round {free0 / 2**20:.1f} MiB, after 9 rounds {free1 / 2**20:.1f} MiB")
    assert free1 >= free0 - (16 << 20)
