"""a6 (the exchange) through the library: two processes (gloo, world size 2) on ONE GPU, each holding a
contiguous shard of the observations, run srmra_em_iter with world = 2.  The sums over i of eq:x_EM,
eq:rho_EM and eq:likelihood_EM go through the library's own world > 1
iteration — FFT path: E/M kernel, reduce-only tail, exchange, fold / finalize / projection / prep tail;
GEMM / direct paths: E/M, pack, exchange (+ the per-shift posterior mass with a joint prior), finalize —
with the exchange provider hook (srmra_options.allreduce) doing the sum over gloo on the host, since NCCL
cannot put two ranks on one GPU.  Both ranks must reproduce the oracle's iteration on the FULL data."""
import os
import socket

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

X_TOL, LL_TOL, RHO_TOL = 1e-4, 1e-6, 1e-4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _DevBuf:
    """__cuda_array_interface__ view of a library-owned float64 device buffer."""

    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def _problem(spec):
    kind, a = spec
    if kind == "cfg":
        return synth.make_config(a[0], N=a[1])
    return synth.make_random(*a[:5], rho_zeros=a[5])


def _joint_prior(L, seed):
    rng = np.random.default_rng(seed)
    pr = rng.uniform(0.05, 1.0, (L, L)) ** 3
    pr.reshape(-1)[rng.choice(L * L, size=3, replace=False)] = 0.0
    return pr / pr.sum()


def _worker(rank, world, port, specs, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    import paper_2204_04754_b200 as srm
    from paper_2204_04754_b200.shard import shard_bounds
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    calls = [0]

    def exchange(ptr, n, stream):
        torch.cuda.ExternalStream(stream).synchronize()   # this rank's partial sums are complete
        t = torch.as_tensor(_DevBuf(ptr, n), device="cuda")
        h = t.cpu()
        dist.all_reduce(h)
        t.copy_(h)
        torch.cuda.synchronize()                           # visible to the library's next launches
        calls[0] += 1
        return 0

    try:
        res = {}
        for key, (spec, path, iters, joint) in specs.items():
            p = _problem(spec)
            lo, hi = shard_bounds(p.N, world, rank)
            try:
                ctx = srm.Context(p.y[lo:hi], p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path=path,
                                  rank=rank, world=world, allreduce=exchange, grid_cap=3 if path == "fft" else 0)
            except srm.SrmraError as e:
                assert e.code == srm.SRMRA_ERR_UNSUPPORTED, e
                res[key] = None
                continue
            with ctx:
                c0 = calls[0]
                if joint:
                    ctx.set_joint_rho(_joint_prior(p.L_high, 17))
                ctx.em_iter(iters)
                x, r1, r2, ll, it = ctx.get_estimate()
                res[key] = dict(x=x, rho1=r1, rho2=r2, trace=ctx.loglik_trace(), it=it, calls=calls[0] - c0,
                                b=ctx.stats()[0], rhoj=ctx.joint_rho() if joint else None)
        out[rank] = res
    finally:
        dist.destroy_process_group()


SPECS = {
    # name: (problem, path, iterations, joint prior)
    # (N = 601 is avoided on purpose: its second iteration has two classes with posterior mass ~1e-5, whose
    # pixels x = b / A rest on single low-probability weights that no float32 E-step resolves to 1e-4 —
    # DESIGN.md §6.5; every config and N >= 1000 keeps all class masses >= 10)
    "c1_fft": (("cfg", ("c1", 2001)), "fft", 2, False),
    "c3_fft": (("cfg", ("c3", 301)), "fft", 1, False),
    "c4_fft": (("cfg", ("c4", 9)), "fft", 1, False),
    "r8_fft_joint": (("rand", (8, 2, 33, 0.3, 2, 0)), "fft", 2, True),
    "r8_direct": (("rand", (8, 2, 33, 0.3, 2, 1)), "direct", 2, False),
    "r8_direct_joint": (("rand", (8, 2, 33, 0.3, 2, 0)), "direct", 2, True),
    "r4K4_gemm": (("rand", (4, 4, 31, 0.25, 4, 0)), "gemm", 2, False),
    "r4K4_gemm_joint": (("rand", (4, 4, 31, 0.25, 4, 0)), "gemm", 2, True),
    "c1_gemm": (("cfg", ("c1", 301)), "gemm", 1, False),
}


@pytest.fixture(scope="module")
def world2():
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), SPECS, out), nprocs=2, join=True)
    return dict(out)


@pytest.mark.parametrize("key", list(SPECS))
def test_world2_exchange_matches_full_data_oracle(world2, oracle_mod, key):
    spec, path, iters, joint = SPECS[key]
    r0, r1 = world2[0][key], world2[1][key]
    if r0 is None:
        pytest.skip(f"path {path} does not support this shape")
    p = _problem(spec)
    x, rho1, rho2 = p.x0.astype(np.float64), p.rho1_0, p.rho2_0
    rho = _joint_prior(p.L_high, 17) if joint else None
    trace = []
    for _ in range(iters):
        if joint:
            r = oracle_mod.em_iter_joint(p.y, p.L_low, p.K, p.sigma, x, rho, project=True)
            rho = r.rho
        else:
            r = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, x, rho1, rho2, project=True)
        x, rho1, rho2 = r.x, r.rho1, r.rho2
        trace.append(r.loglik)
    for rank, g in ((0, r0), (1, r1)):
        xe = np.abs(g["x"] - x).max() / np.abs(x).max()
        re = max(np.abs(g["rho1"] - rho1).max() / rho1.max(), np.abs(g["rho2"] - rho2).max() / rho2.max())
        le = np.max(np.abs(g["trace"] - np.asarray(trace)) / np.abs(np.asarray(trace)))
        print(f"{key} rank {rank}: x_err={xe:.2e} rho_err={re:.2e} ll_err={le:.2e} exchanges={g['calls']}")
        assert g["it"] == iters
        assert xe <= X_TOL and re <= RHO_TOL and le <= LL_TOL, (key, rank, xe, re, le)
        if joint:
            assert np.abs(g["rhoj"] - rho).max() <= RHO_TOL * rho.max(), key
            assert np.all(g["rhoj"][_joint_prior(p.L_high, 17) == 0] == 0.0)
        # one exchange per iteration (FFT with a joint prior: the accumulators and the per-shift mass)
        assert g["calls"] == iters * (2 if (joint and path == "fft") else 1), g["calls"]
    # both ranks hold the same (all-reduced) estimate
    np.testing.assert_array_equal(r0["x"], r1["x"])
    np.testing.assert_array_equal(r0["b"], r1["b"])


def test_exchange_provider_failure_is_reported():
    """A failing exchange provider fails the call with SRMRA_ERR_NCCL (at init: the global-N sum; later: the
    iteration's statistics sum) and leaves the context failed (every later call returns STATE)."""
    import paper_2204_04754_b200 as srm
    p = synth.make_random(8, 2, 9, 0.3, 2)
    args = (p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0)
    with pytest.raises(srm.SrmraError) as ei:
        srm.Context(*args, world=2, rank=0, allreduce=lambda ptr, n, st: 1)
    assert ei.value.code == srm.SRMRA_ERR_NCCL
    calls = [0]

    def flaky(ptr, n, st):  # the init-time N sum succeeds (a one-rank "sum" is the identity), then fail
        calls[0] += 1
        return 0 if calls[0] == 1 else 1
    with srm.Context(*args, world=2, rank=0, allreduce=flaky) as ctx:
        with pytest.raises(srm.SrmraError) as ei:
            ctx.em_iter(1)
        assert ei.value.code == srm.SRMRA_ERR_NCCL
        with pytest.raises(srm.SrmraError) as ei:
            ctx.get_estimate()
        assert ei.value.code == srm.SRMRA_ERR_STATE
