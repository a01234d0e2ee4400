"""Multi-process host logic on CPU (gloo, world size 2): observation sharding, the NCCL-id broadcast,
and the decompositions the library's all-reduces rely on: summing the shard statistics
of the oracle over ranks and finalising gives the full-data iteration; likewise the raw moment sums
(NEXT-2), the per-shift posterior mass of the joint prior (NEXT-3), and the counter-based generator's
shards (NEXT-4) reproduce the one-rank results."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2204_04754_b200.shard import broadcast_nccl_id, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        import oracle
        import synth
        # 1. NCCL-id broadcast (the id maker is only called on rank 0)
        nid = broadcast_nccl_id(lambda: bytes(range(128)))
        assert nid == bytes(range(128))
        # 2. shard statistics -> all-reduce -> finalize == full-data iteration
        p = synth.make_random(4, 2, 37, 0.4, 3, rho_zeros=1)
        lo, hi = shard_bounds(p.N, world, rank)
        r = oracle.em_iter(p.y[lo:hi], p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=False, tau=0.0)
        stats = torch.from_numpy(np.concatenate([r.b.ravel(), r.A.ravel(), r.colsum.ravel(), [r.loglik]]))
        dist.all_reduce(stats)
        L2 = p.L_high ** 2
        b, A, cs, ll = stats[:L2].numpy(), stats[L2:2 * L2].numpy(), stats[2 * L2:3 * L2].numpy(), float(stats[-1])
        x = np.where(A > 0, b / np.where(A > 0, A, 1), p.x0.astype(np.float64).ravel()).reshape(p.L_high, -1)
        cs = cs.reshape(p.L_high, p.L_high)
        # 3. NEXT-2: raw moment sums of the shards -> all-reduce -> / N == the full-data moments
        m1, m2 = oracle.empirical_moments(p.y[lo:hi])
        raw = torch.from_numpy(np.concatenate([m1 * (hi - lo), (m2 * (hi - lo)).ravel()]))
        dist.all_reduce(raw)
        # 4. NEXT-3: per-shift posterior mass of the shards -> all-reduce -> joint rho'
        pr = np.random.default_rng(5).dirichlet(np.ones(p.L_high ** 2)).reshape(p.L_high, p.L_high)
        rj = oracle.em_iter_joint(p.y[lo:hi], p.L_low, p.K, p.sigma, p.x0, pr, project=False, tau=0.0)
        mass = torch.from_numpy(np.ascontiguousarray(rj.colsum, dtype=np.float64).ravel())
        dist.all_reduce(mass)
        # 5. NEXT-4: the counter-based generator's shard [lo, hi) of the global index range
        from synth import philox
        ys, ss = philox.generate(p.x_true, p.rho1_true, p.rho2_true, p.K, p.sigma, hi - lo, seed=99, first_index=lo)
        out[rank] = (x, cs.sum(1) / cs.sum(), cs.sum(0) / cs.sum(), ll, raw.numpy() / p.N,
                     mass.numpy() / mass.sum().item(), ys, ss)
    finally:
        dist.destroy_process_group()


def test_shard_bounds_cover_and_balance():
    for n in (0, 1, 7, 10, 10_000, 100_001):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)


def test_gloo_world2_statistics_allreduce(oracle_mod):
    import synth
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    p = synth.make_random(4, 2, 37, 0.4, 3, rho_zeros=1)
    full = oracle_mod.em_iter(p.y, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, project=False, tau=0.0)
    M1, M2 = oracle_mod.empirical_moments(p.y)
    pr = np.random.default_rng(5).dirichlet(np.ones(p.L_high ** 2)).reshape(p.L_high, p.L_high)
    fj = oracle_mod.em_iter_joint(p.y, p.L_low, p.K, p.sigma, p.x0, pr, project=False, tau=0.0)
    from synth import philox
    yf, sf = philox.generate(p.x_true, p.rho1_true, p.rho2_true, p.K, p.sigma, p.N, seed=99)
    for rank in range(world):
        x, r1, r2, ll, mom, rj, _, _ = out[rank]
        np.testing.assert_allclose(x, full.x, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(r1, full.rho1, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(r2, full.rho2, rtol=1e-12, atol=1e-15)
        assert abs(ll - full.loglik) <= 1e-12 * abs(full.loglik)
        np.testing.assert_allclose(mom[:M1.size], M1, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(mom[M1.size:].reshape(M2.shape), M2, rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(rj.reshape(pr.shape), fj.rho, rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(np.concatenate([out[0][6], out[1][6]]), yf)
    np.testing.assert_array_equal(np.concatenate([out[0][7], out[1][7]]), sf)
