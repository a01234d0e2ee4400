"""Debug: c1 geometry, 2 iterations, world 2 through the exchange hook vs single rank (grid_cap on/off)."""
import os, socket, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, oracle


def errs(g, x, r1, r2):
    return (np.abs(g[0] - x).max() / np.abs(x).max(), max(np.abs(g[1] - r1).max() / r1.max(), np.abs(g[2] - r2).max() / r2.max()))


def single(p, cap, iters):
    import paper_2204_04754_b200 as srm
    out = []
    with srm.Context(p.y, p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path="fft", grid_cap=cap) as ctx:
        for _ in range(iters):
            ctx.em_iter(1)
            out.append(ctx.get_estimate()[:3])
    return out


class _DevBuf:
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False), "version": 3, "strides": None}


def worker(rank, world, port, N, cap, iters, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    import torch, torch.distributed as dist
    import paper_2204_04754_b200 as srm
    from paper_2204_04754_b200.shard import shard_bounds
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)

    def ex(ptr, n, st):
        torch.cuda.ExternalStream(st).synchronize()
        t = torch.as_tensor(_DevBuf(ptr, n), device="cuda")
        h = t.cpu(); dist.all_reduce(h); t.copy_(h); torch.cuda.synchronize()
        return 0
    p = synth.make_config("c1", N=N)
    lo, hi = shard_bounds(p.N, world, rank)
    res = []
    with srm.Context(p.y[lo:hi], p.L_high, p.L_low, p.K, p.sigma, p.x0, p.rho1_0, p.rho2_0, path="fft", rank=rank,
                     world=world, allreduce=ex, grid_cap=cap) as ctx:
        for _ in range(iters):
            ctx.em_iter(1)
            res.append(ctx.get_estimate()[:3])
    out[rank] = res
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    N, iters = 601, 3
    p = synth.make_config("c1", N=N)
    ref, x, r1, r2 = [], p.x0, p.rho1_0, p.rho2_0
    for _ in range(iters):
        r = oracle.em_iter(p.y, p.L_low, p.K, p.sigma, x, r1, r2, project=True)
        x, r1, r2 = r.x, r.rho1, r.rho2
        ref.append((x, r1, r2))
    for cap in (0, 3):
        s = single(p, cap, iters)
        print("single cap", cap, [f"{a:.2e}/{b:.2e}" for a, b in (errs(s[t], *ref[t]) for t in range(iters))], flush=True)
    for cap in (0, 3):
        mgr = mp.Manager(); out = mgr.dict()
        sk = socket.socket(); sk.bind(("127.0.0.1", 0)); port = sk.getsockname()[1]; sk.close()
        mp.spawn(worker, args=(2, port, N, cap, iters, out), nprocs=2, join=True)
        for rank in range(2):
            print("world2 cap", cap, "rank", rank, [f"{a:.2e}/{b:.2e}" for a, b in (errs(out[rank][t], *ref[t]) for t in range(iters))], flush=True)
