"""Host-side multi-GPU plumbing (no compute): contiguous observation shards and the NCCL-id
broadcast over a torch.distributed process group.  The data-path collective itself
(one fp64 all-reduce of the sufficient statistics per iteration) runs inside libsrmra.so."""
from __future__ import annotations


def shard_bounds(n_global: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block [lo, hi) of observations owned by `rank`; sizes differ by at most one."""
    if world < 1 or not 0 <= rank < world or n_global < 0:
        raise ValueError("bad shard request")
    q, r = divmod(n_global, world)
    lo = rank * q + min(rank, r)
    hi = lo + q + (1 if rank < r else 0)
    return lo, hi


def broadcast_nccl_id(make_id, src: int = 0, group=None) -> bytes:
    """Rank `src` calls make_id() (e.g. paper_2204_04754_b200.srmra_nccl_unique_id) and every rank of
    the torch.distributed group receives the same 128-byte id."""
    import torch.distributed as dist
    obj = [make_id() if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src, group=group)
    nid = obj[0]
    if not isinstance(nid, (bytes, bytearray)) or len(nid) != 128:
        raise RuntimeError("bad NCCL unique id")
    return bytes(nid)
