"""Host->device bandwidth of the e2e load: one pinned 41 MB copy vs chunks (CUDA events)."""
import sys
import torch

n = int(sys.argv[1]) if len(sys.argv) > 1 else 40_960_000
h = torch.empty(n // 4, dtype=torch.float32).pin_memory()
d = torch.empty(n // 4, dtype=torch.float32, device="cuda")
for chunk_mb in (0, 2, 4, 8, 16):
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        if chunk_mb == 0:
            d.copy_(h, non_blocking=True)
        else:
            c = chunk_mb * (1 << 20) // 4
            for o in range(0, h.numel(), c):
                d[o:o + c].copy_(h[o:o + c], non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"chunk {chunk_mb or 'whole'} MB: {best:.3f} ms, {n / best / 1e6:.1f} GB/s")
