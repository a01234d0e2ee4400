"""Dense TF32 tensor-core peak as cuBLAS delivers it on this GPU (the GEMM path's roofline denominator, SURVEY
§8(d)): torch.matmul of float32 8192^3 with TF32 allowed, best of 10 (burst) and back to back for 3 s
(sustained); bf16 alongside for the ratio.  Prints one JSON object."""
import json
import time

import torch


def rate(dtype, tf32, n=8192, reps=10, seconds=3.0):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    cnt, t0 = 0, time.time()
    e0.record()
    while time.time() - t0 < seconds:
        a @ b
        cnt += 1
    e1.record()
    torch.cuda.synchronize()
    sus = e0.elapsed_time(e1) / cnt
    f = 2.0 * n ** 3
    return f / (best * 1e-3) / 1e12, f / (sus * 1e-3) / 1e12


if __name__ == "__main__":
    t_b, t_s = rate(torch.float32, True)
    b_b, b_s = rate(torch.bfloat16, False)
    print(json.dumps({"gpu": torch.cuda.get_device_name(), "tf32_tflops_burst": t_b, "tf32_tflops_sustained": t_s,
                      "bf16_tflops_burst": b_b, "bf16_tflops_sustained": b_s, "tf32_over_bf16": t_b / b_b,
                      "how": "torch.matmul 8192^3, float32 with allow_tf32 (cuBLAS TF32 tensor cores) and bfloat16; "
                             "best of 10 (burst), back to back for 3 s (sustained)"}))
