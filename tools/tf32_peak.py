"""Measure the dense TF32 tensor peak on this GPU the way MEASURED_PEAKS.json
measures bf16: torch.matmul 8192^3 with TF32 enabled, best of 10 (burst) and a
4-second back-to-back loop (sustained).  Prints one JSON line."""
import json
import time

import torch


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    n = 8192
    a = torch.randn(n, n, device="cuda", dtype=torch.float32)
    b = torch.randn(n, n, device="cuda", dtype=torch.float32)
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 0.0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(10):
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    t0 = time.time()
    k = 0
    e0.record()
    while time.time() - t0 < 4.0:
        a @ b
        k += 1
        if k % 20 == 0:
            torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    sus = 2 * n ** 3 * k / (e0.elapsed_time(e1) / 1e3) / 1e12
    print(json.dumps({"tf32_tflops": round(best, 1), "tf32_tflops_sustained": round(sus, 1),
                      "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS TF32 tensor cores)"}))


if __name__ == "__main__":
    main()
