"""Measure the FP64 GEMM roofline denominator on this B200.

cuBLAS DGEMM through torch.matmul on float64, 8192^3 (2*N^3 flops): best of 10
(burst) and back-to-back for 4 s (sustained), CUDA-event timed, mirroring how
MEASURED_PEAKS.json measured bf16. Prints one JSON line.
"""
import json
import time

import torch


def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty(n, n, dtype=torch.float64, device="cuda")
    flops = 2.0 * n ** 3
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    burst = flops / best / 1e12
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_end = time.time() + 4.0
    iters = 0
    e0.record()
    while time.time() < t_end:
        torch.matmul(a, b, out=c)
        iters += 1
        if iters % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    sustained = flops * iters / (e0.elapsed_time(e1) * 1e-3) / 1e12
    print(json.dumps({"fp64_dgemm_tflops_burst": round(burst, 2),
                      "fp64_dgemm_tflops_sustained": round(sustained, 2),
                      "n": n, "iters_sustained": iters}))


if __name__ == "__main__":
    main()
