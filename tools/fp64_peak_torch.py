"""Measure the FP64 GEMM ceiling on this B200 with cuBLAS DGEMM (torch float64
matmul at 8192^3), best-of-10 (burst) and back-to-back for ~4 s (sustained),
plus nvidia-smi clocks during the sustained loop. Writes one JSON line.

Measurement tool only; not part of the product path.
"""
import json
import subprocess
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
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    smi = subprocess.Popen(
        ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
         "--format=csv,noheader,nounits", "-lms", "200"],
        stdout=subprocess.PIPE, text=True)
    reps = 0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.time()
    while time.time() - t0 < 4.0:
        for _ in range(10):
            torch.matmul(a, b, out=c)
        reps += 10
        torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    sustained_ms = e0.elapsed_time(e1) / reps
    smi.terminate()
    lines = smi.communicate()[0].strip().splitlines()
    clocks = [float(l.split(",")[0]) for l in lines if l.strip()]
    clocks.sort()
    print(json.dumps({
        "what": "cuBLAS DGEMM via torch.matmul float64 8192^3",
        "fp64_tflops": flops / (best * 1e-3) / 1e12,
        "fp64_tflops_sustained": flops / (sustained_ms * 1e-3) / 1e12,
        "sm_mhz_median_sustained": clocks[len(clocks) // 2] if clocks else None,
        "smi_samples": lines[:5] + lines[-5:],
    }))


if __name__ == "__main__":
    main()
