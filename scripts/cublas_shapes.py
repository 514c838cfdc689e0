#!/usr/bin/env python
"""Calibration only (not part of the product path): cuBLAS bf16 throughput on the TEM step's
GEMM shapes, to judge how far the hand-written tcgen05 kernels are from a library GEMM."""
import torch

def bench(M, N, K, iters=50):
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        torch.matmul(a, b)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(iters):
        torch.matmul(a, b)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / iters * 1e-3
    return t, 2 * M * N * K / t / 1e12

for name, (M, N, K) in {
    "c3 conv2 fwd (R x 512 x 1536)": (26112, 512, 1536),
    "c3 conv1 fwd (R x 512 x 1200)": (26112, 512, 1200),
    "c3 wgrad2 (512 x 1536 x R)": (512, 1536, 26112),
    "c2 conv2 fwd (1632 x 512 x 1536)": (1632, 512, 1536),
    "c2 wgrad2 (512 x 1536 x 1632)": (512, 1536, 1632),
    "square 8192": (8192, 8192, 8192),
}.items():
    t, tf = bench(M, N, K)
    print(f"{name:36s} {t*1e6:8.1f} us  {tf:7.1f} TFLOP/s")
