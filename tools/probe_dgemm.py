"""Throughput of cuBLAS fp64 GEMM (DMMA path, if any) vs the measured DFMA peak."""
import torch
for (m, n, k) in ((8192, 8192, 8192), (65536, 256, 2048)):
    a = torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"dgemm {m}x{n}x{k}: {ms:.3f} ms  {2*m*n*k/ms/1e9:.1f} TFLOP/s")
