"""cuBLAS (torch.matmul, bf16) on the implicit-GEMM shapes of the SDXL-shape convs, for comparison."""
import torch

SH = [(16384, 320, 2880), (16384, 320, 5760), (4096, 640, 2880), (4096, 640, 5760), (4096, 640, 11520),
      (1024, 1280, 5760), (1024, 1280, 11520), (8192, 8192, 8192)]
for m, n, k in SH:
    a = torch.randn(m, k, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, k, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        c = a @ b.T
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        c = a @ b.T
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(f"cuBLAS {m}x{n}x{k}: {us:7.1f} us {2 * m * n * k / us / 1e6:7.0f} TF/s", flush=True)
