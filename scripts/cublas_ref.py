"""cuBLAS (torch.matmul, bf16 in / bf16 out) on the step's GEMM shapes, CUDA-event timed,
as a library reference point for the tcgen05 kernels' per-launch times (not on any product path)."""
import torch

SHAPES = {"fwd.qkv": (16384, 1536, 512), "fwd.gu (gate|up)": (16384, 2752, 512), "head.logits": (16384, 32000, 512),
          "nbr.d_h2": (16384, 512, 2752), "head.d_xf": (16384, 512, 32000), "head.g_unemb": (32000, 512, 16384),
          "square 8192": (8192, 8192, 8192)}
for name, (M, N, K) in SHAPES.items():
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    s.record()
    for _ in range(n):
        c = a @ b
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / n * 1e3
    print(f"{name:20s} M={M:6d} N={N:6d} K={K:6d}  {us:8.1f} us  {2 * M * N * K / us / 1e6:7.1f} TFLOP/s")
