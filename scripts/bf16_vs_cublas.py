"""bf16-variant GEMM (NT) vs cuBLAS (torch.matmul, bf16 in / fp32-accumulate) at n = 4096 / 8192 /
config-5 shape, 20 launches per CUDA graph / loop, same box. Context for the bf16 variant's roofline."""
import subprocess
import sys

import torch

for M, N, K in [(4096, 4096, 4096), (8192, 8192, 8192), (65536, 4096, 4096)]:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    for _ in range(3):
        c = a @ b.t()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        c = a @ b.t()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"cuBLAS bf16 {M}x{N}x{K}: {ms * 1000:.1f} us {2 * M * N * K / ms / 1e9:.0f} TF/s", flush=True)
    del a, b, c
