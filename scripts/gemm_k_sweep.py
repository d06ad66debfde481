"""Presplit 3xBF16 GEMM rate vs K at the config-5 output shape (65536 x 4096), all layouts the
step uses; fp32 C store. python scripts/gemm_k_sweep.py"""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L

M, N = 65536, 4096
c = P.zeros((M, N))
for K in (512, 1000, 1024, 2048, 4096):
    for ta, tb in ((0, 1), (0, 0)):
        ah, al = P.Buffer(2 * M * K), P.Buffer(2 * M * K)
        bh, bl = P.Buffer(2 * N * K), P.Buffer(2 * N * K)
        L.call("b2_memset", ah.ptr, 0, 2 * M * K, None) if hasattr(L.lib(), "b2_memset") else None
        f = lambda: L.call("b2_gemm_3xbf16", ta, tb, M, N, K, ah.ptr, al.ptr, bh.ptr, bl.ptr, c.data_ptr, N,
                           None, 0, None, None, None, None, None)
        for _ in range(2):
            f()
        L.synchronize()
        e0, e1 = L.Event(), L.Event()
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        L.synchronize()
        ms = e0.elapsed_ms(e1) / 5
        print(f"K={K} ta={ta} tb={tb}: {ms:.3f} ms {2 * M * N * K / ms / 1e9:.0f} TF/s", flush=True)
        del ah, al, bh, bl
