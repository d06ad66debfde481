"""Config-5 GEMM shapes with and without the tail-wave K slices: run once
with the default and once with B2_GEMM_SPLITK=0 (read once per process).

    python scripts/tail_probe.py            # default
    B2_GEMM_SPLITK=0 python scripts/tail_probe.py
"""
import os
import sys

sys.path.insert(0, '.')
import numpy as np

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L

tag = "nosplit" if os.environ.get("B2_GEMM_SPLITK") == "0" else "tail"
rng = np.random.default_rng(0)
SHAPES = (("fwd NT", 0, 1, 65536, 4096, 4096), ("dX NN", 0, 0, 65536, 4096, 4096),
          ("dW TN", 1, 0, 4096, 4096, 65536), ("out NT", 0, 1, 65536, 1000, 4096),
          ("dWout TN", 1, 0, 1000, 4096, 65536))
for name, ta, tb, M, N, K in SHAPES:
    ar, ac = (K, M) if ta else (M, K)
    br, bc = (N, K) if tb else (K, N)
    a = P.from_numpy(rng.standard_normal((ar, ac), dtype=np.float32))
    b = P.from_numpy(rng.uniform(-1 / 64, 1 / 64, (br, bc)).astype(np.float32))
    ah, al, bh, bl = (P.Buffer(2 * ar * ac), P.Buffer(2 * ar * ac), P.Buffer(2 * br * bc), P.Buffer(2 * br * bc))
    L.call("b2_bf16x3_split", ah.ptr, al.ptr, a.data_ptr, ar, ac, ac, None)
    L.call("b2_bf16x3_split", bh.ptr, bl.ptr, b.data_ptr, br, bc, bc, None)
    c = P.zeros((M, N))
    for mode, algo in (("3xbf16", L.GEMM_3XBF16), ("bf16", L.GEMM_BF16)):
        d = L.GemmDesc()
        d.algo, d.trans_a, d.trans_b, d.M, d.N, d.K = algo, ta, tb, M, N, K
        d.a[0], d.b[0] = ah.ptr, bh.ptr
        if mode == "3xbf16":
            d.a[1], d.b[1] = al.ptr, bl.ptr
        d.lda, d.ldb, d.C, d.ldc = ac, bc, c.data_ptr, N
        ms = []
        for r in range(5):
            L.call("b2_gemm_fused", L.ctypes.byref(d), None)
            L.synchronize()
            e0, e1 = L.Event(), L.Event()
            e0.record()
            for _ in range(4):
                L.call("b2_gemm_fused", L.ctypes.byref(d), None)
            e1.record()
            L.synchronize()
            ms.append(e0.elapsed_ms(e1) / 4)
        t = float(np.median(ms))
        print(f"{tag:8s} {name:9s} {mode:7s} {M}x{N}x{K}: median {t:.3f} ms "
              f"{2 * M * N * K / t / 1e9:.1f} TFLOP/s (min {min(ms):.3f})", flush=True)
    del a, b, ah, al, bh, bl, c
