"""Speed and accuracy of the 3xBF16 / BF16 GEMM for one B2_GEMM_KC setting
(promotion interval in k-blocks: 64 deep for the bf16 modes, 32 for the tf32
modes; read once per process).

    B2_GEMM_KC=16 python scripts/gemm_kc_probe.py
"""
import os
import sys

sys.path.insert(0, '.')
import numpy as np

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L


def timeit(fn, iters=5):
    fn()
    L.synchronize()
    e0, e1 = L.Event(), L.Event()
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    return e0.elapsed_ms(e1) / iters


def split(x, rows, cols):
    h, l = P.Buffer(2 * rows * cols), P.Buffer(2 * rows * cols)
    L.call("b2_bf16x3_split", h.ptr, l.ptr, x.data_ptr, rows, cols, cols, None)
    return h, l


kc = os.environ.get("B2_GEMM_KC", "default")
rng = np.random.default_rng(0)
for M, N, K in ((65536, 4096, 4096), (8192, 8192, 8192)):
    x = P.from_numpy(rng.standard_normal((M, K), dtype=np.float32))
    w = P.from_numpy(rng.uniform(-1 / 64, 1 / 64, (N, K)).astype(np.float32))
    xh, xl = split(x, M, K)
    wh, wl = split(w, N, K)
    y = P.zeros((M, N))
    f = lambda: L.call("b2_gemm_3xbf16", 0, 1, M, N, K, xh.ptr, xl.ptr, wh.ptr, wl.ptr, y.data_ptr, N,
                       None, 0, None, None, None, None, None)
    ms = timeit(f)
    print(f"KC={kc} 3xbf16 {M}x{N}x{K}: {ms:.3f} ms {2 * M * N * K / ms / 1e9:.1f} TFLOP/s", flush=True)
    del x, w, xh, xl, wh, wl, y

for name, lo in (("signed", -1.0), ("positive", 0.0)):
    M = N = 256
    K = 8192
    A = rng.uniform(lo, 1, (M, K)).astype(np.float32)
    B = rng.uniform(lo, 1, (N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    At, Bt = P.from_numpy(A), P.from_numpy(B)
    for algo_name, algo in (("3xbf16", L.GEMM_3XBF16), ("tf32x", L.GEMM_TF32X)):
        C = P.zeros((M, N))
        L.call("b2_gemm", 0, 1, M, N, K, At.data_ptr, K, Bt.data_ptr, K, C.data_ptr, N, None, 0, algo, None)
        c = C.numpy()
        err = np.abs(c - ref).max() / np.abs(ref).max()
        print(f"KC={kc} {algo_name} {name} K={K}: normwise {err:.2e}", flush=True)
