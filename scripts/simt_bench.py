"""FP32 SIMT GEMM (k_gemm_simt) throughput vs the FP32 FFMA peak, every operand layout.
   python scripts/simt_bench.py [n ...]"""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L


def timeit(fn, iters):
    for _ in range(3): fn()
    L.synchronize()
    e0, e1 = L.Event(), L.Event()
    e0.record()
    for _ in range(iters): fn()
    e1.record()
    return e0.elapsed_ms(e1) / iters


PEAK = 148 * 128 * 2 * 1.965e9 / 1e12  # FFMA lanes x 2 flops x max SM clock
for n in [int(a) for a in sys.argv[1:]] or [2048, 4096, 8192]:
    rng = np.random.default_rng(0)
    A = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    B = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    At, Bt, C = P.from_numpy(A), P.from_numpy(B), P.zeros((n, n))
    for ta, tb in ((0, 1), (0, 0), (1, 0), (1, 1)):
        f = lambda: L.call("b2_gemm", ta, tb, n, n, n, At.data_ptr, n, Bt.data_ptr, n, C.data_ptr, n,
                           None, 0, L.GEMM_SIMT, None)
        ms = timeit(f, 20 if n <= 4096 else 5)
        tf = 2 * n ** 3 / ms / 1e9
        err = ""
        if n <= 2048:
            a = A.T if ta else A
            b = B.T if tb else B
            ref = a.astype(np.float64) @ b.astype(np.float64)
            err = f" err={np.abs(C.numpy() - ref).max() / np.abs(ref).max():.2e}"
        print(f"simt n={n} ta={ta} tb={tb}: {ms:.3f} ms {tf:.1f} TFLOP/s = {tf / PEAK:.2f} of {PEAK:.1f} (FFMA peak at 1965 MHz){err}", flush=True)
