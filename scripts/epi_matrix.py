"""Config-5-shaped 3xBF16 GEMMs (M=65536, N=4096, K in {1000, 1024, 4096}) with
the backward's epilogue stages switched on one by one: C store, split only,
+ ReLU mask bits, + fused column sums. Device time per launch (events, 5
launches after 2 warm-ups), rate and the SM clock right after (NVML).
python scripts/epi_matrix.py [K ...]"""
import sys

sys.path.insert(0, '.')
import numpy as np

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L

try:
    import pynvml
    pynvml.nvmlInit()
    _h = pynvml.nvmlDeviceGetHandleByIndex(0)

    def clk():
        return pynvml.nvmlDeviceGetClockInfo(_h, pynvml.NVML_CLOCK_SM)
except Exception:  # noqa: BLE001
    def clk():
        return -1

Ks = [int(a) for a in sys.argv[1:]] or [1000, 1024, 4096]
M, N = 65536, 4096
rng = np.random.default_rng(0)
for K in Ks:
    gh, gl = P.Buffer(2 * M * K), P.Buffer(2 * M * K)
    wh, wl = P.Buffer(2 * N * K), P.Buffer(2 * N * K)
    g = P.from_numpy(rng.standard_normal((M, K), dtype=np.float32))
    w = P.from_numpy(rng.uniform(-1 / 64, 1 / 64, (K, N)).astype(np.float32))
    L.call("b2_bf16x3_split", gh.ptr, gl.ptr, g.data_ptr, M, K, K, None)
    L.call("b2_bf16x3_split", wh.ptr, wl.ptr, w.data_ptr, K, N, N, None)
    del g, w
    y = P.zeros((M, N))
    yh, yl = P.Buffer(2 * M * N), P.Buffer(2 * M * N)
    cs = P.zeros((N,))
    bits = P.Buffer(8 * M * N // 64)
    for case in ("C", "split", "split+bits", "split+bits+colsum", "split+colsum"):
        d = L.GemmDesc()
        d.algo, d.trans_a, d.trans_b, d.M, d.N, d.K = L.GEMM_3XBF16, 0, 0, M, N, K
        d.a[0], d.a[1], d.b[0], d.b[1] = gh.ptr, gl.ptr, wh.ptr, wl.ptr
        d.lda, d.ldb, d.C, d.ldc = K, N, y.data_ptr, N
        if case != "C":
            d.C = None
            d.c_hi, d.c_lo = yh.ptr, yl.ptr
        if "bits" in case:
            d.mask_bits = bits.ptr
        if "colsum" in case:
            d.colsum = cs.data_ptr
        for _ in range(2):
            L.call("b2_gemm_fused", L.ctypes.byref(d), None)
        e0, e1 = L.Event(), L.Event()
        e0.record()
        for _ in range(5):
            L.call("b2_gemm_fused", L.ctypes.byref(d), None)
        e1.record()
        L.synchronize()
        ms = e0.elapsed_ms(e1) / 5
        print(f"K={K:5d} {case:18s} {ms:7.3f} ms  {2 * M * N * K / ms / 1e9:6.1f} TF/s  sm {clk()} MHz",
              flush=True)
