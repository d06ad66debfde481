"""Device time of one presplit 3xBF16 GEMM launch vs K (M = N fixed): separates the
per-launch fixed cost from the per-k-block cost. Launches b2_gemm_3xbf16 on
pre-made splits directly (no split kernels inside the timed graph)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph

M = N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
rng = np.random.default_rng(0)
for K in (64, 256, 1024, 4096):
    a = P.from_numpy(rng.uniform(-1, 1, (M, K)).astype(np.float32))
    b = P.from_numpy(rng.uniform(-1, 1, (N, K)).astype(np.float32))
    ah, al, bh, bl = P.Buffer(2 * M * K), P.Buffer(2 * M * K), P.Buffer(2 * N * K), P.Buffer(2 * N * K)
    L.call("b2_bf16x3_split", ah.ptr, al.ptr, a.data_ptr, M, K, K, None)
    L.call("b2_bf16x3_split", bh.ptr, bl.ptr, b.data_ptr, N, K, K, None)
    c = P.zeros((M, N))

    def one():
        L.call("b2_gemm_3xbf16", 0, 1, M, N, K, ah.ptr, al.ptr, bh.ptr, bl.ptr, c.data_ptr, N, None, 0,
               None, None, None, None, None)

    g = graph.capture(lambda: [one() for _ in range(20)], warmup=1)
    g.replay()
    L.synchronize()
    e0, e1 = L.Event(), L.Event()
    e0.record()
    g.replay()
    e1.record()
    us = e0.elapsed_ms(e1) / 20 * 1000
    print(f"M=N={M} K={K:5d}: {us:7.2f} us  {2 * M * N * K / us * 1e-6:7.1f} TF/s")
