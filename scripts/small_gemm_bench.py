"""Config-1-sized FP32 GEMMs (the 64x64 cluster split-K latency kernel): device time per launch from a
CUDA-graph replay of 50 launches.  python scripts/small_gemm_bench.py"""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph

rng = np.random.default_rng(0)
for (ta, tb, M, N, K) in [(0, 1, 256, 256, 784), (0, 1, 256, 10, 256), (0, 0, 256, 256, 10), (1, 0, 10, 256, 256),
                          (1, 0, 256, 784, 256)]:
    A = P.from_numpy(rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32))
    B = P.from_numpy(rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32))
    C = P.zeros((M, N))
    lda, ldb = A.shape[1], B.shape[1]

    def body():
        for _ in range(50):
            L.call("b2_gemm", ta, tb, M, N, K, A.data_ptr, lda, B.data_ptr, ldb, C.data_ptr, N, None, 0,
                   L.GEMM_SIMT, None)

    g = graph.capture(body, warmup=1)
    g.replay()
    L.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = L.Event(), L.Event()
        e0.record()
        g.replay()
        e1.record()
        L.synchronize()
        best = min(best, e0.elapsed_ms(e1) / 50 * 1000)
    print(f"small gemm ta={ta} tb={tb} {M}x{N}x{K}: {best:.2f} us/launch", flush=True)
