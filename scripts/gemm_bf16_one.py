"""One bf16-variant GEMM (NT, M=N=K=n) launched 3x (for ncu) and timed 20x in a graph."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
M, N, K = n, n, n
if len(sys.argv) > 2 and sys.argv[2].isdigit():
    M = int(sys.argv[2])
rng = np.random.default_rng(0)
a = P.from_numpy(rng.uniform(-1, 1, (M, K)).astype(np.float32))
b = P.from_numpy(rng.uniform(-1, 1, (N, K)).astype(np.float32))
a16, b16 = P.Buffer(2 * M * K), P.Buffer(2 * N * K)
L.call("b2_bf16_cast", a16.ptr, a.data_ptr, M, K, K, None)
L.call("b2_bf16_cast", b16.ptr, b.data_ptr, N, K, K, None)
c = P.zeros((M, N))


def one():
    L.call("b2_gemm_bf16", 0, 1, M, N, K, a16.ptr, b16.ptr, c.data_ptr, N, None, 0, None, None, None, None)


if "--time" in sys.argv:
    g = graph.capture(lambda: [one() for _ in range(20)], warmup=1)
    g.replay()
    L.synchronize()
    e0, e1 = L.Event(), L.Event()
    e0.record()
    g.replay()
    e1.record()
    us = e0.elapsed_ms(e1) / 20 * 1000
    print(f"bf16 GEMM {M}x{N}x{K}: {us:.1f} us  {2 * M * N * K / us * 1e-6:.0f} TF/s")
else:
    for _ in range(3):
        one()
    L.synchronize()
print("ok")
