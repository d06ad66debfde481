"""Config 3 (square matmul fwd+bwd) device time per iteration in a CUDA graph,
plus each GEMM / split alone -- for few-tile GEMM tuning."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph, core as C

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
rng = np.random.default_rng(0)
A = P.from_numpy(rng.uniform(-1, 1, (n, n)).astype(np.float32), requires_grad=True)
B = P.from_numpy(rng.uniform(-1, 1, (n, n)).astype(np.float32), requires_grad=True)
dC = P.from_numpy(rng.standard_normal((n, n), dtype=np.float32))


def t(name, fn, iters=10, flops=None):
    g = graph.capture(lambda: [fn() for _ in range(iters)], warmup=1)
    g.replay()
    L.synchronize()
    e0, e1 = L.Event(), L.Event()
    e0.record()
    g.replay()
    e1.record()
    us = e0.elapsed_ms(e1) / iters * 1000
    print(f"{name:34s} {us:8.2f} us" + (f"  {flops / us * 1e-6:7.1f} TF/s" if flops else ""))


def fb():
    P.reset_tape()
    A.buffer.version += 1
    B.buffer.version += 1
    Cc = P.mm(A, B)
    P.backward(Cc, seed=dC)


t(f"fwd+bwd n={n}", fb, flops=6 * n ** 3)
hi, lo = P.Buffer(2 * n * n), P.Buffer(2 * n * n)
t("split (3xbf16)", lambda: L.call("b2_bf16x3_split", hi.ptr, lo.ptr, A.data_ptr, n, n, n, None))
out = P.zeros((n, n))
with P.no_grad():
    C._split(A, n, n, n, "3xbf16")
    C._split(B, n, n, n, "3xbf16")
    C._split(dC, n, n, n, "3xbf16")
    t("gemm NN (presplit)", lambda: C._gemm_into(out, A, P.transpose2d(B)), flops=2 * n ** 3)
    t("gemm NT (presplit)", lambda: C._gemm_into(out, dC, B), flops=2 * n ** 3)
    t("gemm TN (presplit)", lambda: C._gemm_into(out, P.transpose2d(A), P.transpose2d(dC)), flops=2 * n ** 3)
    out2 = P.zeros((n, n))

    def grouped():
        with C.gemm_group():
            C._gemm_into(out, dC, B)
            C._gemm_into(out2, P.transpose2d(A), P.transpose2d(dC))

    t("gemm NT + TN grouped (presplit)", grouped, flops=4 * n ** 3)
print("ok")
