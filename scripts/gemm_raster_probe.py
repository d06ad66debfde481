"""Config-5 forward GEMM (3xBF16, 65536x4096x4096, bias+relu, emitted split)
timed 10x for one B2_GEMM_GROUPN (read once per process)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
M, N, K = 65536, 4096, 4096
rng = np.random.default_rng(0)
x = P.from_numpy(rng.standard_normal((M, K), dtype=np.float32))
w = P.from_numpy(rng.uniform(-1/64, 1/64, (N, K)).astype(np.float32))
b = P.zeros((N,))
bufs = [P.Buffer(2 * s) for s in (M * K, M * K, N * K, N * K, M * N, M * N)]
xh, xl, wh, wl, yh, yl = bufs
L.call("b2_bf16x3_split", xh.ptr, xl.ptr, x.data_ptr, M, K, K, None)
L.call("b2_bf16x3_split", wh.ptr, wl.ptr, w.data_ptr, N, K, K, None)
y = P.zeros((M, N))
def f(ta=0, tb=1):
    L.call("b2_gemm_3xbf16", ta, tb, M, N, K, xh.ptr, xl.ptr, wh.ptr, wl.ptr, y.data_ptr, N,
           b.data_ptr, L.EPI_BIAS_RELU, None, yh.ptr, yl.ptr, None, None)
f(); L.synchronize()
e0, e1 = L.Event(), L.Event()
e0.record()
for _ in range(10): f()
e1.record()
ms = e0.elapsed_ms(e1) / 10
print(f"GROUPN={os.environ.get('B2_GEMM_GROUPN','default')} fwd NT: {ms:.3f} ms {2*M*N*K/ms/1e9:.1f} TFLOP/s", flush=True)
