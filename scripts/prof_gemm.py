"""One config-5 forward GEMM (M=65536, N=K=4096) on the default fp32 path (TF32X, 2-CTA) for ncu."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
M, N, K = 65536, 4096, 4096
rng = np.random.default_rng(0)
x = P.from_numpy(rng.standard_normal((M, K), dtype=np.float32))
w = P.from_numpy(rng.uniform(-1/64, 1/64, (N, K)).astype(np.float32))
b = P.zeros((N,))
xh, xl = P.Buffer(2 * M * K), P.Buffer(2 * M * K)
wh, wl = P.Buffer(2 * N * K), P.Buffer(2 * N * K)
L.call("b2_bf16x2_split", xh.ptr, xl.ptr, x.data_ptr, M, K, K, None)
L.call("b2_bf16x2_split", wh.ptr, wl.ptr, w.data_ptr, N, K, K, None)
y = P.zeros((M, N))
for _ in range(3):
    L.call("b2_gemm_tf32x", 0, 1, M, N, K, x.data_ptr, K, xh.ptr, xl.ptr, w.data_ptr, K, wh.ptr, wl.ptr,
           y.data_ptr, N, b.data_ptr, L.EPI_BIAS_RELU, None)
L.synchronize()
print("ok", float(y.numpy()[0, :4].sum()))
