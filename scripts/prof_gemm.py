"""One config-5 forward GEMM (M=65536, N=K=4096, 3xTF32 presplit) for ncu."""
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
xh, xl, wh, wl = P.zeros((M, K)), P.zeros((M, K)), P.zeros((N, K)), P.zeros((N, K))
L.call("b2_tf32_split", xh.data_ptr, xl.data_ptr, x.data_ptr, M, K, K, None)
L.call("b2_tf32_split", wh.data_ptr, wl.data_ptr, w.data_ptr, N, K, K, None)
y = P.zeros((M, N))
for _ in range(3):
    L.call("b2_gemm_presplit", 0, 1, M, N, K, xh.data_ptr, xl.data_ptr, wh.data_ptr, wl.data_ptr,
           y.data_ptr, N, b.data_ptr, L.EPI_BIAS_RELU, None)
L.synchronize()
print("ok", float(y.numpy()[0, :4].sum()))
