"""One config-5-shaped forward GEMM in the BF16 mode (65536x4096x4096) for ncu."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
M, N, K = 65536, 4096, 4096
rng = np.random.default_rng(0)
x = P.from_numpy(rng.standard_normal((M, K), dtype=np.float32))
w = P.from_numpy(rng.uniform(-1/64, 1/64, (N, K)).astype(np.float32))
x16, w16 = P.Buffer(2 * M * K), P.Buffer(2 * N * K)
L.call("b2_bf16_cast", x16.ptr, x.data_ptr, M, K, K, None)
L.call("b2_bf16_cast", w16.ptr, w.data_ptr, N, K, K, None)
y = P.zeros((M, N))
for _ in range(3):
    L.call("b2_gemm_bf16", 0, 1, M, N, K, x16.ptr, w16.ptr, y.data_ptr, N, None, 0, None, None, None, None)
L.synchronize()
print("ok")
