import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
rng = np.random.default_rng(0)
M, N, K = 256, 256, 784
A = P.from_numpy(rng.uniform(-1, 1, (M, K)).astype(np.float32))
B = P.from_numpy(rng.uniform(-1, 1, (N, K)).astype(np.float32))
C = P.zeros((M, N))
for _ in range(4):
    L.call("b2_gemm", 0, 1, M, N, K, A.data_ptr, K, B.data_ptr, K, C.data_ptr, N, None, 0, L.GEMM_SIMT, None)
L.synchronize()
