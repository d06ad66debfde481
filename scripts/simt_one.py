"""One FP32 SIMT GEMM launch set for ncu: python scripts/simt_one.py n ta tb"""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
n, ta, tb = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(0)
At = P.from_numpy(rng.uniform(-1, 1, (n, n)).astype(np.float32))
Bt = P.from_numpy(rng.uniform(-1, 1, (n, n)).astype(np.float32))
C = P.zeros((n, n))
for _ in range(3):
    L.call("b2_gemm", ta, tb, n, n, n, At.data_ptr, n, Bt.data_ptr, n, C.data_ptr, n, None, 0, L.GEMM_SIMT, None)
L.synchronize()
