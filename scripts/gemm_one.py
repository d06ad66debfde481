"""One presplit 3xBF16 GEMM launched 3 times (for ncu): python scripts/gemm_one.py M N K"""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
M, N, K = (int(v) for v in sys.argv[1:4])
rng = np.random.default_rng(0)
a = P.from_numpy(rng.uniform(-1, 1, (M, K)).astype(np.float32))
b = P.from_numpy(rng.uniform(-1, 1, (N, K)).astype(np.float32))
ah, al, bh, bl = P.Buffer(2 * M * K), P.Buffer(2 * M * K), P.Buffer(2 * N * K), P.Buffer(2 * N * K)
L.call("b2_bf16x3_split", ah.ptr, al.ptr, a.data_ptr, M, K, K, None)
L.call("b2_bf16x3_split", bh.ptr, bl.ptr, b.data_ptr, N, K, K, None)
c = P.zeros((M, N))
for _ in range(3):
    L.call("b2_gemm_3xbf16", 0, 1, M, N, K, ah.ptr, al.ptr, bh.ptr, bl.ptr, c.data_ptr, N, None, 0,
           None, None, None, None, None)
L.synchronize()
print("ok")
