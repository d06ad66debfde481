"""One fused-epilogue case of the config-5 dX GEMM, launched twice (for ncu:
-k regex:k_gemm_tc --launch-skip 1 -c 1).  python scripts/epi_case.py plain|full|fwd|fwd_split_only"""
import sys

sys.path.insert(0, '.')
import numpy as np

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L

case = sys.argv[1] if len(sys.argv) > 1 else "plain"
M, N, K = 65536, 4096, 4096
rng = np.random.default_rng(0)
g = P.from_numpy(rng.standard_normal((M, K), dtype=np.float32))
w = P.from_numpy(rng.uniform(-1 / 64, 1 / 64, (K, N)).astype(np.float32))
gh, gl, wh, wl = (P.Buffer(2 * M * K), P.Buffer(2 * M * K), P.Buffer(2 * N * K), P.Buffer(2 * N * K))
L.call("b2_bf16x3_split", gh.ptr, gl.ptr, g.data_ptr, M, K, K, None)
L.call("b2_bf16x3_split", wh.ptr, wl.ptr, w.data_ptr, K, N, N, None)
y = P.zeros((M, N))
yh, yl = P.Buffer(2 * M * N), P.Buffer(2 * M * N)
cs = P.zeros((N,))
bits = P.Buffer(8 * M * N // 64)
b = P.zeros((N,))
d = L.GemmDesc()
d.algo, d.trans_a, d.trans_b, d.M, d.N, d.K = L.GEMM_3XBF16, 0, 0, M, N, K
d.a[0], d.a[1], d.b[0], d.b[1] = gh.ptr, gl.ptr, wh.ptr, wl.ptr
d.lda, d.ldb, d.C, d.ldc = K, N, y.data_ptr, N
if case == "full":
    d.mask_bits, d.colsum = bits.ptr, cs.data_ptr
    d.c_hi, d.c_lo = yh.ptr, yl.ptr
elif case in ("fwd", "fwd_split_only"):
    d.epilogue, d.bias, d.relu_bits_out = L.EPI_BIAS_RELU, b.data_ptr, bits.ptr
    d.c_hi, d.c_lo = yh.ptr, yl.ptr
    if case == "fwd_split_only":  # the product's hidden-layer forward: no fp32 C store
        d.C = None
for _ in range(2):
    L.call("b2_gemm_fused", L.ctypes.byref(d), None)
L.synchronize()
print("ok", case)
