"""One config-5 forward GEMM (M=65536, N=K=4096, bias+relu, emitted operand
split) on the default fp32 path (3xBF16, 2-CTA) for ncu. --algo tf32x for the
previous default."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L

algo = sys.argv[sys.argv.index("--algo") + 1] if "--algo" in sys.argv else "3xbf16"
M, N, K = 65536, 4096, 4096
rng = np.random.default_rng(0)
x = P.from_numpy(rng.standard_normal((M, K), dtype=np.float32))
w = P.from_numpy(rng.uniform(-1/64, 1/64, (N, K)).astype(np.float32))
b = P.zeros((N,))
xh, xl = P.Buffer(2 * M * K), P.Buffer(2 * M * K)
wh, wl = P.Buffer(2 * N * K), P.Buffer(2 * N * K)
yh, yl = P.Buffer(2 * M * N), P.Buffer(2 * M * N)
split = "b2_bf16x3_split" if algo == "3xbf16" else "b2_bf16x2_split"
L.call(split, xh.ptr, xl.ptr, x.data_ptr, M, K, K, None)
L.call(split, wh.ptr, wl.ptr, w.data_ptr, N, K, K, None)
y = P.zeros((M, N))
for _ in range(3):
    if algo == "3xbf16":
        L.call("b2_gemm_3xbf16", 0, 1, M, N, K, xh.ptr, xl.ptr, wh.ptr, wl.ptr, y.data_ptr, N,
               b.data_ptr, L.EPI_BIAS_RELU, None, yh.ptr, yl.ptr, None, None)
    else:
        L.call("b2_gemm_tf32x", 0, 1, M, N, K, x.data_ptr, K, xh.ptr, xl.ptr, w.data_ptr, K, wh.ptr,
               wl.ptr, y.data_ptr, N, b.data_ptr, L.EPI_BIAS_RELU, None)
L.synchronize()
print("ok", algo, float(y.numpy()[0, :4].sum()))
