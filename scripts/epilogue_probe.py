"""Cost of the fused epilogue stages on the config-5 dX GEMM (NN layout,
65536 x 4096 x 4096, 3xBF16): plain / + split emission / + ReLU-pullback mask
/ + column sums, and the ReLU pullback read from 1-bit masks (mask_bits) and
the forward GEMM's bit emission (relu_bits_out), all through b2_gemm_fused."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
M, N, K = 65536, 4096, 4096
rng = np.random.default_rng(0)
g = P.from_numpy(rng.standard_normal((M, K), dtype=np.float32))
w = P.from_numpy(rng.uniform(-1/64, 1/64, (K, N)).astype(np.float32))   # stored [K, N]: MN-major B
mask = P.from_numpy((rng.standard_normal((M, N)) > 0).astype(np.float32))
gh, gl, wh, wl = (P.Buffer(2 * M * K), P.Buffer(2 * M * K), P.Buffer(2 * N * K), P.Buffer(2 * N * K))
L.call("b2_bf16x3_split", gh.ptr, gl.ptr, g.data_ptr, M, K, K, None)
L.call("b2_bf16x3_split", wh.ptr, wl.ptr, w.data_ptr, K, N, N, None)
y = P.zeros((M, N))
yh, yl = P.Buffer(2 * M * N), P.Buffer(2 * M * N)
cs = P.zeros((N,))
bits = P.Buffer(8 * M * N // 64)
b = P.zeros((N,))


def run(emit, msk, col, bit_in=0, bit_out=0):
    d = L.GemmDesc()
    d.algo, d.trans_a, d.trans_b, d.M, d.N, d.K = L.GEMM_3XBF16, 0, 0, M, N, K
    d.a[0], d.a[1], d.b[0], d.b[1] = gh.ptr, gl.ptr, wh.ptr, wl.ptr
    d.lda, d.ldb, d.C, d.ldc = K, N, y.data_ptr, N
    d.epilogue = L.EPI_BIAS_RELU if bit_out else 0
    d.bias = b.data_ptr if bit_out else None
    d.mask = mask.data_ptr if msk else None
    d.mask_bits = bits.ptr if bit_in else None
    d.relu_bits_out = bits.ptr if bit_out == 1 else None  # 2: bias+relu epilogue alone
    d.c_hi, d.c_lo = (yh.ptr, yl.ptr) if emit else (None, None)
    d.colsum = cs.data_ptr if col else None
    L.call("b2_gemm_fused", L.ctypes.byref(d), None)


run(0, 0, 0, 0, 1)  # bits of a real relu pattern
cases = (("plain", (0, 0, 0)), ("+split", (1, 0, 0)), ("+split+mask", (1, 1, 0)),
         ("+split+bits", (1, 0, 0, 1)), ("+split+mask+colsum", (1, 1, 1)),
         ("+split+bits+colsum", (1, 0, 1, 1)), ("+split+colsum", (1, 0, 1)),
         ("fwd bias+relu+split", (1, 0, 0, 0, 2)), ("fwd +bits_out", (1, 0, 0, 0, 1)))
res = {name: [] for name, _ in cases}
order = list(cases)
for r in range(7):  # shuffled rounds, median per case (clocks drift under the power cap)
    rng.shuffle(order)
    for name, args in order:
        run(*args)
        L.synchronize()
        e0, e1 = L.Event(), L.Event()
        e0.record()
        for _ in range(5):
            run(*args)
        e1.record()
        res[name].append(e0.elapsed_ms(e1) / 5)
for name, _ in cases:
    ms = float(np.median(res[name]))
    print(f"dX NN {name:22s}: median {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s "
          f"(min {min(res[name]):.3f})", flush=True)
