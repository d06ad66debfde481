"""bf16-variant GEMMs big enough for 512-row pair tiles (MODE 6), every
epilogue stage, written to an .npz: tests/test_gpu_gemm_group.py runs it with
B2_GEMM_M2=1 (default) and 0 (256-row pair tiles) and compares."""
import ctypes
import sys

import numpy as np

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L


def read(buf, nbytes):
    out = np.empty(nbytes, np.uint8)
    L.call("b2_memcpy_d2h", out.ctypes.data_as(ctypes.c_void_p), buf.ptr, nbytes, None)
    return out


CASES = [  # M, N, K, ta, tb, stages
    (16384, 4096, 4096, 0, 1, "bias_relu_bits_cast"),       # forward-like (x . W^T)
    (16000, 4000, 4096, 0, 0, "maskbits_cast_colsum"),      # dX-like, ragged M and N
    (4096, 4096, 16384, 1, 0, "plain"),                     # dW-like, long K (2 tile waves)
]
out = {}
rng = np.random.default_rng(5)
for ci, (M, N, K, ta, tb, what) in enumerate(CASES):
    ar, ac = (K, M) if ta else (M, K)
    br, bc = (N, K) if tb else (K, N)
    A = P.from_numpy(rng.standard_normal((ar, ac), dtype=np.float32))
    B = P.from_numpy(rng.uniform(-0.05, 0.05, (br, bc)).astype(np.float32))
    a16, b16 = P.Buffer(2 * ar * ac), P.Buffer(2 * br * bc)
    L.call("b2_bf16_cast", a16.ptr, A.data_ptr, ar, ac, ac, None)
    L.call("b2_bf16_cast", b16.ptr, B.data_ptr, br, bc, bc, None)
    del A, B
    bias = P.from_numpy(rng.standard_normal(N).astype(np.float32))
    words = (N + 63) // 64
    mb = P.Buffer(8 * M * words)
    bits = rng.integers(0, 2 ** 63, (M, words), dtype=np.int64)
    L.call("b2_memcpy_h2d", mb.ptr, bits.ctypes.data_as(ctypes.c_void_p), bits.nbytes, None)
    o = {"C": P.Buffer(4 * M * N), "c16": P.Buffer(2 * M * N), "cs": P.Buffer(4 * N),
         "bits": P.Buffer(8 * M * words)}
    d = L.GemmDesc()
    d.algo, d.trans_a, d.trans_b, d.M, d.N, d.K = L.GEMM_BF16, ta, tb, M, N, K
    d.a[0], d.b[0] = a16.ptr, b16.ptr
    d.lda, d.ldb, d.C, d.ldc = ac, bc, o["C"].ptr, N
    if "bias" in what:
        d.bias = bias.data_ptr
        d.epilogue = L.EPI_BIAS_RELU if "relu" in what else L.EPI_BIAS
    if "bits" in what and "mask" not in what:
        d.relu_bits_out = o["bits"].ptr
    if "maskbits" in what:
        d.mask_bits = mb.ptr
    if "cast" in what:
        d.c_hi = o["c16"].ptr
    if "colsum" in what:
        d.colsum = o["cs"].ptr
    L.call("b2_gemm_fused", ctypes.byref(d), None)
    L.synchronize()
    for k, b in o.items():
        out[f"{ci}_{k}"] = read(b, b.nbytes)
np.savez(sys.argv[1], **out)
print("ok")
