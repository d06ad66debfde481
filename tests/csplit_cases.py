"""Few-tile tensor-core GEMMs with every epilogue stage, written to an .npz:
run by tests/test_gpu_gemm_group.py once with cluster split-K (default) and
once with B2_GEMM_CSPLIT=0 (K-slice partials through L2 + k_tail_epilogue)."""
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
    (1024, 1024, 1024, 0, 0, "bias_relu_bits_split_colsum"),   # 32 tiles -> 4 slices
    (1000, 1000, 2048, 1, 1, "maskbits_split_colsum"),        # ragged, 32 tiles -> 4 slices
    (2048, 1024, 1024, 0, 1, "plain"),                         # 64 tiles -> 2 slices
    (768, 768, 4096, 0, 0, "bias_colsum"),                     # 18 tiles -> 8 slices
]
out = {}
rng = np.random.default_rng(3)
for ci, (M, N, K, ta, tb, what) in enumerate(CASES):
    ar, ac = (K, M) if ta else (M, K)
    br, bc = (N, K) if tb else (K, N)
    A = P.from_numpy(rng.standard_normal((ar, ac), dtype=np.float32))
    B = P.from_numpy(rng.uniform(-0.05, 0.05, (br, bc)).astype(np.float32))
    ah, al, bh, bl = (P.Buffer(2 * ar * ac), P.Buffer(2 * ar * ac), P.Buffer(2 * br * bc), P.Buffer(2 * br * bc))
    L.call("b2_bf16x3_split", ah.ptr, al.ptr, A.data_ptr, ar, ac, ac, None)
    L.call("b2_bf16x3_split", bh.ptr, bl.ptr, B.data_ptr, br, bc, bc, None)
    bias = P.from_numpy(rng.standard_normal(N).astype(np.float32))
    words = (N + 63) // 64
    mb = P.Buffer(8 * M * words)
    bits = rng.integers(0, 2 ** 63, (M, words), dtype=np.int64)
    L.call("b2_memcpy_h2d", mb.ptr, bits.ctypes.data_as(ctypes.c_void_p), bits.nbytes, None)
    o = {"C": P.Buffer(4 * M * N), "hi": P.Buffer(2 * M * N), "lo": P.Buffer(2 * M * N),
         "cs": P.Buffer(4 * N), "bits": P.Buffer(8 * M * words)}
    d = L.GemmDesc()
    d.algo, d.trans_a, d.trans_b, d.M, d.N, d.K = L.GEMM_3XBF16, ta, tb, M, N, K
    d.a[0], d.a[1], d.b[0], d.b[1] = ah.ptr, al.ptr, bh.ptr, bl.ptr
    d.lda, d.ldb, d.C, d.ldc = ac, bc, o["C"].ptr, N
    if "bias" in what:
        d.bias = bias.data_ptr
        d.epilogue = L.EPI_BIAS_RELU if "relu" in what else L.EPI_BIAS
    if "bits" in what and "mask" not in what:
        d.relu_bits_out = o["bits"].ptr
    if "maskbits" in what:
        d.mask_bits = mb.ptr
    if "split" in what:
        d.c_hi, d.c_lo = o["hi"].ptr, o["lo"].ptr
    if "colsum" in what:
        d.colsum = o["cs"].ptr
    L.call("b2_gemm_fused", ctypes.byref(d), None)
    L.synchronize()
    for k, b in o.items():
        out[f"{ci}_{k}"] = read(b, b.nbytes)
np.savez(sys.argv[1], **out)
print("ok")
