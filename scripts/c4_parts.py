"""Config-4 (fused form) kernel-by-kernel device times, each replayed 10x in a
CUDA graph (warm L2 state as in the step; inputs 128 MiB each > L2 halves)."""
import sys
sys.path.insert(0, '.')
import ctypes
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph, core as C

R, K = 32768, 1024
rng = np.random.default_rng(0)
X = P.from_numpy(rng.standard_normal((R, K), dtype=np.float32))
W = P.from_numpy(rng.normal(0, 0.03, (K, K)).astype(np.float32))
bias = P.zeros((K,))
T = P.from_numpy(rng.uniform(0, 1, (R, K)).astype(np.float32))
Z = P.from_numpy(rng.standard_normal((R, K), dtype=np.float32))
g = P.ones(())
loss = P.zeros(())
rs, rm, rdot = P.Buffer(4 * R), P.Buffer(4 * R), P.Buffer(8 * R)
hi, lo = P.Buffer(2 * R * K), P.Buffer(2 * R * K)
cs = P.zeros((K,))
out = P.zeros((R, K))


def t(name, fn, n=10, gbytes=None, flops=None):
    gr = graph.capture(lambda: [fn() for _ in range(n)], warmup=1)
    gr.replay()
    L.synchronize()
    e0, e1 = L.Event(), L.Event()
    e0.record()
    gr.replay()
    e1.record()
    us = e0.elapsed_ms(e1) / n * 1000
    extra = ""
    if gbytes:
        extra += f"  {gbytes / us * 1e-3:.2f} TB/s"
    if flops:
        extra += f"  {flops / us * 1e-6:.1f} TF/s"
    print(f"{name:28s} {us:8.1f} us{extra}")


MB = 1 << 20
t("softmax_wmean_fwd", lambda: L.call("b2_softmax_wmean_fwd", loss.data_ptr, None, rs.ptr, rm.ptr, rdot.ptr,
                                       Z.data_ptr, T.data_ptr, R, K, None), gbytes=256 * MB)
t("softmax_wmean_bwd(split+cs)", lambda: L.call("b2_softmax_wmean_bwd", None, hi.ptr, lo.ptr, cs.data_ptr,
                                                 g.data_ptr, float(R * K), Z.data_ptr, T.data_ptr, rs.ptr,
                                                 rm.ptr, R, K, None), gbytes=384 * MB)
t("softmax_wmean_bwd(fp32 gz)", lambda: L.call("b2_softmax_wmean_bwd", out.data_ptr, None, None, None,
                                                g.data_ptr, float(R * K), Z.data_ptr, T.data_ptr, rs.ptr,
                                                rm.ptr, R, K, None), gbytes=384 * MB)
t("softmax_fwd (composed)", lambda: L.call("b2_softmax_fwd", out.data_ptr, rs.ptr, rm.ptr, Z.data_ptr, R, K,
                                            None), gbytes=256 * MB)
t("split X (3xbf16)", lambda: L.call("b2_bf16x3_split", hi.ptr, lo.ptr, X.data_ptr, R, K, K, None),
  gbytes=256 * MB)
P.set_gemm_algo("3xbf16")
with P.no_grad():
    t("linear fwd (X.W^T + b)", lambda: (setattr(X.buffer, "version", X.buffer.version + 1),
                                         C.linear(X, W, bias)), flops=2 * R * K * K)
    Xs = C._split(X, R, K, K, "3xbf16")
    t("gemm NN dX = gz.W (presplit)", lambda: C._gemm_into(out, Z, P.transpose2d(W)), flops=2 * R * K * K)
    t("gemm TN dW = X^T.gz", lambda: C._gemm_into(P.zeros((K, K)), P.transpose2d(X), P.transpose2d(Z)),
      flops=2 * R * K * K)
    dWo = P.zeros((K, K))

    def grp():
        with C.gemm_group():
            C._gemm_into(out, Z, P.transpose2d(W))
            C._gemm_into(dWo, P.transpose2d(X), P.transpose2d(Z))

    t("gemm dX + dW grouped", grp, flops=4 * R * K * K)
P.set_gemm_algo(None)
# the whole fused config-4 step as bench.py times it (nn.Linear + fused loss)
Xg = P.from_numpy(rng.standard_normal((R, K), dtype=np.float32), requires_grad=True)
Wg = P.from_numpy(rng.normal(0, 0.03, (K, K)).astype(np.float32), requires_grad=True)
bg = P.zeros((K,), requires_grad=True)


def step():
    P.reset_tape()
    Xg.buffer.version += 1
    Wg.buffer.version += 1
    z = P.linear(Xg, P.transpose2d(Wg), bg)
    P.backward(P.softmax_mul_mean(z, T))


t("config-4 fused step", step, n=5, flops=6 * R * K * K)
print("ok")
