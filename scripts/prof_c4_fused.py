"""Config 4 in its fused form (nn.Linear with the bias epilogue + softmax_mul_mean)
x3 steps, for an ncu launch list; --graph times the same step in a CUDA graph."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph
rng = np.random.default_rng(0)
X = P.from_numpy(rng.standard_normal((32768, 1024), dtype=np.float32), requires_grad=True)
W = P.from_numpy(rng.normal(0, 0.03, (1024, 1024)).astype(np.float32), requires_grad=True)
bias = P.zeros((1024,), requires_grad=True)
T = P.from_numpy(rng.uniform(0, 1, (32768, 1024)).astype(np.float32))


def step():
    P.reset_tape()
    X.buffer.version += 1
    W.buffer.version += 1
    z = P.linear(X, P.transpose2d(W), bias)
    P.backward(P.softmax_mul_mean(z, T))


if "--graph" in sys.argv:
    g = graph.capture(lambda: [step() for _ in range(5)], warmup=1)
    g.replay()
    L.synchronize()
    e0, e1 = L.Event(), L.Event()
    e0.record()
    g.replay()
    e1.record()
    print("graph ms/step", e0.elapsed_ms(e1) / 5)
else:
    for _ in range(3):
        step()
    L.synchronize()
print("ok")
