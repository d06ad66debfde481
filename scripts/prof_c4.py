"""Config 4 (softmax(X@W+b), loss mean(Y*T), full backward) x3 steps (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
rng = np.random.default_rng(0)
X = P.from_numpy(rng.standard_normal((64, 512, 1024), dtype=np.float32), requires_grad=True)
W = P.from_numpy(rng.normal(0, 0.03, (1024, 1024)).astype(np.float32), requires_grad=True)
bias = P.zeros((1024,), requires_grad=True)
Tt = P.from_numpy(rng.uniform(0, 1, (64, 512, 1024)).astype(np.float32))
for _ in range(3):
    P.reset_tape()
    X.buffer.version += 1
    W.buffer.version += 1
    Y = P.softmax(P.add(P.mm(X, W), bias))
    P.backward(P.mean(P.mul(Y, Tt)))
L.synchronize()
print("ok")
