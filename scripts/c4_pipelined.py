"""Config 4 (fused form) as a training loop would feed it: every step a new
batch X from a 2-slot device-resident feeder whose 3xBF16 split is made on the
feeder's stream during the previous step (as bench.py's config-5 input
pipeline), W changed every step (as after an optimizer update). Eager launches,
device time per step with events."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
from paper_2602_00125_b200.data import PinnedFeeder

rng = np.random.default_rng(0)
x = rng.standard_normal((32768, 1024), dtype=np.float32)
W = P.from_numpy(rng.normal(0, 0.03, (1024, 1024)).astype(np.float32), requires_grad=True)
bias = P.zeros((1024,), requires_grad=True)
T = P.from_numpy(rng.uniform(0, 1, (32768, 1024)).astype(np.float32))
feed = PinnedFeeder(x, np.zeros(32768, np.int64), presplit="3xbf16", resident=True)
P.set_gemm_algo("3xbf16")


def step():
    P.reset_tape()
    X, _ = feed.next()
    X.requires_grad = True
    W.buffer.version += 1
    z = P.linear(X, P.transpose2d(W), bias)
    P.backward(P.softmax_mul_mean(z, T))


for _ in range(3):
    step()
L.synchronize()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
e0, e1 = L.Event(), L.Event()
e0.record()
for _ in range(n):
    step()
e1.record()
print(f"config 4 pipelined (eager): {e0.elapsed_ms(e1) / n:.3f} ms/step")
