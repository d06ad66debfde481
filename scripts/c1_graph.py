"""Config 1 (784-256-10 MLP, batch 256, SGD): device time per step from a CUDA-graph replay of 50 steps."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, nn, optim, graph
from paper_2602_00125_b200.data import build_mlp, linear_params

r1 = np.random.default_rng(0)
c1 = build_mlp([linear_params(r1, 784, 256), linear_params(r1, 256, 10)])
x1 = P.from_numpy(r1.standard_normal((256, 784), dtype=np.float32))
l1 = nn.labels_buffer(r1.integers(0, 10, 256))
sgd = optim.SGD(lr=0.01)


def steps():
    for _ in range(50):
        P.reset_tape()
        loss = nn.cross_entropy(c1(x1), l1)
        optim.step_all(sgd, c1.parameters(), P.backward(loss))


g = graph.capture(steps, warmup=1)
g.replay()
L.synchronize()
best = 1e9
for _ in range(5):
    e0, e1 = L.Event(), L.Event()
    e0.record()
    g.replay()
    e1.record()
    L.synchronize()
    best = min(best, e0.elapsed_ms(e1) / 50 * 1000)
print(f"config 1: {best:.2f} us/step (graph replay, best of 5 x 50 steps)")
