"""Config-1 step (784-256-10 MLP, SGD) eager: host-launch-bound time per step."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, nn, optim
from paper_2602_00125_b200.data import build_mlp, linear_params

r1 = np.random.default_rng(0)
c1 = build_mlp([linear_params(r1, 784, 256), linear_params(r1, 256, 10)])
x1 = P.from_numpy(r1.standard_normal((256, 784), dtype=np.float32))
l1 = nn.labels_buffer(r1.integers(0, 10, 256))
sgd = optim.SGD(lr=0.01)


def step():
    P.reset_tape()
    loss = nn.cross_entropy(c1(x1), l1)
    optim.step_all(sgd, c1.parameters(), P.backward(loss))
    return loss


for _ in range(5):
    step()
L.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    e0, e1 = L.Event(), L.Event()
    e0.record()
    for _ in range(50):
        step()
    e1.record()
    L.synchronize()
    print(f"eager: {e0.elapsed_ms(e1) / 50 * 1000:.1f} us/step device span, "
          f"{(time.perf_counter() - t0) / 50 * 1e6:.1f} us/step host")

from paper_2602_00125_b200 import graph  # noqa: E402

g1 = graph.capture(step, warmup=1)
g1.replay()
L.synchronize()
for rep in range(3):
    e0, e1 = L.Event(), L.Event()
    e0.record()
    for _ in range(50):
        g1.replay()
    e1.record()
    L.synchronize()
    print(f"graph: {e0.elapsed_ms(e1) / 50 * 1000:.1f} us/step")
