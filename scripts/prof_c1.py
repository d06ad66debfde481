"""Config 1 (784-256-10 MLP, batch 256, SGD) steps, eager (for ncu launch lists)."""
import sys
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
for _ in range(3):
    P.reset_tape()
    loss = nn.cross_entropy(c1(x1), l1)
    optim.step_all(sgd, c1.parameters(), P.backward(loss))
L.synchronize()
print("ok", loss.item())
