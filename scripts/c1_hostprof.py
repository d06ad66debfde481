"""Host-side profile of the eager config-1 step (cProfile, top cumulative entries)."""
import cProfile, pstats, sys, time
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


for _ in range(20):
    step()
L.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    step()
t1 = time.perf_counter()
L.synchronize()
t2 = time.perf_counter()
print(f"host {1e6 * (t1 - t0) / 200:.1f} us/step, with drain {1e6 * (t2 - t0) / 200:.1f} us/step")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    step()
pr.disable()
L.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(28)
