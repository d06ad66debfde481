"""Config 2 in one pass (b2_muladd_relu_stats) vs the composed ops, graph-replayed
over rotating input copies (> L2)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph

rng = np.random.default_rng(0)
a0 = rng.standard_normal((4096, 4096), dtype=np.float32)
cps = [P.from_numpy(a0) for _ in range(6)]
b = P.from_numpy(rng.uniform(-1, 1, (1, 4096)).astype(np.float32))
i = [0]


def nxt():
    i[0] = (i[0] + 1) % 6
    return cps[i[0]]


def t(name, fn, n=12):
    g = graph.capture(lambda: [fn() for _ in range(n)], warmup=1)
    g.replay()
    L.synchronize()
    e0, e1 = L.Event(), L.Event()
    e0.record()
    g.replay()
    e1.record()
    us = e0.elapsed_ms(e1) / n * 1000
    print(f"{name:24s} {us:8.1f} us  {256 * 2**20 / us / 1e6:6.2f} TB/s of the 256 MiB single-pass bytes")


t("single pass", lambda: P.muladd_relu_stats(nxt(), b))
