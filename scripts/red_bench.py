"""Config-2 reductions / fused bwd / exp: median of 7 graph-replay timings
(24 calls rotating over 6 input copies, 384 MiB > L2), GB/s of algorithmic bytes."""
import json, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph

rng = np.random.default_rng(0)
a0 = rng.standard_normal((4096, 4096), dtype=np.float32)
copies = [P.from_numpy(a0) for _ in range(6)]
b = P.from_numpy(rng.uniform(-1, 1, (1, 4096)).astype(np.float32))
n = 4096 * 4096
rot = [0]

def nxt():
    rot[0] = (rot[0] + 1) % len(copies)
    return copies[rot[0]]

def timed(fn, iters=24, reps=7):
    def body():
        for _ in range(iters):
            fn()
    g = graph.capture(body, warmup=1)
    g.replay()
    L.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = L.Event(), L.Event()
        e0.record()
        g.replay()
        e1.record()
        out.append(e0.elapsed_ms(e1) / iters)
    return statistics.median(out)

res = {}
with P.no_grad():
    for name, fn, byt in (
            ("exp", lambda: P.exp(nxt()), 8 * n), ("mul_bcast", lambda: P.mul(nxt(), b), 8 * n),
            ("fused_bwd", lambda: P.muladd_relu_sum_grads(nxt(), b), 8 * n),
            ("sum_dim0", lambda: P.sum(nxt(), axis=0), 4 * n), ("max_dim0", lambda: P.max(nxt(), axis=0), 4 * n),
            ("sum_dim1", lambda: P.sum(nxt(), axis=1), 4 * n), ("max_dim1", lambda: P.max(nxt(), axis=1), 4 * n),
            ("sum_all", lambda: P.sum(nxt()), 4 * n)):
        ms = timed(fn)
        res[name] = round(byt / ms / 1e6)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("B2_")}, **res}))
