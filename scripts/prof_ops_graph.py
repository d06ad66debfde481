"""Config-2 ops replayed as ONE CUDA graph (for `ncu --graph-profiling graph`):
the graph's duration and DRAM bytes corroborate bench.py's graph-replay GB/s.
Each op reads its own copy of a (6 x 64 MiB > L2). Prints the algorithmic
bytes of the graph (reads + writes the ops must do)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph

rng = np.random.default_rng(0)
a0 = rng.standard_normal((4096, 4096), dtype=np.float32)
cp = [P.from_numpy(a0) for _ in range(9)]
b = P.from_numpy(rng.uniform(-1, 1, (1, 4096)).astype(np.float32))
n = 4096 * 4096


def ops():
    with P.no_grad():
        P.fused_muladd_relu(cp[0], b)        # read a, write y
        P.muladd_relu_sum_grads(cp[1], b)    # read a, write a_bar
        P.exp(cp[2])                         # read a, write e
        P.mul(cp[3], b)                      # read a, write out
        P.sum(cp[4], axis=0)
        P.max(cp[5], axis=0)
        P.sum(cp[6], axis=1)
        P.max(cp[7], axis=1)
        return P.sum(cp[8])


g = graph.capture(ops, warmup=1)
for _ in range(3):
    g.replay()
L.synchronize()
alg = 4 * n * (2 * 4 + 5)
print("ok algorithmic_bytes", alg)
