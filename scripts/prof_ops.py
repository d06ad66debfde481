"""Config-2 ops on a 4096x4096 fp32 tensor (for ncu): exp, mul-broadcast,
fused relu(a*b+b) fwd/bwd, sum/max over dim 0 / dim 1, full sum."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L

rng = np.random.default_rng(0)
a = P.from_numpy(rng.standard_normal((4096, 4096), dtype=np.float32))
b = P.from_numpy(rng.uniform(-1, 1, (1, 4096)).astype(np.float32))
with P.no_grad():
    for _ in range(2):
        P.exp(a)
        P.mul(a, b)
        P.fused_muladd_relu(a, b)
        P.muladd_relu_sum_grads(a, b)
        P.sum(a, axis=0)
        P.max(a, axis=0)
        P.sum(a, axis=1)
        P.max(a, axis=1)
        P.sum(a)
L.synchronize()
print("ok")
