"""Config-2 reductions over a 4096x4096 fp32 tensor (for ncu)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
a = P.from_numpy(np.random.default_rng(0).standard_normal((4096, 4096), dtype=np.float32))
with P.no_grad():
    for _ in range(2):
        P.sum(a); P.sum(a, axis=0); P.sum(a, axis=1); P.max(a, axis=0); P.max(a, axis=1)
L.synchronize()
print("ok")
