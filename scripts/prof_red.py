"""sum/max over dim 0 and dim 1 of a 4096x4096 tensor, 3x each (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
a = P.from_numpy(np.random.default_rng(0).standard_normal((4096, 4096), dtype=np.float32))
with P.no_grad():
    for _ in range(3):
        P.sum(a, axis=0); P.max(a, axis=0); P.sum(a, axis=1); P.max(a, axis=1); P.sum(a)
L.synchronize()
print("ok")
