"""exp over 4096x4096 (for ncu)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
a = P.from_numpy(np.random.default_rng(0).standard_normal((4096, 4096), dtype=np.float32))
with P.no_grad():
    for _ in range(3):
        P.exp(a)
L.synchronize()
print("ok")
