"""Config 3 at n=1024 (square matmul fwd+bwd), a few iterations, for an ncu launch list."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
rng = np.random.default_rng(0)
A = P.from_numpy(rng.uniform(-1, 1, (n, n)).astype(np.float32), requires_grad=True)
B = P.from_numpy(rng.uniform(-1, 1, (n, n)).astype(np.float32), requires_grad=True)
dC = P.from_numpy(rng.standard_normal((n, n), dtype=np.float32))
for _ in range(3):
    P.reset_tape()
    A.buffer.version += 1
    B.buffer.version += 1
    C = P.mm(A, B)
    P.backward(C, seed=dC)
L.synchronize()
print("ok")
