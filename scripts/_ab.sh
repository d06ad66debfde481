cat > /tmp/c4.py <<'PY'
import sys, json, statistics
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph
rng = np.random.default_rng(0)
X = P.from_numpy(rng.standard_normal((64, 512, 1024), dtype=np.float32), requires_grad=True)
W = P.from_numpy(rng.normal(0, 0.03, (1024, 1024)).astype(np.float32), requires_grad=True)
bias = P.zeros((1024,), requires_grad=True)
Tt = P.from_numpy(rng.uniform(0, 1, (64, 512, 1024)).astype(np.float32))
def c4():
    P.reset_tape(); X.buffer.version += 1; W.buffer.version += 1
    Y = P.softmax(P.add(P.mm(X, W), bias)); P.backward(P.mean(P.mul(Y, Tt)))
def body():
    for _ in range(5): c4()
g = graph.capture(body, warmup=1)
ts=[]
for _ in range(5):
    e0, e1 = L.Event(), L.Event(); e0.record(); g.replay(); e1.record(); ts.append(e0.elapsed_ms(e1)/5)
print(json.dumps({"lib": L.LIB_PATH.split('/')[-1], "c4_ms": statistics.median(ts)}))
PY
for v in libb2_smx3.so libb2.so libb2_smx4.so libb2.so libb2_smx3.so; do B2_LIB_PATH=$PWD/paper_2602_00125_b200/$v python /tmp/c4.py; done > gpurun_out/smx.json 2>&1
