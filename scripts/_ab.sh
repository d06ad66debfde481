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
Z = P.from_numpy(rng.standard_normal((32768, 1024), dtype=np.float32))
def c4():
    P.reset_tape(); X.buffer.version += 1; W.buffer.version += 1
    Y = P.softmax(P.add(P.mm(X, W), bias)); P.backward(P.mean(P.mul(Y, Tt)))
def sm():
    with P.no_grad():
        P.softmax(Z)
res = {"lib": L.LIB_PATH.split('/')[-1]}
for name, fn in (("c4_ms", c4), ("softmax_fwd_ms", sm)):
    def body():
        for _ in range(5): fn()
    g = graph.capture(body, warmup=1)
    ts=[]
    for _ in range(5):
        e0, e1 = L.Event(), L.Event(); e0.record(); g.replay(); e1.record(); ts.append(e0.elapsed_ms(e1)/5)
    res[name] = statistics.median(ts)
print(json.dumps(res))
PY
for v in libb2.so libb2_notma.so libb2.so libb2_notma.so; do B2_LIB_PATH=$PWD/paper_2602_00125_b200/$v python /tmp/c4.py; done > gpurun_out/smx2.json 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "softmax or config4" > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/gpu_tests.log
