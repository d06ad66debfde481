cat > /tmp/ce.py <<'PY'
import sys, json, statistics
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph, nn
rng = np.random.default_rng(0)
z = P.from_numpy(rng.standard_normal((65536, 1000), dtype=np.float32), requires_grad=True)
lab = nn.labels_buffer(rng.integers(0, 1000, 65536))
def body():
    for _ in range(5):
        P.reset_tape(); z.buffer.version += 1
        P.backward(nn.cross_entropy(z, lab))
g = graph.capture(body, warmup=1)
ts=[]
for _ in range(5):
    e0, e1 = L.Event(), L.Event(); e0.record(); g.replay(); e1.record(); ts.append(e0.elapsed_ms(e1)/5)
print(json.dumps({"lib": L.LIB_PATH.split('/')[-1], "ce_fwdbwd_us": 1000*statistics.median(ts)}))
PY
for v in libb2.so libb2_minb1.so libb2.so libb2_minb1.so; do B2_LIB_PATH=$PWD/paper_2602_00125_b200/$v python /tmp/ce.py; done > gpurun_out/ce.json 2>&1
