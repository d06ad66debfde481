"""Fused config-4 loss rows at the same bytes but half the row width ([65536, 512] vs [32768, 1024]):
half the per-lane registers. With a library built -DB2_WMEAN_MINB=4 this probes what more resident
warps would buy a 2-warps-per-row variant. python scripts/wmean_occupancy_probe.py"""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L, graph

MB = 1 << 20
rng = np.random.default_rng(0)
for R, K in ((32768, 1024), (65536, 512)):
    T = P.from_numpy(rng.uniform(0, 1, (R, K)).astype(np.float32))
    Z = P.from_numpy(rng.standard_normal((R, K), dtype=np.float32))
    g, loss = P.ones(()), P.zeros(())
    rs, rm, rdot = P.Buffer(4 * R), P.Buffer(4 * R), P.Buffer(8 * R)
    hi, lo = P.Buffer(2 * R * K), P.Buffer(2 * R * K)
    cs = P.zeros((K,))

    def t(name, fn, gbytes, n=10):
        gr = graph.capture(lambda: [fn() for _ in range(n)], warmup=1)
        gr.replay()
        L.synchronize()
        e0, e1 = L.Event(), L.Event()
        e0.record()
        gr.replay()
        e1.record()
        us = e0.elapsed_ms(e1) / n * 1000
        print(f"[{R} x {K}] {name:12s} {us:8.1f} us  {gbytes / us * 1e-3:.2f} TB/s", flush=True)

    t("wmean_fwd", lambda: L.call("b2_softmax_wmean_fwd", loss.data_ptr, None, rs.ptr, rm.ptr, rdot.ptr,
                                  Z.data_ptr, T.data_ptr, R, K, None), 256 * MB)
    t("wmean_bwd", lambda: L.call("b2_softmax_wmean_bwd", None, hi.ptr, lo.ptr, cs.data_ptr, g.data_ptr,
                                  float(R * K), Z.data_ptr, T.data_ptr, rs.ptr, rm.ptr, R, K, None), 384 * MB)
    del T, Z, hi, lo
