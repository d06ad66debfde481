"""Is the fused-epilogue cost on the config-5 dX GEMM a pipeline stall or the
power cap? Each case runs ~1 s back to back while nvidia-smi samples SM clock
and board power; ms/launch and the median clock are printed side by side."""
import statistics
import subprocess
import sys
import threading

sys.path.insert(0, '.')
import numpy as np

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L

M, N, K = 65536, 4096, 4096
rng = np.random.default_rng(0)
g = P.from_numpy(rng.standard_normal((M, K), dtype=np.float32))
w = P.from_numpy(rng.uniform(-1 / 64, 1 / 64, (K, N)).astype(np.float32))
gh, gl, wh, wl = (P.Buffer(2 * M * K), P.Buffer(2 * M * K), P.Buffer(2 * N * K), P.Buffer(2 * N * K))
L.call("b2_bf16x3_split", gh.ptr, gl.ptr, g.data_ptr, M, K, K, None)
L.call("b2_bf16x3_split", wh.ptr, wl.ptr, w.data_ptr, K, N, N, None)
y = P.zeros((M, N))
yh, yl = P.Buffer(2 * M * N), P.Buffer(2 * M * N)
cs = P.zeros((N,))
bits = P.Buffer(8 * M * N // 64)
b = P.zeros((N,))


def desc(emit, col, bit_in, bit_out):
    d = L.GemmDesc()
    d.algo, d.trans_a, d.trans_b, d.M, d.N, d.K = L.GEMM_3XBF16, 0, 0, M, N, K
    d.a[0], d.a[1], d.b[0], d.b[1] = gh.ptr, gl.ptr, wh.ptr, wl.ptr
    d.lda, d.ldb, d.C, d.ldc = K, N, y.data_ptr, N
    d.epilogue = L.EPI_BIAS_RELU if bit_out else 0
    d.bias = b.data_ptr if bit_out else None
    d.mask_bits = bits.ptr if bit_in else None
    d.relu_bits_out = bits.ptr if bit_out else None
    d.c_hi, d.c_lo = (yh.ptr, yl.ptr) if emit else (None, None)
    d.colsum = cs.data_ptr if col else None
    return d


def sample(rows, stop):
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                          "--format=csv,noheader,nounits", "-lms", "50"],
                         stdout=subprocess.PIPE, text=True)
    while not stop.is_set():
        line = p.stdout.readline()
        if not line:
            break
        try:
            rows.append(tuple(float(v) for v in line.split(",")))
        except ValueError:
            pass
    p.terminate()


L.call("b2_gemm_fused", L.ctypes.byref(desc(0, 0, 0, 1)), None)
cases = (("plain", (0, 0, 0, 0)), ("+split", (1, 0, 0, 0)), ("+split+bits+colsum", (1, 1, 1, 0)),
         ("fwd +split+bits_out", (1, 0, 0, 1)))
for r in range(2):
    for name, args in cases:
        d = desc(*args)
        for _ in range(3):
            L.call("b2_gemm_fused", L.ctypes.byref(d), None)
        L.synchronize()
        rows, stop = [], threading.Event()
        t = threading.Thread(target=sample, args=(rows, stop), daemon=True)
        t.start()
        e0, e1 = L.Event(), L.Event()
        e0.record()
        n = 250
        for _ in range(n):
            L.call("b2_gemm_fused", L.ctypes.byref(d), None)
        e1.record()
        L.synchronize()
        stop.set()
        t.join(timeout=2)
        ms = e0.elapsed_ms(e1) / n
        clk = statistics.median(r[0] for r in rows[len(rows) // 4:]) if rows else float("nan")
        pw = statistics.median(r[1] for r in rows[len(rows) // 4:]) if rows else float("nan")
        print(f"{name:22s}: {ms:.3f} ms  {2 * M * N * K / ms / 1e9:.1f} TFLOP/s  sm {clk:.0f} MHz "
              f"power {pw:.0f} W  ({len(rows)} samples)  ms*MHz {ms * clk:.0f}", flush=True)
