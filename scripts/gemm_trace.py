"""Phase timeline of a few-tile GEMM from a trace build of gemm_tc.cu
(-DB2_GEMM_TRACE: %globaltimer stamps at entry, prologue done, prerequisite
grids done, first operands landed, last chunk's MMAs done, stores issued, all
warps done, teardown -- per CTA). Build here, run on the GPU box:

    python scripts/gemm_trace.py --build      # -> scripts/_trace/libb2_trace.so
    python scripts/gemm_trace.py 1024 1024 64
"""
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "scripts", "_trace", "libb2_trace.so")

if "--build" in sys.argv:
    sys.path.insert(0, ROOT)
    from paper_2602_00125_b200 import build as B

    B.build()
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    obj = os.path.join(os.path.dirname(OUT), "gemm_tc_trace.o")
    subprocess.run([B._nvcc()] + B.ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                    "-DB2_GEMM_TRACE", "-I", os.path.join(ROOT, "include"), "-I", B.CSRC, "-I",
                    B._nccl_include(), "-c", os.path.join(B.CSRC, "gemm_tc.cu"), "-o", obj], check=True)
    objs = [o for o in glob.glob(os.path.join(B.BUILD, "*.o")) if not o.endswith("gemm_tc.o")] + [obj]
    subprocess.run([B._nvcc()] + B.ARCH + ["-shared", "-o", OUT] + objs + ["-ldl", "-lpthread", "-lrt"],
                   check=True)
    print(OUT)
    sys.exit(0)

os.environ["B2_LIB_PATH"] = OUT
sys.path.insert(0, ROOT)
import ctypes  # noqa: E402

import numpy as np  # noqa: E402

import paper_2602_00125_b200 as P  # noqa: E402
from paper_2602_00125_b200 import _lib as L  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4])
rng = np.random.default_rng(0)
a = P.from_numpy(rng.uniform(-1, 1, (M, K)).astype(np.float32))
b = P.from_numpy(rng.uniform(-1, 1, (N, K)).astype(np.float32))
ah, al, bh, bl = P.Buffer(2 * M * K), P.Buffer(2 * M * K), P.Buffer(2 * N * K), P.Buffer(2 * N * K)
L.call("b2_bf16x3_split", ah.ptr, al.ptr, a.data_ptr, M, K, K, None)
L.call("b2_bf16x3_split", bh.ptr, bl.ptr, b.data_ptr, N, K, K, None)
c = P.zeros((M, N))
for _ in range(4):  # the last launch's stamps survive
    L.call("b2_gemm_3xbf16", 0, 1, M, N, K, ah.ptr, al.ptr, bh.ptr, bl.ptr, c.data_ptr, N, None, 0,
           None, None, None, None, None)
L.synchronize()
buf = (ctypes.c_ulonglong * (1024 * 8))()
assert L.lib().b2_gemm_trace_read(buf) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8).astype(np.int64)
used = t[:, 0] > 0
t = t[used]
t0 = t[:, 0].min()
names = ["entry", "prologue", "griddep", "operands", "mma_done", "stores", "alldone", "teardown"]
print(f"GEMM {M}x{N}x{K}: {used.sum()} CTAs; us after the first CTA's entry (min / median / max over CTAs)")
for j, nm in enumerate(names):
    col = t[:, j]
    col = col[col > 0]
    if col.size:
        print(f"  {nm:9s} {(col.min() - t0) / 1e3:7.2f} {(np.median(col) - t0) / 1e3:7.2f} {(col.max() - t0) / 1e3:7.2f}")
