import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
def timeit(fn, iters=10):
    fn(); L.synchronize()
    e0, e1 = L.Event(), L.Event()
    e0.record(); 
    for _ in range(iters): fn()
    e1.record(); return e0.elapsed_ms(e1) / iters
for n in (1024, 4096, 8192):
    rng = np.random.default_rng(0)
    A = rng.uniform(-1,1,(n,n)).astype(np.float32); B = rng.uniform(-1,1,(n,n)).astype(np.float32)
    At, Bt = P.from_numpy(A), P.from_numpy(B)
    C = P.zeros((n,n))
    ref = None
    if n <= 4096:
        ref = A.astype(np.float64) @ B.astype(np.float64).T
    for name, algo in (("1xtf32", L.GEMM_1XTF32), ("3xtf32", L.GEMM_3XTF32), ("tf32x", L.GEMM_TF32X), ("3xbf16", L.GEMM_3XBF16), ("simt", L.GEMM_SIMT)):
        if name == "simt" and n > 4096: continue
        f = lambda: L.call("b2_gemm", 0, 1, n, n, n, At.data_ptr, n, Bt.data_ptr, n, C.data_ptr, n, None, 0, algo, None)
        ms = timeit(f, 5 if n == 8192 else 10)
        err = ""
        if ref is not None:
            c = C.numpy(); err = f"err={np.abs(c-ref).max()/np.abs(ref).max():.2e}"
        print(f"n={n} {name}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s {err}", flush=True)
    # presplit kernel alone
    if True:
        hi, lo, hib, lob = P.zeros((n,n)), P.zeros((n,n)), P.zeros((n,n)), P.zeros((n,n))
        L.call("b2_tf32_split", hi.data_ptr, lo.data_ptr, At.data_ptr, n, n, n, None)
        L.call("b2_tf32_split", hib.data_ptr, lob.data_ptr, Bt.data_ptr, n, n, n, None)
        f = lambda: L.call("b2_gemm_presplit", 0, 1, n, n, n, hi.data_ptr, lo.data_ptr, hib.data_ptr, lob.data_ptr, C.data_ptr, n, None, 0, None)
        ms = timeit(f, 5)
        print(f"n={n} 3xtf32-presplit kernel: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
        f = lambda: L.call("b2_tf32_split", hi.data_ptr, lo.data_ptr, At.data_ptr, n, n, n, None)
        ms = timeit(f, 10)
        print(f"n={n} split: {ms:.3f} ms  {3*4*n*n/ms/1e6:.0f} GB/s", flush=True)
        h16, l16, hb16, lb16 = [P.zeros((n, n // 2)) for _ in range(4)]
        L.call("b2_bf16x2_split", h16.data_ptr, l16.data_ptr, At.data_ptr, n, n, n, None)
        L.call("b2_bf16x2_split", hb16.data_ptr, lb16.data_ptr, Bt.data_ptr, n, n, n, None)
        for ta, tb in ((0, 1), (0, 0), (1, 0)):
            f = lambda: L.call("b2_gemm_tf32x", ta, tb, n, n, n, At.data_ptr, n, h16.data_ptr, l16.data_ptr, Bt.data_ptr, n, hb16.data_ptr, lb16.data_ptr, C.data_ptr, n, None, 0, None)
            ms = timeit(f, 5)
            print(f"n={n} tf32x-presplit kernel ta={ta} tb={tb}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
        f = lambda: L.call("b2_bf16x2_split", h16.data_ptr, l16.data_ptr, At.data_ptr, n, n, n, None)
        ms = timeit(f, 10)
        print(f"n={n} bf16x2 split: {ms:.3f} ms  {2*4*n*n/ms/1e6:.0f} GB/s", flush=True)
        for ta, tb in ((0, 1), (0, 0), (1, 0)):
            L.call("b2_bf16x3_split", h16.data_ptr, l16.data_ptr, At.data_ptr, n, n, n, None)
            L.call("b2_bf16x3_split", hb16.data_ptr, lb16.data_ptr, Bt.data_ptr, n, n, n, None)
            f = lambda: L.call("b2_gemm_3xbf16", ta, tb, n, n, n, h16.data_ptr, l16.data_ptr, hb16.data_ptr, lb16.data_ptr, C.data_ptr, n, None, 0, None, None, None, None, None)
            ms = timeit(f, 5)
            print(f"n={n} 3xbf16-presplit kernel ta={ta} tb={tb}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
        a16, b16 = P.zeros((n, n // 2)), P.zeros((n, n // 2))
        L.call("b2_bf16_cast", a16.data_ptr, At.data_ptr, n, n, n, None)
        L.call("b2_bf16_cast", b16.data_ptr, Bt.data_ptr, n, n, n, None)
        for ta, tb in ((0, 1), (0, 0), (1, 0)):
            f = lambda: L.call("b2_gemm_bf16", ta, tb, n, n, n, a16.data_ptr, b16.data_ptr, C.data_ptr, n, None, 0, None, None, None, None)
            ms = timeit(f, 10)
            print(f"n={n} bf16 kernel ta={ta} tb={tb}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
        try:
            import torch
            ta_, tb_ = torch.randn(n, n, device="cuda", dtype=torch.bfloat16), torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(3): ta_ @ tb_.T
            s.record()
            for _ in range(10): ta_ @ tb_.T
            e.record(); torch.cuda.synchronize()
            ms = s.elapsed_time(e) / 10
            print(f"n={n} cublas bf16 (torch, context only): {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
        except Exception as ex:
            print("torch cublas unavailable", ex)
