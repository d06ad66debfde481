import sys, numpy as np
sys.path.insert(0, '.')
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
rng = np.random.default_rng(0)
M = N = 1024
for K in (256, 1024, 4096, 8192):
    A = rng.uniform(-1,1,(M,K)).astype(np.float32); B = rng.uniform(-1,1,(N,K)).astype(np.float32)
    # tf32-exact inputs: mask low 13 bits
    Ah = (A.view(np.uint32) & 0xFFFFE000).view(np.float32); Bh = (B.view(np.uint32) & 0xFFFFE000).view(np.float32)
    ref = Ah.astype(np.float64) @ Bh.astype(np.float64).T
    At, Bt = P.from_numpy(Ah), P.from_numpy(Bh)
    C = P.zeros((M,N))
    L.call("b2_gemm",0,1,M,N,K,At.data_ptr,K,Bt.data_ptr,K,C.data_ptr,N,None,0,L.GEMM_1XTF32,None)
    c = C.numpy().astype(np.float64)
    e1 = np.abs(c-ref).max()/np.abs(ref).max()
    bias = np.mean(c-ref)/np.abs(ref).max()
    # fp32 RN reference: float32 accumulate sequentially in numpy? approximate with chunked fp32 dot via einsum float32
    c32 = (Ah @ Bh.T).astype(np.float64)  # numpy float32 gemm (blas sgemm)
    e32 = np.abs(c32-ref).max()/np.abs(ref).max()
    out = [f"K={K} tc-acc err={e1:.2e} bias={bias:.2e} sgemm err={e32:.2e}"]
    for ch in (128, 256, 512):
        if ch >= K: continue
        tot = np.zeros((M,N))
        Cc = P.zeros((M,N))
        for k0 in range(0, K, ch):
            a = P.from_numpy(np.ascontiguousarray(Ah[:, k0:k0+ch])); b = P.from_numpy(np.ascontiguousarray(Bh[:, k0:k0+ch]))
            L.call("b2_gemm",0,1,M,N,ch,a.data_ptr,ch,b.data_ptr,ch,Cc.data_ptr,N,None,0,L.GEMM_1XTF32,None)
            tot = (tot.astype(np.float32) + Cc.numpy()).astype(np.float64)  # fp32 RN combine
        out.append(f"chunk{ch}+fp32RN err={np.abs(tot-ref).max()/np.abs(ref).max():.2e}")
    print(" | ".join(out), flush=True)
