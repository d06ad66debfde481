import sys, numpy as np
sys.path.insert(0, '.')
import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
def ref(A,B,ta,tb):
    a = A.astype(np.float64).T if ta else A.astype(np.float64)
    b = B.astype(np.float64) if tb else B.astype(np.float64).T
    return a @ b.T
for (M,N,K) in [(128,256,32),(128,256,64),(256,512,32),(1000,260,1028)]:
  for ta,tb in [(0,1),(0,0),(1,0),(1,1)]:
    rng=np.random.default_rng(0)
    A = rng.uniform(-1,1,(K,M) if ta else (M,K)).astype(np.float32)
    B = rng.uniform(-1,1,(N,K) if tb else (K,N)).astype(np.float32)
    At,Bt=P.from_numpy(A),P.from_numpy(B)
    r=ref(A,B,ta,tb)
    out=[]
    for algo in (L.GEMM_1XTF32, L.GEMM_3XTF32, L.GEMM_TF32X):
        C=P.zeros((M,N))
        L.call("b2_gemm",ta,tb,M,N,K,At.data_ptr,A.shape[1],Bt.data_ptr,B.shape[1],C.data_ptr,N,None,0,algo,None)
        c=C.numpy()
        err=np.abs(c-r).max()/np.abs(r).max()
        nz=(c!=0).mean()
        # which tiles are wrong
        bad = np.abs(c-r) > 1e-2*np.abs(r).max()
        rows = np.where(bad.any(1))[0]; cols=np.where(bad.any(0))[0]
        out.append(f"algo{algo} err={err:.2e} nz={nz:.2f} badrows={rows[:3]}..{rows[-3:] if len(rows) else ''} nbadrows={len(rows)} badcols={len(cols)}")
    print((M,N,K),ta,tb,' | '.join(out), flush=True)
