import numpy as np, sys
a=np.load(sys.argv[1]); b=np.load(sys.argv[2])
M,N=16384,4096
x=a["0_C"].view(np.float32).reshape(M,N); y=b["0_C"].view(np.float32).reshape(M,N)
d=np.abs(x-y)
print("maxdiff", d.max(), "max|y|", np.abs(y).max(), "frac differing", (x!=y).mean())
rows=np.where((x!=y).any(1))[0]; cols=np.where((x!=y).any(0))[0]
print("rows differing", len(rows), rows[:20], "cols", len(cols), cols[:20])
r=rows[0] if len(rows) else 0
print("row", r, x[r,:8], y[r,:8])
# pattern by row mod 512
if len(rows):
    print("row mod 512 hist", np.bincount(rows%512//64, minlength=8))
