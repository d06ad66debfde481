"""Per-GEMM breakdown of the config-5 train step (bench.py's step, N = 1):
every GEMM launch's shape, layout, device time (CUDA events on the engine
stream, incl. its K-slice second stage / column-sum kernels) and rate, plus
the step time, so the GEMMs furthest below the forward GEMM's rate show.
usage: python scripts/step_gemms.py [--batch 65536] [--steps 3]"""
import argparse
import collections
import sys

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_2602_00125_b200 as P  # noqa: E402
from paper_2602_00125_b200 import _lib as L, dist, nn, optim  # noqa: E402
from paper_2602_00125_b200 import core as C  # noqa: E402
from paper_2602_00125_b200.data import PinnedFeeder, build_mlp, mlp_config5, batch_shard  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=65536)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--algo", default=None)
args = ap.parse_args()
if args.algo:
    P.set_gemm_algo(args.algo)
W, CLS, DEPTH = 4096, 1000, 4
env = dist.env_from_os()
comm = dist.Communicator(env)
model = build_mlp(mlp_config5(0, W, CLS, DEPTH))
params = model.parameters()
opt = optim.Adam(lr=1e-3, betas=(0.9, 0.999), eps=1e-8)
x_np, y_np = batch_shard(1234, 0, args.batch, W, CLS)
feeder = PinnedFeeder(x_np, y_np, presplit="3xbf16" if not args.algo else None, resident=True,
                      classes=CLS)

def step2():
    x, y = feeder.next()
    P.reset_tape()
    loss = nn.cross_entropy(model(x), y, denom=args.batch)
    red = dist.GradReducer(comm, params, optimizer=opt)
    store = P.backward(loss, on_leaf_ready=red.hook)
    red.finish()
    red.step_rest(store)
    return loss


for _ in range(4):
    step2()
L.synchronize()
e0, e1 = L.Event(), L.Event()
e0.record()
for _ in range(args.steps):
    step2()
e1.record()
L.synchronize()
step_ms = e0.elapsed_ms(e1) / args.steps
log, labels = [], []
C.GEMM_TIMER, C.GEMM_TIMER_LABELS = log, labels
e0.record()
for _ in range(args.steps):
    step2()
e1.record()
L.synchronize()
C.GEMM_TIMER = C.GEMM_TIMER_LABELS = None
timed_ms = e0.elapsed_ms(e1) / args.steps
agg = collections.OrderedDict()
for (fl, s, e), lab in zip(log, labels):
    agg.setdefault(lab, []).append((fl, s.elapsed_ms(e)))
tot = 0.0
print(f"batch {args.batch}: step {step_ms:.3f} ms (timed pass {timed_ms:.3f} ms)")
print("launch (M N K tA tB per problem)                     n   ms/launch  TF/s(fp32-eq)")
for lab, v in agg.items():
    ms = np.mean([t for _, t in v])
    fl = v[0][0]
    tot += ms * len(v) / args.steps
    name = " + ".join(f"{m}x{n}x{k}{'T' if a else 'N'}{'N' if b else 'T'}" for m, n, k, a, b in lab)
    print(f"{name:52s} {len(v) // args.steps:3d} {ms:10.3f}  {fl / ms / 1e9:8.1f}")
print(f"GEMM total {tot:.3f} ms = {tot / timed_ms:.1%} of the step")
