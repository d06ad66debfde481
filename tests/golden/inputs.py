"""Seeded synthetic inputs for the BASELINE configs.

numpy.random.default_rng streams are stable across NumPy versions, so the
same seed reproduces the same f32 arrays here and on the GPU box. Values are
drawn in float64 and cast to float32 once; both the reference and the device
engine consume the identical f32 arrays.
"""

from __future__ import annotations

import math
import random

import numpy as np


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def kaiming_linear(rng, fan_in, fan_out, zero_bias=True):
    """PyTorch Linear default (kaiming_uniform a=sqrt(5)) == U(+-1/sqrt(in)),
    the same bound as the reference Dense (nn.py:64-76)."""
    bound = 1.0 / math.sqrt(fan_in)
    w = _f32(rng.uniform(-bound, bound, size=(fan_out, fan_in)))
    b = np.zeros(fan_out, np.float32) if zero_bias else _f32(rng.uniform(-bound, bound, fan_out))
    return w, b


def config1_inputs(seed=0, batch=256):
    rng = np.random.default_rng(seed)
    x = _f32(rng.standard_normal((batch, 784)))
    p0 = kaiming_linear(rng, 784, 256)
    p1 = kaiming_linear(rng, 256, 10)
    labels = rng.integers(0, 10, size=batch, dtype=np.int64)
    return [p0, p1], x, labels


def config2_inputs(seed=0, rows=4096, cols=4096):
    rng = np.random.default_rng(seed)
    a = _f32(rng.standard_normal((rows, cols)))
    b = _f32(rng.uniform(-1.0, 1.0, size=(1, cols)))
    return a, b


def config3_inputs(seed=0, n=1024):
    rng = np.random.default_rng(seed)
    A = _f32(rng.uniform(-1.0, 1.0, size=(n, n)))
    B = _f32(rng.uniform(-1.0, 1.0, size=(n, n)))
    dC = _f32(rng.standard_normal((n, n)))
    return A, B, dC


def config4_inputs(seed=0, b=64, s=512, k=1024):
    rng = np.random.default_rng(seed)
    X = _f32(rng.standard_normal((b, s, k)))
    W = _f32(rng.normal(0.0, 0.03, size=(k, k)))
    bias = np.zeros(k, np.float32)
    T = _f32(rng.uniform(0.0, 1.0, size=(b, s, k)))
    return X, W, bias, T


def config5_inputs(seed=0, width=4096, classes=1000, batch=65536, depth=4,
                   zero_bias=False):
    """4 x Linear(4096,4096)+ReLU, Linear(4096,1000); W,b ~ U(+-1/sqrt(in))
    (the reference Dense init)."""
    rng = np.random.default_rng(seed)
    params = [kaiming_linear(rng, width, width, zero_bias) for _ in range(depth)]
    params.append(kaiming_linear(rng, width, classes, zero_bias))
    x = _f32(rng.standard_normal((batch, width)))
    labels = rng.integers(0, classes, size=batch, dtype=np.int64)
    return params, x, labels


# --------------------------------------------------------------------------- small cases


def broadcast_cases(n=60, seed=2000):
    """Random broadcast-compatible pairs, <=4-D, dims 1..5, like the
    reference's acceptance sweep (tests/test_acceptance.py:97-119) but with
    general float values instead of small integers."""
    ops = ("add", "sub", "mul", "div")
    out = []
    for i in range(n):
        r = random.Random(seed + i)
        g = np.random.default_rng(seed + i)
        ndim = r.randint(0, 4)
        target = [r.randint(1, 5) for _ in range(ndim)]

        def degrade():
            s = [d if r.random() < 0.6 else 1 for d in target]
            return tuple(s[r.randint(0, max(ndim - 1, 0)):]) if (ndim and r.random() < 0.3) else tuple(s)

        sa, sb = degrade(), degrade()
        va = _f32(g.standard_normal(sa) * 3.0)
        vb = _f32(g.standard_normal(sb) * 3.0)
        kind = ops[i % 4]
        if kind == "div":
            vb = np.where(np.abs(vb) < 1e-3, np.float32(1.0), vb).astype(np.float32)
        out.append((kind, va, vb))
    return out


def unary_values():
    g = np.random.default_rng(7)
    v = list(g.standard_normal(200) * 4.0) + [0.0, -0.0, 1000.0, -1000.0, 88.5, -104.0,
                                              float("inf"), float("-inf"), 1e-30, -1e-30,
                                              3.0e38, 0.5, 2.0, 100.0]
    return _f32(v)


def reduction_cases(n=40, seed=500):
    out = []
    for i in range(n):
        r = random.Random(seed + i)
        g = np.random.default_rng(seed + i)
        ndim = r.randint(1, 4)
        shape = tuple(r.randint(1, 6) for _ in range(ndim))
        if i % 3 == 0:  # small integers -> exact ties exercise first-max routing
            x = _f32(g.integers(-3, 4, size=shape))
        else:
            x = _f32(g.standard_normal(shape))
        if i % 7 == 0:
            axes = None
        else:
            k = r.randint(1, ndim)
            axes = tuple(r.sample(range(ndim), k))
        keep = r.random() < 0.5
        out.append((x, axes, keep))
    # the BASELINE-shaped 2-D cases at a reduced size
    g = np.random.default_rng(99)
    y = _f32(np.maximum(g.standard_normal((64, 96)), 0))
    out += [(y, (0,), False), (y, (1,), False), (y, None, False), (y, (-1,), True)]
    return out


def matmul_cases():
    g = np.random.default_rng(3)
    shapes = [(1, 1, 1), (3, 5, 4), (7, 16, 9), (33, 65, 17), (64, 128, 48), (5, 0, 3)]
    out = []
    for m, k, d in shapes:
        x = _f32(g.uniform(-1, 1, size=(m, k)))
        w = _f32(g.uniform(-1, 1, size=(d, k)))
        gr = _f32(g.standard_normal((m, d)))
        out.append((x, w, gr))
    return out


def ce_cases():
    g = np.random.default_rng(5)
    out = []
    for b, c in ((1, 2), (4, 10), (37, 13), (64, 1000)):
        z = _f32(g.standard_normal((b, c)) * 3.0)
        labels = g.integers(0, c, size=b, dtype=np.int64)
        out.append((z, labels))
    # huge logits stay finite (tests/test_nn.py:450-455)
    out.append((_f32([[1.0e4, -1.0e4, 0.0], [5.0e3, 5.0e3, -5.0e3]]), np.array([0, 1], np.int64)))
    return out


# Conv2D cases of tests/golden/catalog.npz:
# (B, C_in, H, W, C_out, (kh, kw), stride, padding, bias)
CONV_CASES = [
    (2, 3, 7, 7, 4, (3, 3), 1, 1, True),
    (2, 2, 5, 5, 2, (3, 3), 2, 1, True),
    (1, 3, 6, 5, 5, (2, 3), 1, 0, False),
    (3, 4, 4, 4, 8, (1, 1), 1, 0, True),
    (2, 1, 9, 8, 3, (4, 4), 3, 2, True),
]
