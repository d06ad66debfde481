import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def load(name):
    with np.load(os.path.join(HERE, name)) as z:
        return {k: z[k] for k in z.files}


def bits_equal(a, b):
    """Bit-exact float32 equality (NaN payload-insensitive, -0 != +0)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    if a.shape != b.shape:
        return False
    an, bn = np.isnan(a), np.isnan(b)
    if not np.array_equal(an, bn):
        return False
    return np.array_equal(a.view(np.uint32)[~an], b.view(np.uint32)[~bn])


def normwise(dev, ref):
    """max|dev-ref| / max|ref| -- the SURVEY 8a.3 tolerance metric."""
    dev = np.asarray(dev, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.max(np.abs(ref)) if ref.size else 0.0
    num = np.max(np.abs(dev - ref)) if ref.size else 0.0
    return num / den if den > 0 else num
