"""Settle scripts/exp_exhaustive.cu's candidates against the reference's exp.

Each record is (x, device, libdevice) as float bits: every float input where
the device's f32 exp differs from f32(libdevice exp(double x)). The reference
computes f32(math.exp(x)) (tensorlite core.py:509; CPython's math.exp is
glibc's exp), so for each candidate the device is right iff it equals that.
Inputs outside the candidate list agree with libdevice; the ones where
libdevice itself is off from glibc are exactly the candidates that settle in
the device's favour. Usage: exp_exhaustive_check.py FILE [FILE ...]"""
import json
import math
import sys

import numpy as np


def glibc_f32(v: float) -> np.float32:
    if math.isnan(v):
        return np.float32("nan")
    try:
        return np.float32(math.exp(v))
    except OverflowError:
        return np.float32("inf")


def settle(path):
    rec = np.fromfile(path, dtype=np.uint32).reshape(-1, 3)
    x = rec[:, 0].view(np.float32)
    dev = rec[:, 1].view(np.float32)
    wrong = []
    for xi, di in zip(x, dev):
        r = glibc_f32(float(xi))
        same = (np.isnan(r) and np.isnan(di)) or r.view(np.uint32) == np.float32(di).view(np.uint32)
        if not same:
            wrong.append(float(xi))
    return {"file": path, "candidates": int(len(x)), "device_wrong": len(wrong), "examples": wrong[:10]}


if __name__ == "__main__":
    print(json.dumps([settle(p) for p in sys.argv[1:]], indent=1))
