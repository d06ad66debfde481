"""The training-loop data path (data.py): the double-buffered batch feeder
(pinned host -> device every step, or resident in HBM) with the first GEMM's
3xBF16 split made on its stream, and the one-step-behind loss reader."""

import numpy as np
import pytest

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
from paper_2602_00125_b200.data import PinnedFeeder, ScalarReader

pytestmark = pytest.mark.gpu


def test_scalar_reader_returns_each_value_one_step_behind():
    r = ScalarReader()
    vals = [1.5, -2.25, 3.0, 1e-7, 42.0]
    got = [r.read(P.from_numpy(np.array(v, np.float32))) for v in vals]
    got.append(r.flush())
    assert got[0] is None
    assert got[1:] == [float(np.float32(v)) for v in vals]
    assert r.flush() is None


@pytest.mark.parametrize("resident", [False, True])
def test_feeder_slots_versions_and_presplit(resident):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((256, 64)).astype(np.float32)
    y = rng.integers(0, 10, 256)
    f = PinnedFeeder(x, y, presplit="3xbf16", resident=resident)
    assert f.h2d_bytes == (0 if resident else x.nbytes + y.nbytes)
    seen = set()
    for _ in range(4):
        xb, yb = f.next()
        L.synchronize()
        assert np.array_equal(xb.numpy(), x)
        lab = np.empty(256, np.int64)
        L.call("b2_memcpy_d2h", lab.ctypes.data, yb.ptr, lab.nbytes, None)
        assert np.array_equal(lab, y)
        ent = xb.buffer._splits[("3xbf16", 0, 256, 64, 64)]
        assert ent[0] == xb.buffer.version  # the split made on the feeder stream is current
        hi = np.empty(256 * 64, np.uint16)
        L.call("b2_memcpy_d2h", hi.ctypes.data, ent[1].ptr, hi.nbytes, None)
        want_hi = (x.view(np.uint32) + 0x7FFF + ((x.view(np.uint32) >> 16) & 1)) >> 16
        assert np.array_equal(hi, want_hi.astype(np.uint16).ravel())
        seen.add(id(xb.buffer))
    assert len(seen) == 2  # two slots, alternating
