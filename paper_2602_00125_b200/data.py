"""Synthetic inputs for the BASELINE configs and a pinned-memory batch feeder.

No dataset is involved anywhere (the reference's demos are
synthetic, BASELINE.json names none); batches come from seeded
numpy.random.default_rng streams with the shapes and distributions of
BASELINE.json's configs.

``PinnedFeeder`` is the host->device path of a training loop: batches live in
page-locked host memory and are copied into device buffers with
cudaMemcpyAsync on the engine stream, so a step's H2D is part of its stream
(this is what bench.py's ``e2e`` number times).
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib as L
from . import core as T


def linear_params(rng, fan_in, fan_out):
    """Kaiming-uniform (PyTorch Linear default) == the reference Dense bound
    U(+-1/sqrt(in)) for W and b (nn.py:64-76)."""
    bound = 1.0 / math.sqrt(fan_in)
    w = rng.uniform(-bound, bound, size=(fan_out, fan_in)).astype(np.float32)
    b = rng.uniform(-bound, bound, size=fan_out).astype(np.float32)
    return w, b


def mlp_config5(seed=0, width=4096, classes=1000, depth=4):
    """BASELINE config 5 parameters: depth x Linear(width,width)+ReLU, then
    Linear(width, classes)."""
    rng = np.random.default_rng(seed)
    params = [linear_params(rng, width, width) for _ in range(depth)]
    params.append(linear_params(rng, width, classes))
    return params


def batch_shard(seed, rank, rows, width, classes):
    """This rank's rows of the global batch: x ~ N(0,1) f32, labels ~ U{0..C-1}."""
    rng = np.random.default_rng([seed, rank])
    x = rng.standard_normal((rows, width), dtype=np.float32)
    labels = rng.integers(0, classes, size=rows, dtype=np.int64)
    return x, labels


def build_mlp(params):
    """nn.Sequential of Dense(+ReLU) layers with the given (W, b) values."""
    from . import nn

    layers = []
    for i, (w, b) in enumerate(params):
        d = nn.Dense.__new__(nn.Dense)
        nn.Layer.__init__(d)
        d.in_features, d.out_features = w.shape[1], w.shape[0]
        d.weight = T.from_numpy(w, requires_grad=True)
        d.bias = T.from_numpy(b, requires_grad=True)
        layers.append(d)
        if i < len(params) - 1:
            layers.append(nn.ReLU())
    return nn.Sequential(*layers)


class PinnedHost:
    """A page-locked host array (cudaMallocHost) viewed as a numpy array."""

    def __init__(self, shape, dtype):
        L.ensure_device()
        self.nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
        p = ctypes.c_void_p()
        L.check(L.lib().b2_host_alloc(max(self.nbytes, 1), ctypes.byref(p)))
        self.ptr = p.value
        buf = (ctypes.c_char * max(self.nbytes, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def __del__(self):
        try:
            if self.ptr and L._lib is not None:
                L._lib.b2_host_free(self.ptr)
        except Exception:
            pass


class PinnedFeeder:
    """Host batch (pinned) -> device tensor + int64 label buffer, every step.

    Double-buffered: while step i computes on slot i%2, the H2D copy of step
    i+1's batch runs on a dedicated copy stream into the other slot (the
    copy waits until the compute stream has released that slot; the compute
    stream waits until its slot's copy has landed). Every step still moves its
    full batch host -> device; the copy just overlaps the previous step."""

    def __init__(self, x, labels, presplit=None, resident=False, classes=None):
        """presplit="3xbf16": also make each batch's 3xBF16 operand split on
        the copy stream right after its H2D copy (the first layer's GEMM reads
        x only through that split), so the split of step i+1's batch overlaps
        step i instead of opening step i+1.
        resident=True: the batch is uploaded once into both device slots and
        stays in HBM (bench.py's device-resident `value` loop); each step
        still redoes its split (when presplit) on the copy stream."""
        self.presplit = presplit
        self.resident = resident
        labels = np.asarray(labels)
        if classes is not None and labels.size and (labels.min() < 0 or labels.max() >= classes):
            bad = int(labels[(labels < 0) | (labels >= classes)][0])
            raise ValueError(f"label {bad} out of range for {classes} classes")
        self.copy_stream = None
        self.hx = PinnedHost(x.shape, np.float32)
        self.hx.array[...] = x
        self.hl = PinnedHost(labels.shape, np.int64)
        self.hl.array[...] = labels
        self.dx = [T._empty(x.shape) for _ in range(2)]
        self.dl = [T.Buffer(8 * max(labels.size, 1)) for _ in range(2)]
        rows, cols = (x.shape[0], int(np.prod(x.shape[1:]))) if x.ndim > 1 else (1, x.size)
        self._rc = (rows, cols)
        if presplit not in (None, "3xbf16"):
            raise ValueError("presplit must be None or '3xbf16'")
        if presplit and cols % 8:
            self.presplit = None  # the split kernel needs cols % 8 == 0; the GEMM splits itself
        self.sp = [(T.Buffer(2 * rows * cols), T.Buffer(2 * rows * cols)) for _ in range(2)] \
            if self.presplit else None
        s = ctypes.c_void_p()
        L.check(L.lib().b2_stream_create(ctypes.byref(s)))
        self.copy_stream = s.value
        self.ready = [L.Event(), L.Event()]
        self.released = [L.Event(), L.Event()]
        self.i = 0
        if resident:
            for slot in range(2):
                L.call("b2_memcpy_h2d", self.dx[slot].data_ptr, self.hx.ptr, self.hx.nbytes, None)
                L.call("b2_memcpy_h2d", self.dl[slot].ptr, self.hl.ptr, self.hl.nbytes, None)
            L.synchronize()
        self._issue(0)

    def close(self):
        """Drain the copy stream (a queued copy or split may still write the
        slots) and destroy it; the slot buffers are then safe to free."""
        cs, self.copy_stream = self.copy_stream, None
        if cs is not None and L._lib is not None:
            L._lib.b2_stream_sync(cs)
            L._lib.b2_stream_destroy(cs)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def h2d_bytes(self):
        return 0 if self.resident else self.hx.nbytes + self.hl.nbytes

    def _issue(self, slot):
        cs = self.copy_stream
        if not self.resident:
            L.call("b2_memcpy_h2d", self.dx[slot].data_ptr, self.hx.ptr, self.hx.nbytes, cs)
            L.call("b2_memcpy_h2d", self.dl[slot].ptr, self.hl.ptr, self.hl.nbytes, cs)
        if self.sp is not None:
            hi, lo = self.sp[slot]
            rows, cols = self._rc
            L.call("b2_bf16x3_split", hi.ptr, lo.ptr, self.dx[slot].data_ptr, rows, cols, cols, cs)
        self.ready[slot].record(cs)

    def next(self):
        """Returns this step's (x, labels); queues the next step's copy."""
        cur, nxt = self.i % 2, (self.i + 1) % 2
        L.call("b2_stream_wait_event", None, self.ready[cur].h)  # this slot's batch landed
        # the previous step (already queued) was the last user of `nxt`
        self.released[nxt].record(None)
        L.call("b2_stream_wait_event", self.copy_stream, self.released[nxt].h)
        self._issue(nxt)
        self.i += 1
        buf = self.dx[cur].buffer
        buf.version += 1  # a new batch: cached operand splits are stale
        if self.sp is not None:  # ... except the one made with it on the copy stream
            from .graph import _capturing

            rows, cols = self._rc
            if buf._splits is None:
                buf._splits = {}
            hi, lo = self.sp[cur]
            buf._splits[("3xbf16", 0, rows, cols, cols)] = (buf.version, hi, lo, _capturing[0])
        return self.dx[cur], self.dl[cur]


class ScalarReader:
    """Reads a device scalar (a step's loss) to the host without draining the
    stream: read(t) queues a D2H copy into a pinned slot plus an event and
    returns the PREVIOUS read's value (waiting only for that older copy), so
    the host queues step i+1 before it blocks on step i's loss. flush()
    returns the last one."""

    def __init__(self, slots=2):
        self.host = PinnedHost((slots,), np.float32)
        self.events = [L.Event() for _ in range(slots)]
        self.i = 0
        self.pending = None

    def read(self, t):
        slot = self.i % len(self.events)
        self.i += 1
        L.call("b2_memcpy_d2h_async", self.host.ptr + 4 * slot, t.data_ptr, 4, None)
        self.events[slot].record()
        prev, self.pending = self.pending, slot
        return self._value(prev)

    def _value(self, slot):
        if slot is None:
            return None
        self.events[slot].synchronize()
        return float(self.host.array[slot])

    def flush(self):
        prev, self.pending = self.pending, None
        return self._value(prev)

