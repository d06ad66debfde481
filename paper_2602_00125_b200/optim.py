"""SGD / Adam / RMSprop as single multi-tensor kernel launches (tensorlite/optim.py).

Semantics follow optim.py:16-136: per-parameter slots keyed by identity,
coupled weight decay, SGD momentum ``v = mu*v + g``, Adam debiased with eps
outside the sqrt, slot arithmetic in DOUBLE (the slots live in HBM as fp64)
and one f32 rounding of theta per step. ``step_all`` skips parameters
without a gradient and returns how many it updated. The difference is the
launch shape: every parameter of a step is updated by ONE kernel over a
tensor table (b2_sgd_multi / b2_adam_multi), not a Python loop per element.
"""

from __future__ import annotations

import ctypes

from . import _lib as L
from . import core as T
from .errors import ShapeError


class Optimizer:
    def __init__(self, lr: float, weight_decay: float = 0.0):
        self.lr = lr
        self.weight_decay = weight_decay
        self._state = {}

    _nslots = 1

    def state_for(self, param) -> dict:
        st = self._state.get(id(param))
        if st is None:
            slots = []
            for _ in range(self._nslots):
                b = T.Buffer(8 * max(param.size, 1))
                if param.size:
                    # zero the double slots (two f32 zeros == one double zero)
                    L.call("b2_fill_f32", b.ptr, 0.0, 2 * param.size, None)
                slots.append(b)
            st = {"param": param, "slots": slots, "t": 0}
            self._state[id(param)] = st
        return st

    def _entry(self, param, grad):
        if grad.shape != param.shape:
            raise ShapeError(f"gradient shape {grad.shape} does not match parameter {param.shape}")
        if not param.is_contiguous:
            raise ShapeError("optimizer parameters must be contiguous leaves")
        g = grad if grad.is_contiguous else T._copy_contig(grad)
        st = self.state_for(param)
        st["t"] += 1
        e = L.OptTensor()
        e.param = param.data_ptr
        e.grad = g.data_ptr
        e.slot0 = st["slots"][0].ptr
        e.slot1 = st["slots"][1].ptr if len(st["slots"]) > 1 else None
        e.n = param.size
        e.bc1, e.bc2 = self._bias_corrections(st["t"])
        return e, g

    def _bias_corrections(self, t):
        return 1.0, 1.0

    def _launch(self, table, count, stream=None):
        raise NotImplementedError

    def prepare(self, pairs):
        """Host-side half of a step: validate, make gradients contiguous and
        create slots (both enqueue work on the engine stream), bump the step
        counts and build the tensor table. Returns an opaque handle for
        `launch`."""
        pairs = list(pairs)
        entries, keep = [], []
        for p, g in pairs:
            e, gg = self._entry(p, g)
            entries.append(e)
            keep.append(gg)
        table = (L.OptTensor * len(entries))(*entries) if entries else None
        return pairs, table, keep

    def launch(self, handle, stream=None):
        """Device half: one multi-tensor kernel on `stream` (None: the engine
        stream), which must be ordered after everything `prepare` enqueued."""
        pairs, table, _ = handle
        if not pairs:
            return 0
        self._launch(table, len(pairs), stream)
        for p, _ in pairs:
            p.buffer.version += 1  # in-place write, like param.write_flat
        return len(pairs)

    def step_many(self, pairs):
        """Update every (param, grad) pair with one kernel launch."""
        return self.launch(self.prepare(pairs))

    def step(self, param, grad):
        self.step_many([(param, grad)])
        return param


class SGD(Optimizer):
    """v = mu*v + g + lambda*theta; theta -= lr*v (optim.py:54-72)."""

    def __init__(self, lr=0.01, momentum=0.0, weight_decay=0.0):
        super().__init__(lr, weight_decay)
        self.momentum = momentum

    def _launch(self, table, count, stream=None):
        L.call("b2_sgd_multi", table, count, float(self.lr), float(self.momentum),
               float(self.weight_decay), stream)


class Adam(Optimizer):
    """Debiased moments, eps outside the square root (optim.py:75-100)."""

    _nslots = 2

    def __init__(self, lr=0.001, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0):
        super().__init__(lr, weight_decay)
        self.beta1, self.beta2 = betas
        self.eps = eps

    def _bias_corrections(self, t):
        return 1.0 - self.beta1 ** t, 1.0 - self.beta2 ** t  # optim.py:90-91

    def _launch(self, table, count, stream=None):
        L.call("b2_adam_multi", table, count, float(self.lr), float(self.beta1),
               float(self.beta2), float(self.eps), float(self.weight_decay), stream)


class RMSprop(Optimizer):
    """v = rho*v + (1-rho)*g^2; theta -= lr*g/sqrt(v + eps) (optim.py:103-122)."""

    def __init__(self, lr=0.01, rho=0.99, eps=1e-8, weight_decay=0.0):
        super().__init__(lr, weight_decay)
        self.rho = rho
        self.eps = eps

    def _launch(self, table, count, stream=None):
        L.call("b2_rmsprop_multi", table, count, float(self.lr), float(self.rho), float(self.eps),
               float(self.weight_decay), stream)


def step_all(optimizer: Optimizer, parameters, grad_store):
    """Update every parameter that has a gradient entry; skip the rest
    (optim.py:125-136). Returns the number updated. One kernel launch."""
    pairs = []
    for p in parameters:
        g = grad_store.get(p)
        if g is not None:
            pairs.append((p, g))
    return optimizer.step_many(pairs)
