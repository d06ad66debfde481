"""Device tensors with strided views, broadcasting and recorded ops.

Drop-in for the reference engine module (tensorlite/core.py:1-820): same
function names, argument meanings, shapes, exception classes and messages;
the storage lives in B200 HBM and every op is one (or a few) sm_100a kernel
launches on the engine's CUDA stream through the C ABI (include/b2.h).

Storage and views (core.py:68-191): a ``Buffer`` owns one block from the
caching device allocator (freed in stream order when the last view dies)
and a mutation ``version``. A ``Tensor`` is (buffer, shape, strides,
offset); reshape of contiguous data, transpose2d and stride-0 broadcasts
are views, exactly as in the reference, and kernels read the views in
place (strided / broadcast operands, transposed GEMM operands).

Numerics: + - * / are IEEE fp32 (== the reference's
f32(double op)); exp/log are f32(double libm); sums accumulate in fp64;
max keeps the first maximum; matmul is fp32-accurate (3xBF16 on tcgen05
or FFMA) and lands within the 1e-4 tolerance of the reference's double
dot products.
"""

from __future__ import annotations

import ctypes
import math
import os
import random
import threading
import weakref

import numpy as np

from . import _lib as L
from . import autograd as _autograd
from .autograd import is_recording, no_grad, record
from .errors import BroadcastError, ShapeError

_py_sum = sum
_py_max = max


# ---------------------------------------------------------------------------
# storage


class Buffer:
    """One device allocation plus a version counter (core.py:68-75)."""

    __slots__ = ("ptr", "nbytes", "version", "_splits", "_pending", "__weakref__")

    def __init__(self, nbytes: int):
        L.ensure_device()
        p = ctypes.c_void_p()
        L.check(L.lib().b2_alloc(_py_max(int(nbytes), 4), None, ctypes.byref(p)))
        self.ptr = p.value
        self.nbytes = int(nbytes)
        self.version = 0
        self._splits = None  # {(kind, offset, rows, cols, ld): (version, hi, lo, capture)} GEMM operand splits
        # (hi, lo, n): the fp32 contents are not written yet -- a GEMM epilogue
        # wrote only the 3xBF16 split the next GEMMs read; the first fp32
        # access materialises f32(hi) + f32(lo) (see _materialize)
        self._pending = None

    def __del__(self):
        try:
            if self.ptr and L._lib is not None:
                L._lib.b2_free(self.ptr, None)
        except Exception:
            pass
        self.ptr = 0


class ExternalBuffer(Buffer):
    """Device memory owned by another framework (a DLPack import): never
    returned to the engine's allocator; the producer's deleter runs when the
    last engine view dies."""

    __slots__ = ("_owner",)

    def __init__(self, ptr: int, nbytes: int, owner=None):
        self.ptr = ptr
        self.nbytes = int(nbytes)
        self.version = 0
        self._splits = None
        self._pending = None
        self._owner = owner

    def __del__(self):
        try:
            if self._owner is not None:
                from . import dlpack

                dlpack.release(self._owner)
        except Exception:
            pass
        self._owner = None
        self.ptr = 0


def _contig_strides(shape):
    st = [0] * len(shape)
    acc = 1
    for d in range(len(shape) - 1, -1, -1):
        st[d] = acc
        acc *= shape[d]
    return tuple(st)


def _numel(shape):
    n = 1
    for s in shape:
        n *= s
    return n


def _check_shape(shape):
    if isinstance(shape, int):
        shape = (shape,)
    shape = tuple(shape)
    for s in shape:
        if not isinstance(s, (int, np.integer)) or s < 0:
            raise ShapeError(f"invalid shape {shape}")
    return tuple(int(s) for s in shape)


class Tensor:
    __slots__ = ("buffer", "shape", "strides", "offset", "requires_grad", "node", "__weakref__")

    def __init__(self, buffer, shape, strides=None, offset=0, requires_grad=False):
        self.buffer = buffer
        self.shape = tuple(shape)
        self.strides = _contig_strides(self.shape) if strides is None else tuple(strides)
        self.offset = offset
        self.requires_grad = requires_grad
        self.node = None

    @property
    def size(self) -> int:
        return _numel(self.shape)

    @property
    def ndim(self) -> int:
        return len(self.shape)

    @property
    def is_contiguous(self) -> bool:
        return self.strides == _contig_strides(self.shape)

    @property
    def data_ptr(self) -> int:
        """Address of the first element, with the fp32 contents valid (a
        buffer whose GEMM wrote only its operand split is materialised)."""
        b = self.buffer
        if b._pending is not None:
            _materialize(b)
        return b.ptr + 4 * self.offset

    @property
    def _addr(self) -> int:
        """Address only (alignment checks, split-operand GEMMs): no materialisation."""
        return self.buffer.ptr + 4 * self.offset

    def __repr__(self):
        vals = self.flat()
        head = ", ".join(f"{v:g}" for v in vals[:6])
        if self.size > 6:
            head += ", ..."
        grad = ", requires_grad=True" if self.requires_grad else ""
        return f"Tensor(shape={self.shape}, [{head}]{grad}, device=b200)"

    # -- reading values out (device -> host copies)

    def numpy(self) -> np.ndarray:
        """A host float32 copy in row-major logical order."""
        out = np.empty(self.shape, dtype=np.float32)
        if self.size == 0:
            return out
        src = self if (self.ndim == 0 or self.is_contiguous) else _copy_contig(self)
        L.call("b2_memcpy_d2h", out.ctypes.data, src.data_ptr, self.size * 4, None)
        return out

    def flat(self) -> list:
        return self.numpy().ravel().astype(np.float64).tolist()

    def item(self) -> float:
        if self.size != 1:
            raise ShapeError(f"item() needs a single-element tensor, got shape {self.shape}")
        v = np.empty(1, np.float32)
        L.call("b2_memcpy_d2h", v.ctypes.data, self.data_ptr, 4, None)
        return float(v[0])

    def tolist(self):
        if self.ndim == 0:
            return self.item()
        return self.numpy().astype(np.float64).tolist()

    # -- mutation (bumps the buffer version so stale pullbacks are caught)

    def fill_(self, value: float):
        if self.is_contiguous:
            L.call("b2_fill_f32", self.data_ptr, float(value), self.size, None)
            self.buffer.version += 1
            return self
        return self.write_flat([value] * self.size)

    def set_flat(self, index: int, value: float):
        if not 0 <= index < self.size:
            raise IndexError(f"flat index {index} out of range for shape {self.shape}")
        off = self.offset
        rem = index
        for d in range(self.ndim - 1, -1, -1):
            off += (rem % self.shape[d]) * self.strides[d]
            rem //= self.shape[d]
        v = np.array([value], np.float32)
        L.call("b2_memcpy_h2d", self.data_ptr - 4 * self.offset + 4 * off, v.ctypes.data, 4, None)
        self.buffer.version += 1
        return self

    def write_flat(self, values):
        arr = np.asarray(values if isinstance(values, np.ndarray) else list(values),
                         dtype=np.float32).ravel()
        if arr.size != self.size:
            raise ShapeError(f"expected {self.size} values, got {arr.size}")
        arr = np.ascontiguousarray(arr)
        if self.size:
            if self.is_contiguous:
                L.call("b2_memcpy_h2d", self.data_ptr, arr.ctypes.data, arr.nbytes, None)
                L.synchronize()  # arr is pageable and may be freed by the caller
            else:
                src = from_numpy(arr.reshape(self.shape))
                L.call("b2_write_strided", self.data_ptr, self.ndim, L.i64s(self.shape),
                       L.i64s(self.strides), src.data_ptr, None)
        self.buffer.version += 1
        return self

    def detach(self) -> "Tensor":
        return Tensor(self.buffer, self.shape, self.strides, self.offset)

    # -- DLPack (zero-copy device exchange, dlpack.py)
    def __dlpack__(self, stream=None):
        from . import dlpack

        return dlpack.to_capsule(self, stream)

    def __dlpack_device__(self):
        from . import dlpack

        return (dlpack.kDLCUDA, dlpack.device_id())

    def copy(self) -> "Tensor":
        return _copy_contig(self)


def _empty(shape) -> Tensor:
    shape = tuple(shape)
    return Tensor(Buffer(4 * _numel(shape)), shape)


def _copy_contig(t: Tensor) -> Tensor:
    out = _empty(t.shape)
    if t.size:
        L.call("b2_copy_strided", out.data_ptr, t.ndim, L.i64s(t.shape), t.data_ptr,
               L.i64s(t.strides), None)
    return out


# ---------------------------------------------------------------------------
# constructors (core.py:254-357)


def from_dlpack(obj, requires_grad=False) -> Tensor:
    """Wrap a CUDA float32 tensor from any DLPack producer (torch, CuPy, ...)
    without a copy; the engine's ops read and write its memory in place."""
    from . import dlpack

    t = dlpack.from_dlpack(obj)
    t.requires_grad = requires_grad
    return t


def from_numpy(arr, requires_grad=False) -> Tensor:
    """Upload a host array (any float dtype is rounded to f32 once)."""
    # np.require keeps 0-d arrays 0-d (ascontiguousarray would return shape (1,))
    a = np.require(np.asarray(arr, dtype=np.float32), requirements="C")
    t = _empty(a.shape)
    if a.size:
        L.call("b2_memcpy_h2d", t.data_ptr, a.ctypes.data, a.nbytes, None)
        L.synchronize()
    t.requires_grad = requires_grad
    return t


def _infer_nested(data):
    if isinstance(data, (int, float)) and not isinstance(data, bool) or isinstance(data, bool):
        return (), [float(data)]
    if not isinstance(data, (list, tuple)):
        raise TypeError(f"cannot build a tensor from {type(data).__name__}")
    if not data:
        return (0,), []
    parts = [_infer_nested(d) for d in data]
    child = parts[0][0]
    if any(s != child for s, _ in parts[1:]):
        raise ShapeError("ragged nested data")
    flat = []
    for _, f in parts:
        flat.extend(f)
    return (len(data),) + child, flat


def tensor(data, requires_grad=False) -> Tensor:
    """A tensor from a number or nested lists of numbers (core.py:254-259)."""
    shape, flat = _infer_nested(data)
    t = from_numpy(np.array(flat, dtype=np.float32).reshape(shape))
    t.requires_grad = requires_grad
    return t


def from_flat(values, shape, requires_grad=False) -> Tensor:
    shape = _check_shape(shape)
    arr = np.asarray(values if isinstance(values, np.ndarray) else list(values), dtype=np.float32)
    if arr.size != _numel(shape):
        raise ShapeError(f"{arr.size} values cannot fill shape {shape}")
    t = from_numpy(arr.reshape(shape))
    t.requires_grad = requires_grad
    return t


def from_buffer(obj, shape, requires_grad=False) -> Tensor:
    """Upload external float32 storage (core.py:290-312 validation rules).

    The reference aliases host memory; HBM cannot alias a host buffer, so
    this copies once (documented divergence)."""
    mv = memoryview(obj)
    if mv.format != "f":
        raise TypeError(f"expected float32 storage (format 'f'), got {mv.format!r}")
    if mv.readonly:
        raise ValueError("buffer must be writable")
    if not mv.c_contiguous:
        raise ValueError("buffer must be C-contiguous")
    shape = _check_shape(shape)
    arr = np.frombuffer(mv.cast("B"), dtype=np.float32)
    if arr.size != _numel(shape):
        raise ShapeError(f"{arr.size} buffered values cannot fill shape {shape}")
    return from_numpy(arr.reshape(shape), requires_grad=requires_grad)


def full(shape, value, requires_grad=False) -> Tensor:
    shape = _check_shape(shape)
    t = _empty(shape)
    if t.size:
        L.call("b2_fill_f32", t.data_ptr, float(value), t.size, None)
    t.requires_grad = requires_grad
    return t


def zeros(shape, requires_grad=False) -> Tensor:
    return full(shape, 0.0, requires_grad)


def ones(shape, requires_grad=False) -> Tensor:
    return full(shape, 1.0, requires_grad)


def zeros_like(t, requires_grad=False) -> Tensor:
    return zeros(t.shape, requires_grad=requires_grad)


def ones_like(t, requires_grad=False) -> Tensor:
    return ones(t.shape, requires_grad=requires_grad)


def uniform(shape, low=-1.0, high=1.0, rng=None, requires_grad=False) -> Tensor:
    """Same Python MT19937 stream as the reference (core.py:333-341), so a
    seeded Dense gets bit-identical initial weights."""
    if rng is None:
        rng = random.Random()
    elif isinstance(rng, int):
        rng = random.Random(rng)
    shape = _check_shape(shape)
    vals = [rng.uniform(low, high) for _ in range(_numel(shape))]
    return from_flat(vals, shape, requires_grad=requires_grad)


class _Scalar:
    """A Python number operand: f32-rounded like tensor(float(x))
    (core.py:352-357), passed to kernels by value instead of being uploaded."""

    __slots__ = ("value",)
    shape = ()
    requires_grad = False

    def __init__(self, v):
        self.value = float(np.float32(v))


def _as_operand(x):
    if isinstance(x, (Tensor, _Scalar)):
        return x
    if isinstance(x, (int, float)) and not isinstance(x, bool) or isinstance(x, (bool, np.floating)):
        return _Scalar(x)
    raise TypeError(f"expected a Tensor or number, got {type(x).__name__}")


def _as_tensor(x) -> Tensor:
    if isinstance(x, Tensor):
        return x
    if isinstance(x, _Scalar):
        return full((), x.value)
    if isinstance(x, (int, float)):
        return full((), float(x))
    raise TypeError(f"expected a Tensor or number, got {type(x).__name__}")


# ---------------------------------------------------------------------------
# broadcasting (core.py:364-423)


def broadcast_shapes(s1, s2):
    n1, n2 = len(s1), len(s2)
    n = _py_max(n1, n2)
    out = []
    for i in range(n):
        a = s1[n1 - n + i] if n1 - n + i >= 0 else 1
        b = s2[n2 - n + i] if n2 - n + i >= 0 else 1
        if a == b or b == 1:
            out.append(a)
        elif a == 1:
            out.append(b)
        else:
            raise BroadcastError(f"cannot broadcast {tuple(s1)} with {tuple(s2)}")
    return tuple(out)


def _expand_strides(t, shape):
    pad = len(shape) - t.ndim
    st = [0] * len(shape)
    for i in range(t.ndim):
        if t.shape[i] == shape[pad + i]:
            st[pad + i] = t.strides[i]
        elif t.shape[i] == 1:
            st[pad + i] = 0
        else:
            raise BroadcastError(f"cannot expand {t.shape} to {tuple(shape)}")
    return tuple(st)


def _expand_view(t: Tensor, shape) -> Tensor:
    return Tensor(t.buffer, shape, _expand_strides(t, shape), t.offset,
                  requires_grad=t.requires_grad)


def broadcast_to(x: Tensor, shape) -> Tensor:
    shape = _check_shape(shape)
    if len(shape) < x.ndim:
        raise BroadcastError(f"cannot broadcast {x.shape} to smaller rank {shape}")
    v = _expand_view(x, shape)
    out = Tensor(v.buffer, v.shape, v.strides, v.offset)
    return record("broadcast_to", (x,), out, (lambda g: reduce_to_shape(g, x.shape),))


def reduce_to_shape(t: Tensor, shape) -> Tensor:
    """Sum t down to `shape` (adjoint of broadcasting; core.py:405-423). A
    cotangent whose producing kernel already summed its columns (fp64, one f32
    rounding: the same values) returns those sums instead of re-reading t."""
    shape = _check_shape(shape)
    if t.shape == shape:
        return t
    cs = _COLSUM.get(t) if t.ndim == 2 else None
    if cs is not None and shape in ((t.shape[1],), (1, t.shape[1])):
        return reshape(cs, shape)
    pad = t.ndim - len(shape)
    if pad < 0:
        raise ShapeError(f"cannot reduce {t.shape} to larger rank {shape}")
    padded = (1,) * pad + shape
    axes = []
    for i, (have, want) in enumerate(zip(t.shape, padded)):
        if want == have:
            continue
        if want == 1:
            axes.append(i)
        else:
            raise ShapeError(f"{shape} is not a broadcast source of {t.shape}")
    out = sum(t, axis=tuple(axes), keepdims=True) if axes else t
    return reshape(out, shape)


# ---------------------------------------------------------------------------
# elementwise (core.py:430-546)


def _launch_binary(op, a, b, shape) -> Tensor:
    out = _empty(shape)
    if out.size == 0:
        return out
    nd = len(shape)
    if isinstance(a, _Scalar) or isinstance(b, _Scalar):
        if isinstance(a, _Scalar) and isinstance(b, _Scalar):
            a = full((), a.value)
        if isinstance(b, _Scalar):
            L.call("b2_binary_scalar", op, out.data_ptr, nd, L.i64s(shape), a.data_ptr,
                   L.i64s(_expand_strides(a, shape)), b.value, 0, None)
        else:
            L.call("b2_binary_scalar", op, out.data_ptr, nd, L.i64s(shape), b.data_ptr,
                   L.i64s(_expand_strides(b, shape)), a.value, 1, None)
        return out
    L.call("b2_binary", op, out.data_ptr, nd, L.i64s(shape), a.data_ptr,
           L.i64s(_expand_strides(a, shape)), b.data_ptr, L.i64s(_expand_strides(b, shape)), None)
    return out


def _binary(kind, op, a, b, pullbacks, save):
    a = _as_operand(a)
    b = _as_operand(b)
    shape = broadcast_shapes(a.shape, b.shape)
    out = _launch_binary(op, a, b, shape)
    pa, pb = pullbacks(a, b, out)
    saved = tuple(t for t in save(a, b) if isinstance(t, Tensor))
    return record(kind, (a, b), out, (pa, pb), saved=saved)


def add(a, b) -> Tensor:
    return _binary("add", L.ADD, a, b,
                   lambda a, b, out: (lambda g: reduce_to_shape(g, a.shape),
                                      lambda g: reduce_to_shape(g, b.shape)),
                   lambda a, b: ())


def sub(a, b) -> Tensor:
    return _binary("sub", L.SUB, a, b,
                   lambda a, b, out: (lambda g: reduce_to_shape(g, a.shape),
                                      lambda g: reduce_to_shape(neg(g), b.shape)),
                   lambda a, b: ())


def mul(a, b) -> Tensor:
    return _binary("mul", L.MUL, a, b,
                   lambda a, b, out: (lambda g: reduce_to_shape(mul(g, b), a.shape),
                                      lambda g: reduce_to_shape(mul(g, a), b.shape)),
                   lambda a, b: (a, b))


def div(a, b) -> Tensor:
    return _binary("div", L.DIV, a, b,
                   lambda a, b, out: (
                       lambda g: reduce_to_shape(div(g, b), a.shape),
                       # d(a/b)/db = -a/b^2, composed exactly like core.py:492
                       lambda g: reduce_to_shape(neg(div(mul(g, a), mul(b, b))), b.shape)),
                   lambda a, b: (a, b))


def _launch_unary(op, x, alpha=0.0, beta=0.0) -> Tensor:
    out = _empty(x.shape)
    if out.size:
        L.call("b2_unary", op, out.data_ptr, x.ndim, L.i64s(x.shape), x.data_ptr,
               L.i64s(x.strides), float(alpha), float(beta), None)
    return out


def _unary(kind, op, x, pullback, save):
    x = _as_tensor(_as_operand(x))
    out = _launch_unary(op, x)
    # pullbacks see a node-less alias of `out`: output -> node -> closure -> output
    # would be a reference cycle that keeps HBM alive until the cyclic GC runs
    keep = out.detach()
    return record(kind, (x,), out, (pullback(x, keep),), saved=save(x, keep))


def neg(x) -> Tensor:
    return _unary("neg", L.NEG, x, lambda x, out: lambda g: neg(g), lambda x, out: ())


def exp(x) -> Tensor:
    return _unary("exp", L.EXP, x, lambda x, out: lambda g: mul(g, out), lambda x, out: (out,))


def log(x) -> Tensor:
    return _unary("log", L.LOG, x, lambda x, out: lambda g: div(g, x), lambda x, out: (x,))


def sqrt(x) -> Tensor:
    return _unary("sqrt", L.SQRT, x, lambda x, out: lambda g: div(g, mul(out, 2.0)),
                  lambda x, out: (out,))


def _sign_mul(g, x):
    shape = broadcast_shapes(g.shape, x.shape)
    return _launch_binary(L.SIGN_MUL, g, x, shape)


def absolute(x) -> Tensor:
    return _unary("abs", L.ABS, x, lambda x, out: lambda g: _sign_mul(g, x), lambda x, out: (x,))


abs_ = absolute


def relu(x) -> Tensor:
    """nn.relu (nn.py:108-111): v if v > 0 else 0.0; grad mask v > 0."""
    x = _as_tensor(_as_operand(x))
    out = _launch_unary(L.RELU, x)

    def pull(g):
        return _launch_binary(L.RELU_BWD, g, x, broadcast_shapes(g.shape, x.shape))

    return record("relu", (x,), out, (pull,), saved=(x,))


def _activation(kind, op, bwd_op, x, from_input):
    """nn._pointwise (nn.py:95-105): out = f32(fn(x)); pullback g * f32(dfn(v))
    with v the saved input (from_input) or output -- one kernel each way."""
    x = _as_tensor(_as_operand(x))
    out = _launch_unary(op, x)
    v = x if from_input else out.detach()

    def pull(g):
        return _launch_binary(bwd_op, g, v, broadcast_shapes(g.shape, v.shape))

    return record(kind, (x,), out, (pull,), saved=(v,))


def sigmoid(x) -> Tensor:
    """nn.sigmoid (nn.py:114-124): sign-split logistic; grad y * (1 - y)."""
    return _activation("sigmoid", L.SIGMOID, L.SIGMOID_BWD, x, False)


def tanh(x) -> Tensor:
    """nn.tanh (nn.py:127-129): math.tanh; grad 1 - y * y."""
    return _activation("tanh", L.TANH, L.TANH_BWD, x, False)


def gelu(x) -> Tensor:
    """nn.gelu (nn.py:132-144): 0.5 x (1 + erf(x / sqrt 2)); grad Phi(x) + x phi(x)."""
    return _activation("gelu", L.GELU, L.GELU_BWD, x, True)


def clamp(x, low, high) -> Tensor:
    """min(max(x, low), high). Not a reference op (the BASELINE config-2 clamp
    happens on the host there); gradient passes where low<=x<=high."""
    x = _as_tensor(_as_operand(x))
    out = _launch_unary(L.CLAMP, x, low, high)

    def pull(g):
        inside = _launch_unary(L.CLAMP_MASK, x, low, high)
        return _launch_binary(L.RELU_BWD, g, inside, broadcast_shapes(g.shape, x.shape))

    return record("clamp", (x,), out, (pull,), saved=(x,))


# ---------------------------------------------------------------------------
# reductions (core.py:556-728)


def _normalize_axes(axis, ndim):
    if axis is None:
        return tuple(range(ndim))
    if isinstance(axis, (int, np.integer)):
        axis = (int(axis),)
    axes = []
    for a in axis:
        if not isinstance(a, (int, np.integer)):
            raise ShapeError(f"axis must be an int, got {a!r}")
        a = int(a)
        if a < 0:
            a += ndim
        if not 0 <= a < ndim:
            raise ShapeError(f"axis {a} out of range for {ndim}-d tensor")
        axes.append(a)
    if len(set(axes)) != len(axes):
        raise ShapeError(f"duplicate axes in {axis}")
    return tuple(sorted(axes))


def _reduced_shapes(shape, axes, keepdims):
    kshape = tuple(1 if i in axes else s for i, s in enumerate(shape))
    oshape = kshape if keepdims else tuple(s for i, s in enumerate(shape) if i not in axes)
    return kshape, oshape


def _mask(axes):
    m = 0
    for a in axes:
        m |= 1 << a
    return m


def _reduce(op, x, axes, oshape, want_arg=False):
    out = _empty(oshape)
    arg = None
    if want_arg:
        arg = Buffer(8 * _py_max(out.size, 1))
    if x.ndim == 0:
        L.call("b2_copy_strided", out.data_ptr, 0, L.i64s(()), x.data_ptr, L.i64s(()), None)
        if arg is not None:
            L.call("b2_fill_f32", arg.ptr, 0.0, 2, None)  # int64 zero
        return out, arg
    L.call("b2_reduce", op, out.data_ptr, arg.ptr if arg else None, x.ndim, L.i64s(x.shape),
           x.data_ptr, L.i64s(x.strides), _mask(axes), None)
    return out, arg


def _sum_pullback(x, axes, kshape):
    # the cotangent of a sum is g broadcast over the reduced axes: returned as
    # a stride-0 view (no HBM write); consumers read it through their strides
    def pull(g):
        return _expand_view(reshape(g, kshape), x.shape)

    return pull


def sum(x, axis=None, keepdims=False) -> Tensor:
    x = _as_tensor(_as_operand(x))
    axes = _normalize_axes(axis, x.ndim)
    kshape, oshape = _reduced_shapes(x.shape, axes, keepdims)
    out, _ = _reduce(L.RED_SUM, x, axes, oshape)
    return record("sum", (x,), out, (_sum_pullback(x, axes, kshape),))


def mean(x, axis=None, keepdims=False) -> Tensor:
    x = _as_tensor(_as_operand(x))
    axes = _normalize_axes(axis, x.ndim)
    kshape, oshape = _reduced_shapes(x.shape, axes, keepdims)
    count = 1
    for a in axes:
        count *= x.shape[a]
    if len(axes) == x.ndim and x.ndim > 0:
        oshape = kshape if keepdims else ()
    out, _ = _reduce(L.RED_MEAN, x, axes, oshape)
    fcount = _Scalar(float(count))

    def pull(g):
        # div(expand(g), float(count)): every element of a broadcast row is the
        # same f32(g / count), so divide the kept-shape cotangent once and
        # return it as a stride-0 view (bit-identical, no full-size write)
        gk = reshape(g, kshape)
        q = _empty(kshape)
        if q.size:
            L.call("b2_binary_scalar", L.DIV, q.data_ptr, len(kshape), L.i64s(kshape), gk.data_ptr,
                   L.i64s(gk.strides), fcount.value, 0, None)
        return _expand_view(q, x.shape)

    return record("mean", (x,), out, (pull,))


def max(x, axis=None, keepdims=False) -> Tensor:
    """Maximum over axes; ties resolve to the first element in row-major
    order, which is also where the gradient goes (core.py:692-728)."""
    x = _as_tensor(_as_operand(x))
    axes = _normalize_axes(axis, x.ndim)
    kshape, oshape = _reduced_shapes(x.shape, axes, keepdims)
    for a in axes:
        if x.shape[a] == 0:
            raise ShapeError("max over a zero-extent axis is undefined")
    # the first-max index is only the gradient's routing (core.py:721-726):
    # without a node to record, the value-only scan runs (no index tracking)
    out, arg = _reduce(L.RED_MAX, x, axes, oshape, want_arg=is_recording() and x.requires_grad)
    if arg is None:
        return out
    in_shape = x.shape
    mask = _mask(axes)

    def pull(g):
        gc = g if g.is_contiguous else _copy_contig(g)
        gx = _empty(in_shape)
        if gx.size:
            L.call("b2_max_scatter", gx.data_ptr, len(in_shape), L.i64s(in_shape), mask,
                   gc.data_ptr, arg.ptr, None)
        return gx

    return record("max", (x,), out, (pull,), saved=(x,))


def argmax(x, axis=-1) -> np.ndarray:
    """First-maximum indices along one axis (the max reduction's routing
    index, core.py:709-713 scan order), read back to the host as int64 -- for
    callers' metrics such as the demos' accuracy (demos.py:85-96)."""
    x = _as_tensor(_as_operand(x))
    axes = _normalize_axes(axis, x.ndim)
    if len(axes) != 1:
        raise ShapeError("argmax takes exactly one axis")
    if x.shape[axes[0]] == 0:
        raise ShapeError("max over a zero-extent axis is undefined")
    _, oshape = _reduced_shapes(x.shape, axes, False)
    out, arg = _reduce(L.RED_MAX, x, axes, oshape, want_arg=True)
    idx = np.empty(_py_max(out.size, 1), np.int64)
    L.call("b2_memcpy_d2h", idx.ctypes.data, arg.ptr, 8 * idx.size, None)
    return idx[:out.size].reshape(oshape)


# ---------------------------------------------------------------------------
# shape ops (core.py:735-761)


def reshape(x, shape) -> Tensor:
    x = _as_tensor(_as_operand(x))
    shape = list(shape) if not isinstance(shape, int) else [shape]
    if shape.count(-1) > 1:
        raise ShapeError("at most one -1 allowed in reshape")
    if -1 in shape:
        rest = _numel([s for s in shape if s != -1])
        if rest == 0 or x.size % rest:
            raise ShapeError(f"cannot infer -1 reshaping {x.shape} to {tuple(shape)}")
        shape[shape.index(-1)] = x.size // rest
    shape = _check_shape(shape)
    if _numel(shape) != x.size:
        raise ShapeError(f"cannot reshape {x.shape} ({x.size} elements) to {shape}")
    if x.ndim == 0 or x.is_contiguous:
        out = Tensor(x.buffer, shape, offset=x.offset)
    else:
        c = _copy_contig(x)
        out = Tensor(c.buffer, shape)
    old = x.shape
    return record("reshape", (x,), out, (lambda g: reshape(g, old),))


def transpose2d(x) -> Tensor:
    x = _as_tensor(_as_operand(x))
    if x.ndim != 2:
        raise ShapeError(f"transpose2d needs a 2-d tensor, got shape {x.shape}")
    out = Tensor(x.buffer, (x.shape[1], x.shape[0]), (x.strides[1], x.strides[0]), x.offset)
    return record("transpose2d", (x,), out, (lambda g: transpose2d(g),))


# ---------------------------------------------------------------------------
# matrix product (core.py:768-820)


def _as_A(t):
    """Operand with logical shape (M, K) -> (trans, ld, tensor)."""
    M, K = t.shape
    s0, s1 = t.strides
    if (s1 == 1 or K <= 1) and (M <= 1 or s0 >= K):
        return 0, (s0 if M > 1 else K), t
    if (s0 == 1 or M <= 1) and (K <= 1 or s1 >= M):
        return 1, (s1 if K > 1 else M), t
    c = _copy_contig(t)
    return 0, K, c


def _as_B(t):
    """Operand with logical shape (N, K) (the reference's w) -> (trans_b, ld, tensor).
    trans_b=1: stored [N, K] row-major; trans_b=0: stored [K, N]."""
    N, K = t.shape
    s0, s1 = t.strides
    if (s1 == 1 or K <= 1) and (N <= 1 or s0 >= K):
        return 1, (s0 if N > 1 else K), t
    if (s0 == 1 or N <= 1) and (K <= 1 or s1 >= N):
        return 0, (s1 if K > 1 else N), t
    c = _copy_contig(t)
    return 1, K, c


_PENDING = weakref.WeakSet()  # buffers whose fp32 contents are still only a split
_LAZY_FP32 = os.environ.get("B2_LAZY_FP32", "1") != "0"  # 0: every GEMM stores its fp32 C


def _set_pending(buf, hi, lo, n):
    """Mark buf's fp32 contents as not yet written: only its 3xBF16 split
    (hi, lo) is. Inside a CUDA-graph capture the capture remembers it, so
    every replay (which rewrites hi/lo) marks the buffer pending again."""
    from .graph import _capturing, _captured_pending

    buf._pending = (hi, lo, n)
    _PENDING.add(buf)
    if _capturing[0]:
        _captured_pending.append((weakref.ref(buf), hi, lo, n))


def _materialize(buf):
    """Write a pending buffer's fp32 contents from its 3xBF16 split (exact
    f32(hi) + f32(lo): within 2^-16 relative of the GEMM's fp32 result -- hi
    keeps 8 significant bits, lo the next 8 of the residual -- and exactly the
    operand the following GEMMs consumed)."""
    hi, lo, n = buf._pending
    buf._pending = None
    _PENDING.discard(buf)
    L.call("b2_bf16x3_join", buf.ptr, hi.ptr, lo.ptr, n, None)


def materialize_pending():
    """Materialise every pending buffer (before a CUDA-graph capture: a
    materialisation recorded inside a capture would only run at replay)."""
    for b in list(_PENDING):
        if b._pending is not None:
            _materialize(b)


def _split_pair(xa, ashape, wb, bshape, kind):
    """_split of a GEMM's two operands; when both are fresh 3xBF16 splits of
    different regions, one launch makes both (b2_bf16x3_split2)."""
    if kind == "3xbf16":
        from .graph import _capturing

        cap = _capturing[0]
        ka = ("3xbf16", xa.offset) + tuple(ashape)
        kb = ("3xbf16", wb.offset) + tuple(bshape)

        def fresh(t, key):
            ent = (t.buffer._splits or {}).get(key)
            return not (ent is not None and ent[0] == t.buffer.version and (not cap or ent[3] == cap))

        if fresh(xa, ka) and fresh(wb, kb) and not (xa.buffer is wb.buffer and ka == kb):
            (ra, ca, lda), (rb, cb, ldb) = ashape, bshape
            ahi, alo = Buffer(2 * ra * ca), Buffer(2 * ra * ca)
            bhi, blo = Buffer(2 * rb * cb), Buffer(2 * rb * cb)
            L.call("b2_bf16x3_split2", ahi.ptr, alo.ptr, xa.data_ptr, ra, ca, lda, bhi.ptr, blo.ptr,
                   wb.data_ptr, rb, cb, ldb, None)
            for t, key, hi, lo in ((xa, ka, ahi, alo), (wb, kb, bhi, blo)):
                if t.buffer._splits is None:
                    t.buffer._splits = {}
                t.buffer._splits[key] = (t.buffer.version, hi, lo, cap)
            return ahi, alo, bhi, blo
    ahi, alo = _split(xa, *ashape, kind)
    bhi, blo = _split(wb, *bshape, kind)
    return ahi, alo, bhi, blo


def _split(t, rows, cols, ld, kind):
    """Cached split of the stored matrix region of t for a tensor-core GEMM:
    kind "tf32x" -> (bf16 hi, bf16 lo) of trunc_tf32(x) / x - trunc (2 B each),
    kind "3xbf16" -> (bf16 hi, bf16 lo) of bf16_rn(x) / bf16_rn(x - hi),
    kind "3xtf32" -> (fp32 hi, fp32 lo), kind "bf16" -> (bf16 cast, None).
    Invalidated by the buffer version."""
    from .graph import _capturing

    buf = t.buffer
    key = (kind, t.offset, rows, cols, ld)
    if buf._splits is None:
        buf._splits = {}
    ent = buf._splits.get(key)
    cap = _capturing[0]
    # inside a CUDA-graph capture only splits made by this capture are trusted
    if ent is not None and ent[0] == buf.version and (not cap or ent[3] == cap):
        return ent[1], ent[2]
    n = rows * cols
    if kind == "bf16":  # bf16 variant: one RN cast, no low part
        hi, lo = Buffer(2 * n), None
        L.call("b2_bf16_cast", hi.ptr, t.data_ptr, rows, cols, ld, None)
        buf._splits[key] = (buf.version, hi, lo, cap)
        return hi, lo
    esz = 4 if kind == "3xtf32" else 2
    hi, lo = Buffer(esz * n), Buffer(esz * n)
    fn = {"tf32x": "b2_bf16x2_split", "3xbf16": "b2_bf16x3_split", "3xtf32": "b2_tf32_split"}[kind]
    L.call(fn, hi.ptr, lo.ptr, t.data_ptr, rows, cols, ld, None)
    buf._splits[key] = (buf.version, hi, lo, cap)
    return hi, lo


_ALGO_OVERRIDE = None
GEMM_TIMER = None  # bench/profiling: a list receiving (flops, start_event, end_event) per GEMM kernel


def set_gemm_algo(name):
    """Force 'simt' | '3xtf32' | '1xtf32' | 'tf32x' | '3xbf16' | 'bf16' | 'ref' |
    None (auto) for subsequent matmuls. 'bf16' is the reduced-precision variant
    (bf16 operands, fp32 accumulation, fp32 master values everywhere else) and
    is only ever used when asked for. 'ref' is the reference's own arithmetic
    (exact fp32 products summed in fp64, one f32 rounding: core.py:802-807) on
    the FP64 pipe -- the parity mode, not a performance path. 'ref_bf16' is the
    same arithmetic on bf16-rounded operands: the exact-arithmetic control of
    the bf16 variant."""
    global _ALGO_OVERRIDE
    _ALGO_OVERRIDE = {None: None, "auto": None, "simt": L.GEMM_SIMT, "3xtf32": L.GEMM_3XTF32,
                      "1xtf32": L.GEMM_1XTF32, "tf32x": L.GEMM_TF32X, "3xbf16": L.GEMM_3XBF16,
                      "bf16": L.GEMM_BF16, "ref": L.GEMM_REF, "ref_bf16": L.GEMM_REF_BF16}[name]


def get_gemm_algo():
    return _ALGO_OVERRIDE


def _gemm_into(out, x, w, bias=None, epi=L.EPI_NONE, mask=None, emit_split=False, colsum=None,
               mask_bits=None, bits_out=None):
    """out[M,N] = x[M,K] . w[N,K]^T (+bias)(relu); x, w arbitrary 2-D views.

    mask (contiguous [M,N]): multiply out by (mask > 0), the ReLU pullback --
    fused into the tensor-core epilogue, else applied by a separate pass.
    emit_split: let the tensor-core epilogue also write out's operand split into
    out's split cache (the next GEMMs reading out skip the split pass).
    colsum ([N] tensor): receives the column sums of the final out (after the
    mask), f32(fp64 sum) -- fused into the tensor-core epilogue, else a
    separate reduction.
    mask_bits (Buffer): the same ReLU pullback from the bits a forward ReLU
    GEMM wrote (only passed together with mask, the fallback); bits_out
    (Buffer, [M][ceil(N/64)] words): record out > 0 as bits. Returns whether
    bits_out was written (tensor-core path only)."""
    M, K = x.shape
    N = w.shape[0]
    ta, lda, xa = _as_A(x)
    tb, ldb, wb = _as_B(w)
    algo = _ALGO_OVERRIDE
    if algo is None:
        sel = ctypes.c_int()
        L.check(L.lib().b2_gemm_select(ta, tb, M, N, K, lda, ldb, ctypes.byref(sel)))
        algo = sel.value
    bptr = bias.data_ptr if bias is not None else None
    tc_ok = (K > 0 and (M if ta else K) % 8 == 0 and (K if tb else N) % 8 == 0
             and lda % 4 == 0 and ldb % 4 == 0 and xa._addr % 16 == 0 and wb._addr % 16 == 0)
    ar, ac = (K, M) if ta else (M, K)
    br, bc = (N, K) if tb else (K, N)
    mask_done = False
    cs_ptr = colsum.data_ptr if colsum is not None else None
    cs_done = False
    fused = {L.GEMM_TF32X: ("tf32x", L.GEMM_TF32X), L.GEMM_3XBF16: ("3xbf16", L.GEMM_3XBF16),
             L.GEMM_BF16: ("bf16", L.GEMM_BF16)}.get(algo) if tc_ok else None
    if fused is not None:
        kind, dalgo = fused
        ahi, alo, bhi, blo = _split_pair(xa, (ar, ac, lda), wb, (br, bc, ldb), kind)
        d = L.GemmDesc()
        d.algo, d.trans_a, d.trans_b, d.M, d.N, d.K = dalgo, ta, tb, M, N, K
        if kind == "tf32x":
            d.a[0], d.a[1], d.a[2] = xa.data_ptr, ahi.ptr, alo.ptr
            d.b[0], d.b[1], d.b[2] = wb.data_ptr, bhi.ptr, blo.ptr
        else:
            d.a[0], d.a[1] = ahi.ptr, (alo.ptr if alo is not None else None)
            d.b[0], d.b[1] = bhi.ptr, (blo.ptr if blo is not None else None)
        # a 3xBF16 output whose consumers read only its split (and bits /
        # column sums) skips the fp32 store; it is materialised on first use
        from .graph import _capturing

        lazy = (_LAZY_FP32 and emit_split and kind == "3xbf16"
                and out.offset == 0 and out.buffer.nbytes == 4 * M * N and (M * N) % 8 == 0
                and N % 8 == 0 and out.is_contiguous and out.buffer._pending is None)
        d.lda, d.ldb, d.C, d.ldc, d.bias, d.epilogue = lda, ldb, (None if lazy else out.data_ptr), N, bptr, epi
        if mask_bits is not None:
            d.mask_bits, mask_done = mask_bits.ptr, True
        elif mask is not None and mask.is_contiguous and mask.shape == out.shape \
                and mask.data_ptr % 16 == 0:
            d.mask, mask_done = mask.data_ptr, True
        shi = slo = None
        if emit_split and N % 8 == 0 and out.is_contiguous:
            shi = Buffer(2 * M * N)
            slo = Buffer(2 * M * N) if kind != "bf16" else None
            d.c_hi, d.c_lo = shi.ptr, (slo.ptr if slo is not None else None)
        if bits_out is not None:
            d.relu_bits_out = bits_out.ptr
        cs_done = cs_ptr is not None and (mask is None or mask_done)
        if cs_done:
            d.colsum = cs_ptr

        def after():
            if shi is not None:
                from .graph import _capturing

                buf = out.buffer
                if buf._splits is None:
                    buf._splits = {}
                buf._splits[(kind, out.offset, M, N, N)] = (buf.version, shi, slo, _capturing[0])
                if lazy:
                    _set_pending(buf, shi, slo, M * N)
            _gemm_fallbacks(out, mask, mask_done, cs_ptr, cs_done)

        grp = _GROUP.pending
        if grp is not None:  # launched with the other GEMMs of this pullback (gemm_group)
            # the descriptor holds raw pointers: keep their owners alive until the launch
            keep = (xa, wb, ahi, alo, bhi, blo, out, bias, mask, mask_bits, bits_out, colsum)
            grp.append((d, after, 2.0 * M * N * K, keep, (M, N, K, ta, tb)))
            return bits_out is not None
        ev = _timer_start()
        L.call("b2_gemm_fused", ctypes.byref(d), None)
        _timer_end(ev, 2.0 * M * N * K, ((M, N, K, ta, tb),))
        after()
        return bits_out is not None
    elif algo == L.GEMM_3XTF32 and tc_ok:
        ahi, alo = _split(xa, ar, ac, lda, "3xtf32")
        bhi, blo = _split(wb, br, bc, ldb, "3xtf32")
        ev = _timer_start()
        L.call("b2_gemm_presplit", ta, tb, M, N, K, ahi.ptr, alo.ptr, bhi.ptr, blo.ptr,
               out.data_ptr, N, bptr, epi, None)
    else:
        if algo in (L.GEMM_3XTF32, L.GEMM_TF32X, L.GEMM_3XBF16, L.GEMM_BF16):
            algo = L.GEMM_SIMT
        ev = _timer_start()
        L.call("b2_gemm", ta, tb, M, N, K, xa.data_ptr, lda, wb.data_ptr, ldb, out.data_ptr, N,
               bptr, epi, algo, None)
    _timer_end(ev, 2.0 * M * N * K, ((M, N, K, ta, tb),))
    _gemm_fallbacks(out, mask, mask_done, cs_ptr, cs_done)
    return False


def _gemm_fallbacks(out, mask, mask_done, cs_ptr, cs_done):
    """The epilogue stages a GEMM could not fuse, as separate kernels."""
    if mask is not None and not mask_done:
        L.call("b2_binary", L.RELU_BWD, out.data_ptr, 2, L.i64s(out.shape), out.data_ptr,
               L.i64s(out.strides), mask.data_ptr, L.i64s(mask.strides), None)
    if cs_ptr is not None and not cs_done:
        L.call("b2_reduce", L.RED_SUM, cs_ptr, None, 2, L.i64s(out.shape), out.data_ptr,
               L.i64s(out.strides), 1, None)


class _GroupState(threading.local):
    pending = None


_GROUP = _GroupState()
_GROUP_ON = os.environ.get("B2_GEMM_GROUP", "1") != "0"  # 0: one launch per GEMM (A/B)


class gemm_group:
    """Defer the fused tensor-core GEMMs issued inside the block and launch
    them together (b2_gemm_fused_group, up to 3 per launch) when it exits --
    for the pullbacks of one node (x_bar and w_bar of a matmul/linear read the
    same cotangent and write independent outputs). Nothing inside the block
    may read a deferred GEMM's output. Values are bit-identical to separate
    launches. Nested blocks join the outermost one."""

    __slots__ = ("items",)

    def __enter__(self):
        if _GROUP.pending is not None or not _GROUP_ON:
            self.items = None
        else:
            self.items = _GROUP.pending = []
        return self

    def __exit__(self, et, ev_, tb):
        items = self.items
        if items is None:
            return False
        _GROUP.pending = None
        if et is not None:
            return False
        for i in range(0, len(items), 3):
            part = items[i:i + 3]
            ev = _timer_start()
            if len(part) == 1:
                L.call("b2_gemm_fused", ctypes.byref(part[0][0]), None)
            else:
                arr = (L.GemmDesc * len(part))(*[it[0] for it in part])
                L.call("b2_gemm_fused_group", arr, len(part), None)
            _timer_end(ev, _py_sum(it[2] for it in part), tuple(it[4] for it in part))
            for it in part:
                it[1]()
        return False


_autograd.PULL_GROUP = gemm_group


def _timer_start():
    if GEMM_TIMER is None:
        return None
    ev = L.Event()
    ev.record()
    return ev


GEMM_TIMER_LABELS = None  # profiling: receives the (M, N, K, ta, tb) problems of each timed launch


def _timer_end(ev, flops, probs=()):
    if ev is not None:
        end = L.Event()
        end.record()
        GEMM_TIMER.append((flops, ev, end))
        if GEMM_TIMER_LABELS is not None:
            GEMM_TIMER_LABELS.append(probs)


def matmul(x, w) -> Tensor:
    """y = x @ w^T: (m, k) with (d, k) gives (m, d) (core.py:784-820)."""
    x = _as_tensor(_as_operand(x))
    w = _as_tensor(_as_operand(w))
    if x.ndim != 2 or w.ndim != 2:
        raise ShapeError(f"matmul needs 2-d tensors, got {x.shape} and {w.shape}")
    m, k = x.shape
    d, k2 = w.shape
    if k != k2:
        raise ShapeError(f"inner dimensions differ: {x.shape} vs {w.shape}")
    out = _empty((m, d))
    if out.size:
        _gemm_into(out, x, w)
    return record("matmul", (x, w), out,
                  (lambda g: matmul(g, transpose2d(w)),               # x_bar = g w
                   lambda g: matmul(transpose2d(g), transpose2d(x))),  # w_bar = g^T x
                  saved=(x, w), group=True)


def mm(a, b) -> Tensor:
    """PyTorch-convention product a @ b for a (..., k) and b (k, n): the
    reference's matmul(a, transpose2d(b)) with leading dims flattened
    (rank-3 matmul via reshape)."""
    a = _as_tensor(_as_operand(a))
    b = _as_tensor(_as_operand(b))
    if b.ndim != 2 or a.ndim < 2:
        raise ShapeError(f"mm needs (..., k) @ (k, n), got {a.shape} and {b.shape}")
    lead = a.shape[:-1]
    a2 = reshape(a, (-1, a.shape[-1])) if a.ndim > 2 else a
    y = matmul(a2, transpose2d(b))
    return reshape(y, lead + (b.shape[1],)) if a.ndim > 2 else y


_RELU_OUTPUTS = weakref.WeakKeyDictionary()  # outputs of relu-fused linear layers -> has a bias
_PREMASKED = weakref.WeakSet()     # cotangents whose ReLU mask is already applied
_COLSUM = weakref.WeakKeyDictionary()  # premasked cotangent -> its column sums (fused)
_RELU_BITS = weakref.WeakKeyDictionary()  # relu-fused output -> (buffer version, y > 0 bits)
_RELU_BITS_ON = os.environ.get("B2_RELU_BITS", "1") != "0"  # 0: read the fp32 outputs instead


def linear(x, weight, bias=None, relu_out=False) -> Tensor:
    """Fused Dense forward: relu?(x @ W^T + b) in ONE tcgen05 GEMM whose
    epilogue adds the bias and applies the ReLU. Values are bit-identical to
    the reference's add(matmul(x, W), b) then relu (nn.py:78-82, 108-111):
    f32(f32(acc) + b) then v > 0 ? v : 0. One tape node; its pullback applies
    the ReLU mask once and feeds the NN (x_bar), TN (W_bar) GEMMs and the
    bias column sum, exactly the cotangents of the composed ops."""
    x = _as_tensor(_as_operand(x))
    if x.ndim != 2 or weight.ndim != 2:
        raise ShapeError(f"matmul needs 2-d tensors, got {x.shape} and {weight.shape}")
    m, k = x.shape
    d, k2 = weight.shape
    if k != k2:
        raise ShapeError(f"inner dimensions differ: {x.shape} vs {weight.shape}")
    if bias is not None and bias.shape != (d,):
        raise BroadcastError(f"cannot broadcast {(m, d)} with {bias.shape}")
    out = _empty((m, d))
    if out.size:
        epi = (L.EPI_BIAS_RELU if relu_out else L.EPI_BIAS) if bias is not None else \
            (L.EPI_RELU if relu_out else L.EPI_NONE)
        bc = bias if (bias is None or bias.is_contiguous) else _copy_contig(bias)
        # a hidden layer's output is the next layer's GEMM operand: let the
        # epilogue write its operand split too (no separate split pass)
        bits = Buffer(8 * m * ((d + 63) // 64)) if relu_out and _RELU_BITS_ON else None
        if _gemm_into(out, x, weight, bc, epi, emit_split=relu_out, bits_out=bits):
            _RELU_BITS[out] = (out.buffer.version, bits)
    memo = [None, None]
    y = out.detach()  # no output->node->closure->output cycle (see _unary)
    if relu_out:
        _RELU_OUTPUTS[out] = bias is not None
    x_is_relu = x in _RELU_OUTPUTS
    x_has_bias = x_is_relu and _RELU_OUTPUTS.get(x, False)

    def pre(g):  # cotangent at the pre-activation (relu pullback, nn.py:101-103)
        if not relu_out or g in _PREMASKED:  # the layer above already applied this mask
            return g
        if memo[0] is not g:
            memo[0] = g
            memo[1] = _launch_binary(L.RELU_BWD, g, y, y.shape)
        return memo[1]

    def x_bar(g):
        # matmul(g, W) (core.py:816). When x is the ReLU output of the layer
        # below, that layer's pullback starts with g * (x > 0): apply it in this
        # GEMM's epilogue and emit the split its own dX/dW GEMMs read.
        gp = pre(g)
        if not x_is_relu:
            return matmul(gp, transpose2d(weight))
        xm = x.detach()
        res = _empty(x.shape)
        cs = _empty((x.shape[1],)) if x_has_bias else None
        if res.size:
            vb = _RELU_BITS.get(x)
            bits = vb[1] if vb is not None and vb[0] == x.buffer.version else None
            _gemm_into(res, gp, transpose2d(weight), mask=xm, emit_split=True, colsum=cs,
                       mask_bits=bits)
        _PREMASKED.add(res)
        if cs is not None and res.size:
            _COLSUM[res] = cs  # the layer below's bias gradient, summed in this epilogue
        return res

    pulls = [x_bar,
             lambda g: matmul(transpose2d(pre(g)), transpose2d(x))]
    inputs = [x, weight]
    if bias is not None:
        inputs.append(bias)

        def b_bar(g):  # add pullback (core.py:457-458): sum of the cotangent over the batch
            cs = _COLSUM.get(g) if relu_out and g in _PREMASKED else None
            return cs if cs is not None else reduce_to_shape(pre(g), bias.shape)

        pulls.append(b_bar)
    return record("linear_relu" if relu_out else "linear", tuple(inputs), out, tuple(pulls),
                  saved=(x, weight, y) if relu_out else (x, weight), group=True)


# ---------------------------------------------------------------------------
# fused / row-wise ops


def softmax(x, axis=-1) -> Tensor:
    """Row softmax over the last axis, bit-identical to the reference
    composition with the max detached; one kernel each way."""
    x = _as_tensor(_as_operand(x))
    if x.ndim == 0:
        raise ShapeError("softmax needs at least one axis")
    ax = _normalize_axes(axis, x.ndim)
    if ax != (x.ndim - 1,):
        raise ShapeError("softmax is implemented over the last axis")
    xc = x if x.is_contiguous else _copy_contig(x)
    C = x.shape[-1]
    R = x.size // C if C else 0
    y = _empty(x.shape)
    rs, rm = Buffer(4 * _py_max(R, 1)), Buffer(4 * _py_max(R, 1))
    if y.size:
        L.call("b2_softmax_fwd", y.data_ptr, rs.ptr, rm.ptr, xc.data_ptr, R, C, None)

    def pull(g):
        gc = g if g.is_contiguous else _copy_contig(g)
        gz = _empty(x.shape)
        if gz.size:
            L.call("b2_softmax_bwd", gz.data_ptr, gc.data_ptr, xc.data_ptr, rs.ptr, rm.ptr, R, C,
                   None)
        return gz

    return record("softmax", (x,), y, (pull,), saved=(xc,))


def _gemm_consumes_as_3xbf16(rows, cols) -> bool:
    """Would a GEMM reading an [rows, cols] cotangent (x_bar = g . W, W_bar =
    g^T . x) run the 3xBF16 tensor-core scheme? Then a producer can emit the
    split that GEMM reads instead of the fp32 tensor."""
    algo = _ALGO_OVERRIDE
    if algo is None:
        sel = ctypes.c_int()
        L.check(L.lib().b2_gemm_select(0, 0, rows, cols, cols, cols, cols, ctypes.byref(sel)))
        algo = sel.value
    return algo == L.GEMM_3XBF16


def softmax_mul_mean(z, t) -> Tensor:
    """mean(softmax(z, -1) * t) -- BASELINE config 4's loss -- with one row pass
    each way (b2_softmax_wmean_fwd/bwd), bit-identical to the composition
    softmax -> mul -> mean (core.py:469-476, 663-689). The
    backward hands its consumers what they read: the 3xBF16 split of z's
    cotangent when a tensor-core GEMM consumes it (the fp32 values are then
    materialised only on first fp32 use, as for split-only GEMM outputs), and
    its column sums (the bias gradient of a Linear that produced z, picked up
    by reduce_to_shape). Falls back to the composed ops for shapes the fused
    kernels do not take or a t that requires a gradient."""
    z = _as_tensor(_as_operand(z))
    t = _as_tensor(_as_operand(t))
    if z.shape != t.shape:
        t = _expand_view(t, broadcast_shapes(z.shape, t.shape)) if z.ndim else t
    C = z.shape[-1] if z.ndim else 0
    R = z.size // C if C else 0
    fusable = (z.ndim >= 1 and C % 4 == 0 and 0 < C <= 1024 and R > 0 and not t.requires_grad
               and t.shape == z.shape and t.is_contiguous)
    zc = z if z.is_contiguous else _copy_contig(z)
    if fusable and (zc.data_ptr % 16 or t.data_ptr % 16):
        fusable = False
    if not fusable:
        return mean(mul(softmax(z), t))
    loss = _empty(())
    rs, rm = Buffer(4 * R), Buffer(4 * R)
    rdot = Buffer(8 * R)
    L.call("b2_softmax_wmean_fwd", loss.data_ptr, None, rs.ptr, rm.ptr, rdot.ptr, zc.data_ptr,
           t.data_ptr, R, C, None)
    count_f32 = float(np.float32(float(z.size)))  # mean's divisor, promoted like a scalar

    def pull(g):
        from .graph import _capturing

        gz = _empty(z.shape)
        cs = _empty((C,)) if z.ndim == 2 else None
        split = (_LAZY_FP32 and z.ndim == 2 and C % 8 == 0 and _gemm_consumes_as_3xbf16(R, C))
        hi = Buffer(2 * R * C) if split else None
        lo = Buffer(2 * R * C) if split else None
        L.call("b2_softmax_wmean_bwd", None if split else gz.data_ptr, hi.ptr if split else None,
               lo.ptr if split else None, cs.data_ptr if cs is not None else None, g.data_ptr,
               count_f32, zc.data_ptr, t.data_ptr, rs.ptr, rm.ptr, R, C, None)
        if split:
            buf = gz.buffer
            buf._splits = {("3xbf16", 0, R, C, C): (buf.version, hi, lo, _capturing[0])}
            _set_pending(buf, hi, lo, R * C)
        if cs is not None:
            _COLSUM[gz] = cs
        return gz

    return record("softmax_mul_mean", (z,), loss, (pull,), saved=(zc, t))


def fused_muladd_relu(a, b, c=None) -> Tensor:
    """relu(a*b + c) for a (R, C) and row vectors b, c of length C in one pass
    (the BASELINE config-2 chain, core.py:453-483 + nn.py:108-111); c defaults
    to b. One tape node whose pullback is the composed reference pullback in
    GradStore order (autograd.py:140-145), so gradients are bit-identical."""
    if c is None:
        c = b
    if a.ndim != 2 or b.size != a.shape[1] or c.size != a.shape[1]:
        raise ShapeError("fused_muladd_relu expects a (R, C) with row vectors of length C")
    R, C = a.shape
    if not (a.is_contiguous and b.is_contiguous and c.is_contiguous) or C % 4:
        return relu(add(mul(a, b), c))
    y = _empty(a.shape)
    L.call("b2_fused_muladd_relu_fwd", y.data_ptr, a.data_ptr, b.data_ptr, c.data_ptr, R, C, None)
    memo = [None, None]
    yk = y.detach()

    def pre(g):
        if memo[0] is not g:
            memo[0], memo[1] = g, _launch_binary(L.RELU_BWD, g, yk, yk.shape)
        return memo[1]

    if c is b:
        return record("muladd_relu", (a, b), y,
                      (lambda g: mul(pre(g), b),
                       lambda g: add(reduce_to_shape(pre(g), b.shape),
                                     reduce_to_shape(mul(pre(g), a), b.shape))),
                      saved=(a, b))
    return record("muladd_relu", (a, b, c), y,
                  (lambda g: mul(pre(g), b),
                   lambda g: reduce_to_shape(mul(pre(g), a), b.shape),
                   lambda g: reduce_to_shape(pre(g), c.shape)), saved=(a, b, c))


def muladd_relu_stats(a, b, clip=(-10.0, 10.0)) -> dict:
    """BASELINE config 2's whole workload with ONE read of `a` (b2_muladd_relu_stats):
    y = relu(a*b + b), e = exp(clamp(a)), the sum/mean/max of y over dim 0
    and dim 1, its full sum, and the gradients of sum(y) w.r.t. a and b --
    bit-identical to the separate ops (fused_muladd_relu, clamp/exp, sum, mean,
    max, muladd_relu_sum_grads). Nothing is recorded on the tape. Returns a
    dict with keys y, e, sum0, mean0, max0, sum1, mean1, max1, sum_all,
    grad_a, grad_b. Falls back to those ops for layouts the kernel does not
    take (a non-contiguous, cols % 4 != 0)."""
    a = _as_tensor(_as_operand(a))
    b = _as_tensor(_as_operand(b))
    if a.ndim != 2 or b.size != a.shape[1]:
        raise ShapeError("muladd_relu_stats expects a (R, C) and a row vector b of length C")
    R, C = a.shape
    lo, hi = float(clip[0]), float(clip[1])
    if not (a.is_contiguous and b.is_contiguous and C % 4 == 0 and R > 0 and C > 0
            and a.data_ptr % 16 == 0 and b.data_ptr % 16 == 0):
        with no_grad():
            y = fused_muladd_relu(a, b)
            out = {"y": y, "e": exp(clamp(a, lo, hi)), "sum_all": sum(y)}
            for d in (0, 1):
                out[f"sum{d}"], out[f"mean{d}"], out[f"max{d}"] = sum(y, d), mean(y, d), max(y, d)
        out["grad_a"], out["grad_b"] = muladd_relu_sum_grads(a, b)
        return out
    out = {"y": _empty((R, C)), "e": _empty((R, C)), "grad_a": _empty((R, C)),
           "grad_b": _empty(b.shape), "sum0": _empty((C,)), "mean0": _empty((C,)),
           "max0": _empty((C,)), "sum1": _empty((R,)), "mean1": _empty((R,)), "max1": _empty((R,)),
           "sum_all": _empty(())}
    ptr = {k: v.data_ptr for k, v in out.items()}
    L.call("b2_muladd_relu_stats", ptr["y"], ptr["e"], ptr["grad_a"], ptr["grad_b"], ptr["sum0"],
           ptr["mean0"], ptr["max0"], ptr["sum1"], ptr["mean1"], ptr["max1"], ptr["sum_all"],
           a.data_ptr, b.data_ptr, lo, hi, R, C, None)
    return out


def muladd_relu_sum_grads(a, b):
    """Gradients of sum(relu(a*b + b)) w.r.t. a (R, C) and b (C,) / (1, C) in
    ONE pass over a (fused op+grad kernel): ga = f32(mask*b) and
    gb = f32(count) + f32(sum64(mask*a)) in GradStore order. Bit-identical to
    backward(sum(relu(add(mul(a, b), b)))) on the reference."""
    R, C = a.shape
    ga = _empty(a.shape)
    gb = _empty(b.shape)
    L.call("b2_fused_muladd_relu_bwd", ga.data_ptr, gb.data_ptr, a.data_ptr, b.data_ptr, R, C, None)
    return ga, gb
