"""DLPack exchange of device tensors (host exchange fidelity).

The reference aliases NumPy storage (tlnp.py:272-305); HBM cannot alias host
memory, so the zero-copy exchange that makes sense on a B200 is device-side:
``__dlpack__`` hands any DLPack consumer (``torch.from_dlpack``, CuPy, JAX) a
view of the tensor's HBM -- same pointer, shape, element strides, byte
offset -- and ``from_dlpack`` wraps a producer's CUDA float32 tensor as an
engine tensor without a copy. Stream contract: the producer side
synchronises the engine stream before handing out a capsule; on import the
producer is asked to make its data ready for the engine stream.
"""

from __future__ import annotations

import ctypes
from ctypes import (CFUNCTYPE, POINTER, Structure, c_int, c_int32, c_int64, c_uint8, c_uint16,
                    c_uint64, c_void_p)

from . import _lib as L

kDLCUDA = 2
kDLFloat = 2


class DLDevice(Structure):
    _fields_ = [("device_type", c_int32), ("device_id", c_int32)]


class DLDataType(Structure):
    _fields_ = [("code", c_uint8), ("bits", c_uint8), ("lanes", c_uint16)]


class DLTensor(Structure):
    _fields_ = [("data", c_void_p), ("device", DLDevice), ("ndim", c_int32),
                ("dtype", DLDataType), ("shape", POINTER(c_int64)),
                ("strides", POINTER(c_int64)), ("byte_offset", c_uint64)]


class DLManagedTensor(Structure):
    pass


_Deleter = CFUNCTYPE(None, POINTER(DLManagedTensor))
DLManagedTensor._fields_ = [("dl_tensor", DLTensor), ("manager_ctx", c_void_p),
                            ("deleter", _Deleter)]

_api = ctypes.pythonapi
_api.PyCapsule_New.restype = ctypes.py_object
_api.PyCapsule_New.argtypes = [c_void_p, ctypes.c_char_p, c_void_p]
_api.PyCapsule_GetPointer.restype = c_void_p
_api.PyCapsule_GetPointer.argtypes = [ctypes.py_object, ctypes.c_char_p]
_api.PyCapsule_IsValid.restype = c_int
_api.PyCapsule_IsValid.argtypes = [ctypes.py_object, ctypes.c_char_p]
_api.PyCapsule_SetName.restype = c_int
_api.PyCapsule_SetName.argtypes = [ctypes.py_object, ctypes.c_char_p]

_LIVE = {}  # manager_ctx -> (engine tensor keep-alive, shape, strides, managed struct)


def _free(ptr):
    if not ptr:
        return
    key = ptr.contents.manager_ctx
    _LIVE.pop(key, None)


_DELETER = _Deleter(_free)

_CapsuleDtor = CFUNCTYPE(None, c_void_p)
# raw-pointer prototypes for use inside the capsule destructor, where the
# capsule is mid-destruction and must not be wrapped in a new reference
_IsValidRaw = ctypes.PYFUNCTYPE(c_int, c_void_p, ctypes.c_char_p)(("PyCapsule_IsValid", _api))
_GetPointerRaw = ctypes.PYFUNCTYPE(c_void_p, c_void_p, ctypes.c_char_p)(("PyCapsule_GetPointer", _api))


def _capsule_dtor(cap_ptr):
    # an unconsumed capsule still carries the name "dltensor": release it
    if _IsValidRaw(cap_ptr, b"dltensor"):
        p = _GetPointerRaw(cap_ptr, b"dltensor")
        _free(ctypes.cast(p, POINTER(DLManagedTensor)))


_CAPSULE_DTOR = _CapsuleDtor(_capsule_dtor)
_serial = [0]


def device_id() -> int:
    """The engine's device (one GPU per process, b2_init(LOCAL_RANK))."""
    import os

    try:
        return int(os.environ.get("LOCAL_RANK", 0))
    except ValueError:
        return 0


def to_capsule(t, stream=None):
    """A DLPack capsule viewing tensor t's HBM (no copy)."""
    # materialise fp32 contents a GEMM left as a split only FIRST: the join is
    # queued on the engine stream and must precede the event / sync below
    t.data_ptr
    if stream is not None and stream not in (-1, 0, 1, 2):
        # the consumer will use `stream`; make the engine's queued work visible to it
        ev = L.Event()
        ev.record(None)
        L.call("b2_stream_wait_event", ctypes.c_void_p(int(stream)), ev.h)
    else:
        L.synchronize()
    nd = t.ndim
    shape = (c_int64 * max(nd, 1))(*t.shape)
    strides = (c_int64 * max(nd, 1))(*t.strides)
    mt = DLManagedTensor()
    mt.dl_tensor.data = t.buffer.ptr
    mt.dl_tensor.device = DLDevice(kDLCUDA, device_id())
    mt.dl_tensor.ndim = nd
    mt.dl_tensor.dtype = DLDataType(kDLFloat, 32, 1)
    mt.dl_tensor.shape = ctypes.cast(shape, POINTER(c_int64))
    mt.dl_tensor.strides = ctypes.cast(strides, POINTER(c_int64))
    mt.dl_tensor.byte_offset = 4 * t.offset
    _serial[0] += 1
    key = _serial[0]
    mt.manager_ctx = key
    mt.deleter = _DELETER
    _LIVE[key] = (t, shape, strides, mt)
    return _api.PyCapsule_New(ctypes.addressof(mt), b"dltensor",
                              ctypes.cast(_CAPSULE_DTOR, c_void_p))


def from_dlpack(obj):
    """Wrap a DLPack producer's CUDA float32 tensor as an engine Tensor that
    aliases its memory (no copy). The producer stays alive as long as the
    engine tensor (or any view of it) does."""
    from . import core

    L.ensure_device()
    if hasattr(obj, "__dlpack__"):
        s = ctypes.c_void_p()
        L.check(L.lib().b2_default_stream(ctypes.byref(s)))
        try:
            cap = obj.__dlpack__(stream=s.value or 1)
        except TypeError:
            cap = obj.__dlpack__()
    else:
        cap = obj
    if not _api.PyCapsule_IsValid(cap, b"dltensor"):
        raise TypeError("expected a DLPack capsule or an object with __dlpack__")
    p = ctypes.cast(_api.PyCapsule_GetPointer(cap, b"dltensor"), POINTER(DLManagedTensor))
    dl = p.contents.dl_tensor
    if dl.device.device_type != kDLCUDA:
        raise TypeError("from_dlpack needs a CUDA tensor (host arrays: tlnp.wrap_host_array)")
    if (dl.dtype.code, dl.dtype.bits, dl.dtype.lanes) != (kDLFloat, 32, 1):
        raise TypeError("from_dlpack supports float32 tensors only")
    nd = dl.ndim
    shape = tuple(dl.shape[i] for i in range(nd))
    if dl.strides:
        strides = tuple(dl.strides[i] for i in range(nd))
    else:
        strides = core._contig_strides(shape)
    if dl.byte_offset % 4:
        raise TypeError("byte offset is not a multiple of 4")
    _api.PyCapsule_SetName(cap, b"used_dltensor")
    span = 1 + sum((s - 1) * st for s, st in zip(shape, strides) if s > 0)
    buf = core.ExternalBuffer(dl.data, 4 * (span + dl.byte_offset // 4), owner=(obj, cap, p))
    return core.Tensor(buf, shape, strides, offset=dl.byte_offset // 4)


def release(owner):
    """Call a consumed managed tensor's deleter (ExternalBuffer teardown)."""
    _obj, _cap, p = owner
    if p and p.contents.deleter:
        p.contents.deleter(p)
