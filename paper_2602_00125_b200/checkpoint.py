"""Checkpoint / resume (optional ``state_dict`` via named
parameters -> NumPy .npz).

The reference has no checkpointing (a non-goal there); its stable parameter
names ``layer{i}.{name}`` (nn.py:531-536) make one natural. A checkpoint
holds every named parameter and buffer of a model (float32) and, optionally,
an optimizer's step counts and fp64 slots -- everything a resumed run needs
to continue bit-identically (the update kernels are deterministic).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib as L
from .errors import ShapeError


def model_state(model) -> dict:
    """{name: float32 array} of the model's parameters and buffers."""
    out = {}
    for name, p in model.named_parameters():
        out[name] = p.numpy()
    for name, b in model.named_buffers():
        out[name] = b.numpy()
    return out


def load_model_state(model, state: dict):
    """Write a model_state() dict back into the model's tensors (in place)."""
    named = dict(model.named_parameters())
    named.update(dict(model.named_buffers()))
    missing = [k for k in named if k not in state]
    if missing:
        raise KeyError(f"checkpoint lacks {', '.join(missing)}")
    for name, t in named.items():
        arr = np.asarray(state[name], np.float32)
        if arr.shape != t.shape:
            raise ShapeError(f"{name}: checkpoint shape {arr.shape} != {t.shape}")
        t.write_flat(arr)


def _read_slot(buf, n) -> np.ndarray:
    out = np.empty(max(n, 1), np.float64)
    L.call("b2_memcpy_d2h", out.ctypes.data_as(ctypes.c_void_p), buf.ptr, 8 * max(n, 1), None)
    return out[:n]


def _write_slot(buf, arr):
    arr = np.ascontiguousarray(arr, np.float64)
    if arr.size:
        L.call("b2_memcpy_h2d", buf.ptr, arr.ctypes.data_as(ctypes.c_void_p), arr.nbytes, None)
        L.synchronize()


def optimizer_state(optimizer, named_params) -> dict:
    """{f"{name}/t": step, f"{name}/slot{k}": fp64 slot} for every parameter
    the optimizer has state for (named_params: [(name, tensor)])."""
    out = {}
    for name, p in named_params:
        st = optimizer._state.get(id(p))
        if st is None:
            continue
        out[f"{name}/t"] = np.array(st["t"], np.int64)
        for k, buf in enumerate(st["slots"]):
            out[f"{name}/slot{k}"] = _read_slot(buf, p.size)
    return out


def load_optimizer_state(optimizer, named_params, state: dict):
    for name, p in named_params:
        if f"{name}/t" not in state:
            continue
        st = optimizer.state_for(p)
        st["t"] = int(state[f"{name}/t"])
        for k, buf in enumerate(st["slots"]):
            slot = np.asarray(state[f"{name}/slot{k}"], np.float64)
            if slot.size != p.size:
                raise ShapeError(f"{name}: optimizer slot has {slot.size} values, expected {p.size}")
            _write_slot(buf, slot)


def save(path, model, optimizer=None):
    """One .npz with the model state and, if given, the optimizer state."""
    arrays = {f"model/{k}": v for k, v in model_state(model).items()}
    if optimizer is not None:
        st = optimizer_state(optimizer, model.named_parameters())
        arrays.update({f"optim/{k}": v for k, v in st.items()})
    np.savez(path, **arrays)


def load(path, model, optimizer=None):
    with np.load(path) as z:
        model_part = {k[len("model/"):]: z[k] for k in z.files if k.startswith("model/")}
        optim_part = {k[len("optim/"):]: z[k] for k in z.files if k.startswith("optim/")}
    load_model_state(model, model_part)
    if optimizer is not None:
        load_optimizer_state(optimizer, model.named_parameters(), optim_part)
