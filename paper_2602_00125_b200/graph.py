"""CUDA-graph capture of engine work (b2_graph_* in include/b2.h).

A small step (BASELINE config 1: ~40 kernels of a few microseconds each) is
launch-latency bound when driven eagerly from Python; capturing it once and
replaying the graph issues the whole step as a single launch.

    g = graph.capture(step)   # runs step() once eagerly (warm-up), then captures it
    g.replay()                 # replays every kernel of step() on the same buffers

The captured function must only launch kernels: no host reads (``item()``,
``numpy()``) and no host->device uploads inside it. Buffers it allocates stay
owned by the graph; tensors it returns (``g.outputs``) are rewritten by every
replay. Cached 3xTF32/TF32X operand splits made before the capture are not
trusted inside it, so every split the step needs is part of the graph.
"""

from __future__ import annotations

import ctypes

from . import _lib as L

_capturing = [0]  # id of the open capture (unique per capture), 0 when none
_serial = [0]
_captured_pending = []  # (weakref(buffer), hi, lo, n) split-only outputs made by the open capture


def capturing() -> bool:
    return _capturing[0] != 0


class CudaGraph:
    def __init__(self, gid: int, outputs, repend=()):
        self.id = gid
        self.outputs = outputs
        # split-only GEMM / loss-pullback outputs still pending when the
        # capture ended: every replay rewrites their split, so their fp32
        # contents are pending again (materialised on first fp32 use)
        self._repend = list(repend)

    def replay(self, stream=None):
        L.call("b2_graph_launch", self.id, stream)
        if self._repend:
            from .core import _PENDING

            for ref, hi, lo, n in self._repend:
                buf = ref()
                if buf is not None:
                    buf._pending = (hi, lo, n)
                    _PENDING.add(buf)

    def __del__(self):
        try:
            if L._lib is not None and self.id:
                L._lib.b2_graph_destroy(self.id)
        except Exception:
            pass
        self.id = 0


def capture(fn, *args, warmup: int = 1, **kwargs) -> CudaGraph:
    for _ in range(warmup):
        fn(*args, **kwargs)
    from .core import materialize_pending

    materialize_pending()  # a materialisation captured in the graph would only run at replay
    L.synchronize()
    L.call("b2_graph_begin", None)
    _serial[0] += 1
    _capturing[0] = _serial[0]
    _captured_pending.clear()
    try:
        out = fn(*args, **kwargs)
    except BaseException:
        gid = ctypes.c_int(0)
        L.lib().b2_graph_end(None, ctypes.byref(gid))
        raise
    finally:
        _capturing[0] = 0
    gid = ctypes.c_int(0)
    L.check(L.lib().b2_graph_end(None, ctypes.byref(gid)))
    repend = [e for e in _captured_pending if e[0]() is not None and e[0]()._pending is not None]
    _captured_pending.clear()
    return CudaGraph(gid.value, out, repend)
