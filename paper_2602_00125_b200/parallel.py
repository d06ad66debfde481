"""Work partitioning controls (tensorlite/parallel.py:16-63) on a device engine.

The reference splits big kernels at fixed 65536-element boundaries and
combines chunk results in chunk order, so its numbers never depend on how
many host workers run the chunks; ``max_workers`` / ``thread_limit`` /
``TENSORLITE_THREADS`` only choose that worker count. Here the kernels run on
the GPU with partitions fixed by the problem shape and the device (two-stage
and cluster reductions fold their partials in a fixed order -- DESIGN.md
section 4), so the same contract holds by construction: the worker setting is
kept (programs written against the reference read and set it) and has no
effect on any result. ``spans`` is the reference's worker-independent chunk
partition, for host code that sizes per-chunk work.
"""

from __future__ import annotations

import os
import threading
from contextlib import contextmanager

CHUNK = 1 << 16

_forced = threading.local()  # thread_limit() nests per host thread, like the tape


def max_workers() -> int:
    """The host worker count a reference program would get: the innermost
    thread_limit(), else TENSORLITE_THREADS, else min(cpu_count, 8)."""
    forced = getattr(_forced, "stack", None)
    if forced:
        return forced[-1]
    try:
        return max(1, int(os.environ["TENSORLITE_THREADS"]))
    except (KeyError, ValueError):
        return min(os.cpu_count() or 1, 8)


@contextmanager
def thread_limit(n: int):
    """Set max_workers() for the dynamic extent. Device results do not depend on it."""
    stack = getattr(_forced, "stack", None)
    if stack is None:
        stack = _forced.stack = []
    stack.append(max(1, int(n)))
    try:
        yield
    finally:
        stack.pop()


def spans(n: int):
    """[start, stop) chunk boundaries covering range(n) at CHUNK multiples."""
    return [(lo, min(lo + CHUNK, n)) for lo in range(0, max(n, 0), CHUNK)]
