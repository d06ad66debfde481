"""Data-parallel training over NCCL (new: the reference is single-process,
SURVEY 2.1 / 8e).

One process per GPU (torchrun / torch.distributed.run env). The NCCL unique
id travels over torch.distributed's TCPStore -- torch is plumbing here; the
communicator itself lives in libb2 (b2_comm_init / b2_allreduce_f32) and the
all-reduce runs on a libb2 stream next to the backward kernels.

Config 5 is the only partitioned path: every rank holds a full replica,
takes a contiguous 1/N slice of the global batch, computes the mean loss of
its slice, and gradients are averaged (ncclAvg) -- the mean of equal-shard
means is the global mean. Gradient all-reduces are issued as soon as a
parameter's last gradient contribution has been queued by ``backward``
(reverse layer order), on a dedicated communication stream, so they overlap
the remaining backward GEMMs; the optimizer's stream waits for them.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

from . import _lib as L

AVG, SUM, MAX = 1, 0, 2


@dataclass
class Env:
    rank: int = 0
    world: int = 1
    local_rank: int = 0
    master_addr: str = "127.0.0.1"
    master_port: int = 29500


def env_from_os() -> Env:
    return Env(rank=int(os.environ.get("RANK", 0)), world=int(os.environ.get("WORLD_SIZE", 1)),
               local_rank=int(os.environ.get("LOCAL_RANK", 0)),
               master_addr=os.environ.get("MASTER_ADDR", "127.0.0.1"),
               master_port=int(os.environ.get("MASTER_PORT", 29500)))


def shard_rows(global_rows: int, rank: int, world: int):
    """Contiguous [start, stop) rows of rank's shard; equal shards required so
    that the average of shard means is the global mean."""
    if global_rows % world:
        raise ValueError(f"global batch {global_rows} is not divisible by {world} ranks")
    per = global_rows // world
    return rank * per, (rank + 1) * per


def exchange_unique_id(store, rank: int, make_uid, key="b2/nccl_uid") -> bytes:
    """Rank 0 publishes `make_uid()` under `key`; everyone returns it.
    `store` is any torch.distributed Store (TCPStore / FileStore / HashStore)."""
    if rank == 0:
        uid = bytes(make_uid())
        store.set(key, uid)
        return uid
    store.wait([key])
    return bytes(store.get(key))


def make_store(env: Env, port_offset=1):
    """The key-value store the NCCL unique id travels through. Under torchrun
    (TORCHELASTIC_USE_AGENT_STORE=True) every rank joins the elastic agent's
    own TCPStore at MASTER_PORT as a client -- no second port to collide on;
    otherwise (bench.py's launcher, a hand-set env) rank 0 hosts a TCPStore at
    MASTER_PORT + port_offset."""
    import datetime

    from torch.distributed import TCPStore

    timeout = datetime.timedelta(seconds=300)
    if os.environ.get("TORCHELASTIC_USE_AGENT_STORE", "").lower() == "true":
        return TCPStore(env.master_addr, env.master_port, env.world, False, timeout=timeout)
    return TCPStore(env.master_addr, env.master_port + port_offset, env.world, env.rank == 0,
                    timeout=timeout)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    L.check(L.lib().b2_comm_unique_id(buf))
    return buf.raw


class Communicator:
    """libb2's NCCL communicator for this process's GPU.

    ``active`` is True when NCCL is in use: always for world > 1, and for a
    single process when ``force_nccl`` is set (exercises the exact N>1 code
    path -- uid exchange, comm stream, in-place ncclAvg -- on one GPU)."""

    def __init__(self, env: Env, store=None, force_nccl=False):
        self.env = env
        L.ensure_device(env.local_rank)
        self.comm_stream = None
        self.active = env.world > 1 or force_nccl
        if self.active:
            if store is None:
                if env.world > 1:
                    store = make_store(env)
                else:
                    from torch.distributed import HashStore

                    store = HashStore()
            self._store = store
            # SMs for the collectives: with more than one rank (or B2_COMM_SMS
            # set) NCCL is capped to `sm_reserve` CTAs and, while a backward's
            # collectives are in flight (GradReducer), the persistent GEMMs
            # leave as many SMs free, so the reduce-scatters / all-gathers of
            # the upper layers run beside the lower layers' backward GEMMs
            # instead of waiting for a GEMM boundary (NCCL's kernels cannot be
            # co-resident with a 640-thread, ~200 KB-smem GEMM CTA)
            self.sm_reserve = 0
            if env.world > 1 or "B2_COMM_SMS" in os.environ:
                # 8 SMs at 2 ranks, 16 beyond (measured on one GPU: reserving 8 / 16
                # SMs costs the 65536-row step 1.3% / 2.2% at the power cap and
                # nothing at the 8192 rows per rank of N = 8, where it even
                # lets the overlapped optimizer run beside the GEMMs)
                self.sm_reserve = max(0, int(os.environ.get("B2_COMM_SMS", "8" if env.world <= 2 else "16")))
                if self.sm_reserve:
                    os.environ.setdefault("NCCL_MAX_CTAS", str(self.sm_reserve))
            uid = exchange_unique_id(store, env.rank, nccl_unique_id)
            L.check(L.lib().b2_comm_init(env.rank, env.world, uid))
            s = ctypes.c_void_p()
            L.check(L.lib().b2_stream_create_priority(ctypes.byref(s)))
            self.comm_stream = s.value

    @property
    def world(self):
        return self.env.world

    def allreduce_(self, t, op=AVG, stream=None):
        if self.active and t.size:
            L.call("b2_allreduce_f32", t.data_ptr, t.size, op, stream)
        return t

    def check(self):
        """Raise if the communicator reports an asynchronous NCCL error."""
        if not self.active:
            return
        err = ctypes.c_int(0)
        L.check(L.lib().b2_comm_async_error(ctypes.byref(err)))
        if err.value not in (0, 7):  # 7 = ncclInProgress
            raise RuntimeError(f"NCCL asynchronous error {err.value}")

    def wait(self, timeout_s: float):
        """Host wait for the communication stream with a deadline; on an NCCL
        error or a timeout the communicator is aborted and RuntimeError raised
        (a dead peer fails the step instead of hanging it)."""
        if self.active:
            L.check(L.lib().b2_stream_wait_timeout(self.comm_stream, float(timeout_s) * 1000.0))

    def barrier(self):
        if self.active:
            from . import core as T

            t = T.ones((1,))
            self.allreduce_(t, SUM)
        L.call("b2_device_sync")

    # ---- the device plumbing GradReducer drives (a test double replaces these)

    _side = None  # per-process side stream for single-process optimizer overlap

    def side_stream(self):
        """The stream gradient averaging / overlapped updates run on."""
        if self.active:
            return self.comm_stream
        if Communicator._side is None:
            s = ctypes.c_void_p()
            L.check(L.lib().b2_stream_create(ctypes.byref(s)))
            Communicator._side = s.value
        return Communicator._side

    def after_compute(self, stream):
        """Order `stream` after everything queued so far on the engine stream;
        returns the event (kept alive by the caller until the step ends)."""
        ev = L.Event()
        ev.record(None)
        L.call("b2_stream_wait_event", stream, ev.h)
        return ev

    def join(self, stream):
        """Order the engine stream after everything queued so far on `stream`."""
        done = L.Event()
        done.record(stream)
        L.call("b2_stream_wait_event", None, done.h)

    def private_copy(self, t):
        """A fresh contiguous copy of t (engine stream)."""
        from .core import _copy_contig

        return _copy_contig(t)

    # ---- sharded optimizer step (ZeRO-1 style)

    def shard_view(self, p):
        """This rank's contiguous 1/world slice of parameter p as a persistent
        1-D view (the optimizer keys its slots by it, so they hold 1/world of
        the parameter)."""
        if not hasattr(self, "_shards"):
            self._shards = {}
        v = self._shards.get(id(p))
        if v is None or v.buffer is not p.buffer:
            from .core import Tensor

            cnt = p.size // self.world
            v = Tensor(p.buffer, (cnt,), offset=p.offset + self.env.rank * cnt)
            self._shards[id(p)] = v
        return v

    def new_shard(self, cnt):
        from .core import _empty

        return _empty((cnt,))

    def reduce_scatter_(self, send, recv, op=AVG, stream=None):
        L.call("b2_reduce_scatter_f32", send.data_ptr, recv.data_ptr, recv.size, op, stream)
        return recv

    def all_gather_(self, t, cnt, stream=None):
        L.call("b2_all_gather_f32", t.data_ptr, cnt, self.env.rank, stream)
        return t

    def max_scalar(self, v: float) -> float:
        """Max of a host float over ranks (device NCCL allreduce)."""
        if not self.active:
            return v
        from . import core as T

        t = T.full((1,), v)
        self.allreduce_(t, MAX)
        return t.item()


class GradReducer:
    """Overlapped gradient averaging -- and optionally the optimizer update --
    for one backward pass.

    Pass ``hook`` as ``backward(loss, on_leaf_ready=reducer.hook)``; call
    ``finish()`` before the next use of the parameters. Each leaf gradient is
    averaged in place on the communication stream as soon as backward has
    queued its last contribution, so the all-reduces of the upper layers
    overlap the GEMMs of the lower ones. With ``optimizer`` (and ``params``),
    the parameter's update is launched on the same side stream right after
    its all-reduce (or right away for a single process): a layer's weights
    are no longer read once its last gradient is queued, so the HBM-bound
    update kernels overlap the remaining tensor-core GEMMs of the backward.
    Leaf gradients of Dense layers are fresh tensors and are averaged in
    place; an aliased or strided one is averaged as a private copy."""

    def __init__(self, comm: Communicator, params=None, timeout_s=None, optimizer=None, shard=None):
        self.comm = comm
        # sharded update (default when several ranks exchange gradients):
        # reduce-scatter -> the optimizer on this rank's 1/N shard -> all-gather
        # of the updated parameter; same wire bytes as the all-reduce, 1/N of
        # the optimizer's HBM traffic and fp64 slot memory
        self.shard = (comm.active and comm.world > 1) if shard is None else bool(shard)
        self._pending = []
        if timeout_s is None:
            env = os.environ.get("B2_COMM_TIMEOUT_S")
            timeout_s = float(env) if env else None
        self.timeout_s = timeout_s  # None: stay asynchronous (no host wait)
        self.optimizer = optimizer
        self.params = list(params) if params is not None else []
        self._by_node = None
        self._used = False
        self._reserved = False
        self._updated = set()
        if optimizer is not None and not params:
            raise ValueError("GradReducer(optimizer=...) needs the parameter list")

    def _param(self, node_id):
        if self._by_node is None:
            self._by_node = {p.node.id: p for p in self.params if p.node is not None}
        return self._by_node.get(node_id)

    def hook(self, node_id, grad):
        """on_leaf_ready hook: average `grad` over the ranks on the side stream
        (and launch the parameter's update after it). A gradient that does not
        own its whole buffer exclusively -- a view, or a first contribution the
        store shares with another cotangent (autograd.grad_is_exclusive) -- is
        first copied to a fresh contiguous tensor on the engine stream; that
        copy is what gets averaged, updated from, and returned so the store
        holds the averaged gradient."""
        if not self.comm.active and self.optimizer is None:
            return None
        if not self._reserved and self.comm.active and getattr(self.comm, "sm_reserve", 0):
            # collectives from here on: the remaining backward GEMMs leave SMs free
            L.call("b2_gemm_set_sm_reserve", self.comm.sm_reserve)
            self._reserved = True
        if self.optimizer is not None and self.shard and self.comm.active:
            p = self._param(node_id)
            if p is not None and p.is_contiguous and p.size and p.size % self.comm.world == 0:
                return self._sharded_step(p, grad)
        from .autograd import grad_is_exclusive

        if (self.comm.active and not grad_is_exclusive(grad)) or not grad.is_contiguous:
            grad = self.comm.private_copy(grad)  # averaged / updated from a private copy
        handle = None
        if self.optimizer is not None:
            p = self._param(node_id)
            if p is not None:
                # slot creation goes on the engine stream BEFORE the event the
                # side stream waits on
                handle = self.optimizer.prepare([(p, grad)])
                self._updated.add(id(p))
        s = self.comm.side_stream()
        ev = self.comm.after_compute(s)  # grad produced on the compute stream
        if self.comm.active:
            self.comm.allreduce_(grad, AVG, s)
        if handle is not None:
            self.optimizer.launch(handle, stream=s)
        self._pending.append((ev, grad, handle))
        self._used = True
        return grad

    def _sharded_step(self, p, grad):
        """reduce-scatter(grad) -> update of this rank's shard -> all-gather(p),
        in that order on the side stream after the gradient is produced. The
        gradient itself is only read (never averaged in place), so aliasing
        cannot bite; the store keeps this rank's local gradient."""
        g = grad if grad.is_contiguous else self.comm.private_copy(grad)
        cnt = p.size // self.comm.world
        view = self.comm.shard_view(p)
        gs = self.comm.new_shard(cnt)
        handle = self.optimizer.prepare([(view, gs)])  # slot creation on the engine stream first
        self._updated.add(id(p))
        s = self.comm.side_stream()
        ev = self.comm.after_compute(s)
        self.comm.reduce_scatter_(g, gs, AVG, s)
        self.optimizer.launch(handle, stream=s)
        self.comm.all_gather_(p, cnt, s)
        self._pending.append((ev, g, (gs, handle)))
        self._used = True
        return None

    def finish(self):
        if self._reserved:  # the GEMMs queued after the backward use every SM again
            L.call("b2_gemm_set_sm_reserve", 0)
            self._reserved = False
        if not self._used:
            return
        if self.comm.active and self.timeout_s is not None:
            self.comm.wait(self.timeout_s)  # failure detection: error/timeout -> abort + raise
        self.comm.join(self.comm.side_stream())  # the next user of the params waits
        self._pending.clear()

    def step_rest(self, store):
        """Optimizer step (engine stream) for parameters that have a gradient
        but were not updated by the hook; returns how many."""
        if self.optimizer is None:
            return 0
        rest = [(p, store.get(p)) for p in self.params
                if id(p) not in self._updated and store.get(p) is not None]
        return self.optimizer.step_many(rest)
