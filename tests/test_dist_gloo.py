"""World-size-2 CPU tests (gloo) of the data-parallel host logic
(paper_2602_00125_b200/dist.py): NCCL unique-id exchange over the TCP store,
equal contiguous batch shards, and the DP semantics the device path relies
on -- averaging the per-shard gradients of per-shard MEAN losses reproduces
the full-batch gradient (checked with the oracle on each rank)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as tdist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outq):
    import datetime
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import tensorlite_np as O
    from paper_2602_00125_b200 import dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    tdist.init_process_group("gloo", rank=rank, world_size=world,
                             timeout=datetime.timedelta(seconds=120))
    env = dist.env_from_os()
    assert env.rank == rank and env.world == world
    # 1) unique-id exchange over the TCP store (what Communicator does for NCCL)
    store = dist.make_store(env, port_offset=7)
    uid = dist.exchange_unique_id(store, rank, lambda: bytes(range(128)) if rank == 0 else b"x" * 128)
    # 2) shards + DP gradient semantics with the oracle
    rng = np.random.default_rng(0)
    B, D, H, Cc = 32, 12, 16, 5
    x = rng.standard_normal((B, D)).astype(np.float32)
    labels = rng.integers(0, Cc, B)
    params = [(rng.uniform(-0.3, 0.3, (H, D)).astype(np.float32), np.zeros(H, np.float32)),
              (rng.uniform(-0.3, 0.3, (Cc, H)).astype(np.float32), np.zeros(Cc, np.float32))]

    class NoOpt:
        def step(self, key, th, g):
            return th

    lo, hi = dist.shard_rows(B, rank, world)
    r = O.mlp_train_step(params, x[lo:hi], labels[lo:hi], NoOpt())
    grads = [torch.from_numpy(np.ascontiguousarray(g)) for pair in r["grads"] for g in pair]
    for g in grads:
        tdist.all_reduce(g, op=tdist.ReduceOp.SUM)
        g /= world
    full = O.mlp_train_step(params, x, labels, NoOpt())
    ref = [g for pair in full["grads"] for g in pair]
    err = max(float(np.max(np.abs(g.numpy() - rf)) / max(np.max(np.abs(rf)), 1e-30))
              for g, rf in zip(grads, ref))
    outq.put((rank, uid, (lo, hi), err))
    tdist.barrier()
    tdist.destroy_process_group()


def test_gloo_world2_uid_exchange_shards_and_dp_semantics():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, uid0, sh0, e0), (r1, uid1, sh1, e1) = res
    assert uid0 == uid1 == bytes(range(128))
    assert sh0 == (0, 16) and sh1 == (16, 32)
    assert e0 <= 1e-5 and e1 <= 1e-5


def test_shard_rows_requires_equal_shards():
    from paper_2602_00125_b200 import dist

    assert dist.shard_rows(65536, 3, 8) == (24576, 32768)
    with pytest.raises(ValueError):
        dist.shard_rows(10, 0, 3)


# ------------------------------------------------------- GradReducer over gloo
# The overlapped gradient exchange (dist.GradReducer driven by the autograd
# engine's leaf-ready hook) with its device plumbing replaced by a gloo
# communicator over host arrays: which gradients are averaged, in which order,
# in place or as a private copy, and what the optimizer sees.


class _HostBuf:
    """Host storage standing in for a device Buffer (version-counted)."""

    def __init__(self, arr):
        self.arr = np.ascontiguousarray(arr, np.float32)
        self.nbytes = self.arr.nbytes
        self.version = 0


def _ht(arr, grad=False):
    from paper_2602_00125_b200 import core as C

    a = np.ascontiguousarray(arr, np.float32)
    return C.Tensor(_HostBuf(a), a.shape, requires_grad=grad)


def _arr(t):
    return t.buffer.arr.reshape(t.shape)


class _GlooComm:
    """dist.Communicator's interface over torch.distributed gloo."""

    def __init__(self, world):
        self.active = world > 1
        self.world = world
        self.log = []

    def allreduce_(self, t, op=1, stream=None):
        self.log.append(("allreduce", id(t.buffer)))
        g = torch.from_numpy(t.buffer.arr)
        tdist.all_reduce(g, op=tdist.ReduceOp.SUM)
        if op == 1:
            g /= self.world
        return t

    def side_stream(self):
        return None

    def after_compute(self, stream):
        return None

    def join(self, stream):
        self.log.append(("join",))

    def private_copy(self, t):
        self.log.append(("copy", id(t.buffer)))
        return _ht(_arr(t).copy())

    def wait(self, timeout_s):
        pass


def _host_model_step(x, params, on_leaf_ready):
    """loss = mean((relu-free) (x W1^T + B) W2^T)^2 recorded on the tape with
    host pullbacks. B has h's shape, so the add's pullback hands the SAME
    cotangent to B (a leaf: ready at the add) and to h (still to be consumed
    by the first matmul) -- the aliasing case the reducer must copy."""
    from paper_2602_00125_b200 import autograd as A

    W1, B, W2 = params
    xa = np.asarray(x, np.float32)

    def mm(a, w):  # a . w^T
        out = _ht(_arr(a) @ _arr(w).T)
        return A.record("mm", (a, w), out,
                        (lambda g: _ht(_arr(g) @ _arr(w)), lambda g: _ht(_arr(g).T @ _arr(a))))

    def add(a, b):
        out = _ht(_arr(a) + _arr(b))
        return A.record("add", (a, b), out, (lambda g: g, lambda g: g))

    def mean_sq(z):
        v = _arr(z)
        out = _ht(np.array([np.mean(v.astype(np.float64) ** 2)], np.float32))
        return A.record("mean_sq", (z,), out,
                        (lambda g: _ht(_arr(g)[0] * 2.0 * v / v.size),))

    A.reset_tape()
    h = mm(_ht(xa), W1)
    h2 = add(h, B)
    loss = mean_sq(mm(h2, W2))
    return A.backward(loss, seed=_ht(np.ones(1, np.float32)), on_leaf_ready=on_leaf_ready)


def _reducer_worker(rank, world, port, outq):
    import datetime
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2602_00125_b200 import dist

    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                             world_size=world, timeout=datetime.timedelta(seconds=120))
    rng = np.random.default_rng(1)
    Bt, D, H, O = 8, 6, 5, 3
    x = rng.standard_normal((Bt, D)).astype(np.float32)
    w1 = rng.standard_normal((H, D)).astype(np.float32) * 0.3
    w2 = rng.standard_normal((O, H)).astype(np.float32) * 0.3
    bfull = rng.standard_normal((Bt, H)).astype(np.float32) * 0.1
    lo, hi = dist.shard_rows(Bt, rank, world)

    class RecOpt:  # records what the overlapped update would read
        def __init__(self):
            self.seen = []

        def prepare(self, pairs):
            return [(p, g) for p, g in pairs]

        def launch(self, handle, stream=None):
            for p, g in handle:
                self.seen.append((p.node.id, _arr(g).copy()))

    params = [_ht(w1, True), _ht(bfull[lo:hi], True), _ht(w2, True)]
    comm = _GlooComm(world)
    opt = RecOpt()
    red = dist.GradReducer(comm, params, optimizer=opt, shard=False)
    by_buf = {}

    def hook(nid, g):  # the reducer's hook, noting which leaf each averaged buffer belongs to
        out = red.hook(nid, g)
        by_buf[id(out.buffer)] = nid
        return out

    store = _host_model_step(x[lo:hi], params, hook)
    red.finish()
    got = {name: _arr(store[p]).copy() for name, p in zip(("W1", "B", "W2"), params)}
    order = [by_buf.get(e[1]) for e in comm.log if e[0] == "allreduce"]
    ids = [p.node.id for p in params]
    copies = sum(1 for e in comm.log if e[0] == "copy")
    seen = {nid: g for nid, g in opt.seen}
    # single-process full-batch reference (no reducer)
    fparams = [_ht(w1, True), _ht(bfull, True), _ht(w2, True)]
    fstore = _host_model_step(x, fparams, None)
    full = {name: _arr(fstore[p]).copy() for name, p in zip(("W1", "B", "W2"), fparams)}
    outq.put((rank, got, full, order, ids, copies, {k: v for k, v in seen.items()},
              [e[0] for e in comm.log][-1]))
    tdist.barrier()
    tdist.destroy_process_group()


def test_gloo_world2_grad_reducer_hook_order_aliasing_and_averages():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_reducer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got, full, order, ids, copies, seen, last in res:
        w1_id, b_id, w2_id = ids
        # leaf-ready order = reverse layer order: W2 (last matmul), B (add), W1
        assert order == [w2_id, b_id, w1_id], order
        assert copies == 1  # only B's gradient aliases a pending cotangent
        assert last == "join"
        # W's are data-parallel gradients: mean of shard means == full batch
        # (only if B's aliased cotangent was NOT averaged in place)
        for name in ("W1", "W2"):
            np.testing.assert_allclose(got[name], full[name], rtol=1e-5, atol=1e-7)
        # the optimizer read exactly the averaged gradients the store holds
        for nid, name in ((w1_id, "W1"), (b_id, "B"), (w2_id, "W2")):
            np.testing.assert_array_equal(seen[nid], got[name])
    # B is per-row: its averaged gradient is the mean of the two ranks' shard
    # gradients, each of which is world x the full-batch one on its rows
    (_, g0, f0, *_), (_, g1, *_) = res
    np.testing.assert_allclose(g0["B"], f0["B"][:4] + f0["B"][4:], rtol=1e-5, atol=1e-7)
    np.testing.assert_array_equal(g0["B"], g1["B"])


# ------------------------------------------------- sharded update over gloo


class _ShardComm(_GlooComm):
    """_GlooComm plus the sharded-update plumbing (reduce-scatter emulated by
    an all-reduce + slice: gloo has no reduce-scatter)."""

    def __init__(self, world, rank):
        super().__init__(world)

        class _E:
            pass

        self.env = _E()
        self.env.rank = rank
        self._views = {}

    def shard_view(self, p):
        from paper_2602_00125_b200 import core as C

        cnt = p.size // self.world
        return self._views.setdefault(id(p), C.Tensor(p.buffer, (cnt,), offset=p.offset + self.env.rank * cnt))

    def new_shard(self, cnt):
        return _ht(np.zeros(cnt, np.float32))

    def reduce_scatter_(self, send, recv, op=1, stream=None):
        self.log.append(("reduce_scatter", recv.size))
        full = torch.from_numpy(np.array(_flat(send)))
        tdist.all_reduce(full, op=tdist.ReduceOp.SUM)
        if op == 1:
            full /= self.world
        r, n = self.env.rank, recv.size
        recv.buffer.arr.reshape(-1)[recv.offset:recv.offset + n] = full.numpy()[r * n:(r + 1) * n]
        return recv

    def all_gather_(self, t, cnt, stream=None):
        self.log.append(("all_gather", cnt))
        mine = torch.from_numpy(np.array(_flat(t)[self.env.rank * cnt:(self.env.rank + 1) * cnt]))
        parts = [torch.zeros_like(mine) for _ in range(self.world)]
        tdist.all_gather(parts, mine)
        t.buffer.arr.reshape(-1)[t.offset:t.offset + t.size] = torch.cat(parts).numpy()
        return t


def _flat(t):
    return t.buffer.arr.reshape(-1)[t.offset:t.offset + t.size]


class _HostSGD:
    """The optimizer interface GradReducer drives, over host views."""

    def __init__(self, lr):
        self.lr = lr
        self.seen = []

    def prepare(self, pairs):
        return list(pairs)

    def launch(self, handle, stream=None):
        for p, g in handle:
            self.seen.append(p.size)
            _flat(p)[:] = _flat(p) - np.float32(self.lr) * _flat(g)


def _shard_worker(rank, world, port, outq):
    import datetime
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from paper_2602_00125_b200 import dist

    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                             world_size=world, timeout=datetime.timedelta(seconds=120))
    rng = np.random.default_rng(5)
    Bt, D, H, O = 8, 6, 4, 2                      # W1: 24 elements, W2: 8 (both split in 2)
    x = rng.standard_normal((Bt, D)).astype(np.float32)
    w1 = rng.standard_normal((H, D)).astype(np.float32) * 0.3
    w2 = rng.standard_normal((O, H)).astype(np.float32) * 0.3
    bfull = rng.standard_normal((Bt, H)).astype(np.float32) * 0.1
    lo, hi = dist.shard_rows(Bt, rank, world)
    # data parallel: every parameter is replicated (B too: the same rows on both ranks)
    init = {"W1": w1.copy(), "W2": w2.copy(), "B": bfull[:hi - lo].copy()}
    params = [_ht(w1.copy(), True), _ht(bfull[:hi - lo].copy(), True), _ht(w2.copy(), True)]
    comm = _ShardComm(world, rank)
    opt = _HostSGD(0.5)
    red = dist.GradReducer(comm, params, optimizer=opt, shard=True)
    assert red.shard
    store = _host_model_step(x[lo:hi], params, red.hook)
    red.finish()
    local = {n: _arr(store[p]).copy() for n, p in zip(("W1", "B", "W2"), params)}
    avg = {}
    for n, g in local.items():
        t = torch.from_numpy(g.copy())
        tdist.all_reduce(t)
        avg[n] = (t / world).numpy()
    outq.put((rank, {n: _arr(p).copy() for n, p in zip(("W1", "B", "W2"), params)}, avg,
              sorted(opt.seen), [e[0] for e in comm.log], init))
    tdist.barrier()
    tdist.destroy_process_group()


def test_gloo_world2_sharded_update_equals_the_full_update_on_every_rank():
    """reduce-scatter -> update of the rank's half -> all-gather: every rank
    ends with the parameters a full update with the averaged gradient gives,
    while its optimizer only ever touched half of each parameter."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=180) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, params, avg, seen, log, init in res:
        assert seen == [4, 8, 12]  # half of W2 (8 elements), of this rank's B rows (16), of W1 (24)
        assert log.count("reduce_scatter") == 3 and log.count("all_gather") == 3
        for n in ("W1", "W2", "B"):
            want = init[n] - np.float32(0.5) * avg[n]
            np.testing.assert_allclose(params[n], want, rtol=1e-6, atol=1e-7)
    np.testing.assert_array_equal(res[0][1]["W1"], res[1][1]["W1"])
