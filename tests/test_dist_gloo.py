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
