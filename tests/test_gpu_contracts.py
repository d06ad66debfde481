"""Host-contract tests on the device: the per-thread tape AND engine stream
(pkg/tests/test_autograd.py:316-331; SURVEY 8b "one CUDA stream per (thread,
device)"), label validation / the kernel's out-of-range guard, the input
feeder's teardown, DLPack export ordering of split-only GEMM outputs, the
value-only max and the memory released by ``keep_intermediate=False``."""

import threading

import numpy as np
import pytest

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
from paper_2602_00125_b200 import autograd, nn, optim
from tests.golden import inputs as I
from tests.golden.load import bits_equal

pytestmark = pytest.mark.gpu


def dev(a, grad=False):
    return P.from_numpy(np.asarray(a, np.float32), requires_grad=grad)


def test_tapes_and_engine_streams_are_thread_local():
    x = dev([1.0], True)
    P.mul(x, x)
    main_len = len(P.tape())
    main_stream = L.default_stream()
    seen = {}

    def worker():
        y = dev([2.0], True)
        z = P.mul(y, y)
        seen["len"] = len(P.tape())  # leaf + mul on a fresh tape
        seen["stream"] = L.default_stream()
        seen["grad"] = P.backward(P.sum(z))[y].numpy().tolist()

    t = threading.Thread(target=worker)
    t.start()
    t.join()
    assert seen["len"] == 2
    assert len(P.tape()) == main_len
    assert seen["stream"] != main_stream
    assert seen["grad"] == [4.0]


def _config1_steps(params, x, labels, steps, out, key):
    layers = []
    for i, (w, b) in enumerate(params):
        d = nn.Dense(w.shape[1], w.shape[0], rng=0)
        d.weight.write_flat(w.ravel())
        d.bias.write_flat(b.ravel())
        layers.append(d)
        if i < len(params) - 1:
            layers.append(nn.ReLU())
    model = nn.Sequential(*layers)
    opt = optim.SGD(lr=0.01)
    xt = dev(x)
    losses = []
    for _ in range(steps):
        P.reset_tape()
        loss = nn.cross_entropy(model(xt), labels)
        optim.step_all(opt, model.parameters(), P.backward(loss))
        losses.append(loss.item())
    out[key] = (losses, [p.numpy() for p in model.parameters()])


def test_two_threads_train_concurrently_bit_identical_to_sequential():
    """Each thread's ops queue on its own stream with its own tape: two
    threads training their own config-1 model at the same time produce the
    bits a sequential run produces."""
    params, x, labels = I.config1_inputs()
    params2, x2, labels2 = I.config1_inputs(seed=1)
    seq = {}
    _config1_steps(params, x, labels, 3, seq, "a")
    _config1_steps(params2, x2, labels2, 3, seq, "b")
    par = {}
    ts = [threading.Thread(target=_config1_steps, args=(params, x, labels, 3, par, "a")),
          threading.Thread(target=_config1_steps, args=(params2, x2, labels2, 3, par, "b"))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for k in ("a", "b"):
        assert par[k][0] == seq[k][0], k
        for g, w in zip(par[k][1], seq[k][1]):
            assert bits_equal(g, w), k


def test_labels_buffer_validates_and_kernel_guards_unchecked_labels():
    z = dev(np.zeros((4, 10), np.float32))
    with pytest.raises(ValueError, match="out of range"):
        nn.labels_buffer([0, 1, 10, 2], classes=10)
    bad = nn.labels_buffer([0, 1, 10, -3])  # unchecked: the kernel must not read past the row
    assert np.isnan(nn.cross_entropy(z, bad).item())
    ok = nn.labels_buffer([0, 1, 9, 2], classes=10)
    assert abs(nn.cross_entropy(z, ok).item() - np.log(10.0)) < 1e-6


def test_pinned_feeder_rejects_bad_labels_and_closes_cleanly():
    from paper_2602_00125_b200.data import PinnedFeeder

    x = np.random.default_rng(0).standard_normal((64, 128)).astype(np.float32)
    with pytest.raises(ValueError, match="out of range"):
        PinnedFeeder(x, np.arange(64) % 11, classes=10)
    f = PinnedFeeder(x, np.arange(64) % 10, presplit="3xbf16", classes=10)
    xb, _ = f.next()
    assert bits_equal(xb.numpy(), x)
    f.close()
    f.close()  # idempotent
    assert f.copy_stream is None


def test_dlpack_export_of_a_split_only_output_orders_the_materialisation():
    """A hidden layer's GEMM writes only its operand split; exporting it over
    DLPack must queue the fp32 materialisation BEFORE the consumer's stream
    is ordered after the engine (the consumer reads fp32 values)."""
    torch = pytest.importorskip("torch")
    from paper_2602_00125_b200 import core as C

    rng = np.random.default_rng(3)
    x = rng.standard_normal((512, 512)).astype(np.float32)
    w = (rng.standard_normal((512, 512)) * 0.05).astype(np.float32)
    b = np.zeros(512, np.float32)
    P.set_gemm_algo("3xbf16")
    try:
        with P.no_grad():
            h = C.linear(dev(x), dev(w), dev(b), relu_out=True)
            h2 = C.linear(dev(x), dev(w), dev(b), relu_out=True)
    finally:
        P.set_gemm_algo(None)
    assert h.buffer._pending is not None  # split-only: fp32 not written yet
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        th = torch.from_dlpack(h)
        got = th.cpu().numpy()
    assert bits_equal(got, h2.numpy())


def test_keep_intermediate_false_frees_cotangents_during_backward():
    """Same gradients, and the hidden cotangents are released as soon as their
    pullback consumed them (only leaf gradients remain in the store)."""
    params, x, labels = I.config5_inputs(width=256, classes=16, batch=256, depth=3)

    def run(keep):
        model = nn.Sequential(*[m for i, (w, b) in enumerate(params) for m in (
            [nn.Dense(w.shape[1], w.shape[0], rng=0)] + ([nn.ReLU()] if i < len(params) - 1 else []))])
        dense = [m for m in model.layers if isinstance(m, nn.Dense)]
        for d, (w, b) in zip(dense, params):
            d.weight.write_flat(w.ravel())
            d.bias.write_flat(b.ravel())
        P.reset_tape()
        loss = nn.cross_entropy(model(dev(x)), labels)
        store = P.backward(loss, keep_intermediate=keep)
        return len(store), [store[p].numpy() for p in model.parameters()]

    n_keep, g_keep = run(True)
    n_drop, g_drop = run(False)
    assert n_drop == len(g_drop) and n_keep > n_drop
    for a, b in zip(g_keep, g_drop):
        assert bits_equal(a, b)


def test_backward_schedule_prunes_unreachable_nodes():
    x = dev([1.0, 2.0], True)
    y = dev([3.0, 4.0], True)
    side = P.exp(y)  # recorded, but not on the loss's path
    loss = P.sum(P.mul(x, x))
    sch = autograd.schedule(loss)
    assert side.node.id not in sch.order
    calls = P.tape().pullback_calls
    store = P.backward(loss)
    assert P.tape().pullback_calls - calls == len(sch.order) == 2
    assert store[x].numpy().tolist() == [2.0, 4.0]
    assert y not in store


def test_bench_spawn_launcher_runs_an_nccl_rank_and_prints_one_line():
    """bench.py's own N-rank launcher (used when no torchrun env is present),
    taken at N = 1 with a 1-rank NCCL communicator: the rank process gets the
    torchrun-style env, NCCL initialises (its INFO lines on stderr), rank 0
    prints exactly one JSON line with n_gpus = 1."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(B2_BENCH_SPAWN="1", B2_FORCE_NCCL="1", NCCL_DEBUG="INFO")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "1", "--steps", "2", "--warmup", "3",
                        "--no-ops", "--no-cpu", "--no-bf16", "--global-batch", "4096"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["config"]["parallelism"] == "dp1"
    assert "NCCL INFO" in r.stderr  # the launcher routes NCCL's log to stderr


def test_bench_under_torchrun_joins_the_agent_store_for_the_nccl_id():
    """The driver's N > 1 launch (python -m torch.distributed.run ... bench.py
    --gpus N) at N = 1 with a 1-rank NCCL communicator: the NCCL unique id goes
    through torchrun's own agent store (no second port), one JSON line."""
    import json
    import os
    import socket
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env.update(B2_FORCE_NCCL="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "1",
                        "--steps", "2", "--warmup", "3", "--no-ops", "--no-cpu", "--no-bf16",
                        "--global-batch", "4096"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert json.loads(lines[0])["n_gpus"] == 1


# ---------------------------------------------------------------- edge cases of the round-2 paths


@pytest.mark.parametrize("shape", [(1, 1, 1), (3, 5, 4), (33, 65, 17), (130, 70, 300), (64, 128, 0)])
@pytest.mark.parametrize("ta,tb", [(0, 1), (0, 0), (1, 0), (1, 1)])
def test_reference_arithmetic_gemm_ragged_layouts_and_empty_k(shape, ta, tb):
    """B2_GEMM_REF on ragged tiles, every layout, K = 0, with the bias+ReLU
    epilogue: f32 of the compensated double dot (here checked against a
    float64 numpy dot, equal up to 1 ulp where numpy's sum is uncompensated)."""
    M, N, K = shape
    rng = np.random.default_rng(M * 31 + N * 7 + K + ta * 2 + tb)
    A = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    a64 = A.astype(np.float64).T if ta else A.astype(np.float64)
    b64 = B.astype(np.float64) if tb else B.astype(np.float64).T
    want = np.maximum(np.float32(a64 @ b64.T) + bias, np.float32(0))
    At, Bt, bt = dev(A), dev(B), dev(bias)
    C = P.zeros((M, N))
    L.call("b2_gemm", ta, tb, M, N, K, At.data_ptr if A.size else None, A.shape[1] if A.ndim else 1,
           Bt.data_ptr if B.size else None, B.shape[1], C.data_ptr, N, bt.data_ptr, L.EPI_BIAS_RELU,
           L.GEMM_REF, None)
    got = C.numpy()
    ulp = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
    assert ulp.max(initial=0) <= 1


def test_softmax_mul_mean_fallback_and_edge_shapes():
    """Shapes the fused kernels do not take (cols % 4, cols > 1024, strided z)
    go through the composed ops; one-row and 4-column inputs use the kernels;
    every case equals the composition bit for bit."""
    rng = np.random.default_rng(21)
    for R, C in ((1, 4), (7, 1024), (5, 6), (3, 1100), (64, 36)):
        z = rng.standard_normal((R, C)).astype(np.float32) * 3
        t = rng.uniform(0, 1, (R, C)).astype(np.float32)
        P.reset_tape()
        zt = dev(z, True)
        loss = P.softmax_mul_mean(zt, dev(t))
        g = P.backward(loss)[zt].numpy()
        P.reset_tape()
        zc = dev(z, True)
        lc = P.mean(P.mul(P.softmax(zc), dev(t)))
        gc = P.backward(lc)[zc].numpy()
        assert bits_equal(loss.numpy(), lc.numpy()), (R, C)
        assert bits_equal(g, gc), (R, C)


def test_sharded_grad_reducer_falls_back_for_indivisible_parameters():
    """A parameter whose size the world does not divide keeps the all-reduce
    path (a 1-rank communicator divides everything, so this checks the rule
    on the host side: the shard predicate)."""
    from paper_2602_00125_b200 import dist

    comm = dist.Communicator(dist.Env(), force_nccl=True)
    red = dist.GradReducer(comm, [P.zeros((3,), requires_grad=True)], optimizer=optim.SGD(lr=0.1),
                           shard=True)
    assert red.shard and comm.world == 1


def test_muladd_relu_stats_single_row_and_nan_row():
    a = np.array([[np.nan, -1.0, 2.0, 0.0]], np.float32)
    b = np.array([[0.5, -2.0, 1.0, 3.0]], np.float32)
    from oracle import tensorlite_np as O

    ref = O.broadcast_reduce_config(a, b)
    out = P.muladd_relu_stats(dev(a), dev(b))
    for k in ("y", "e", "sum0", "sum1", "mean0", "mean1", "max0", "max1", "sum_all", "grad_a", "grad_b"):
        assert bits_equal(out[k].numpy(), ref[k]), k
