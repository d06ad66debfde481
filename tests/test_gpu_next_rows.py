"""Device parity for the SURVEY 8f rows: pointwise activations and their
pullbacks (nn.py:95-144), multi-tensor RMSprop (optim.py:103-122), and the
reference's training callers with their log contract (demos.py:42-130) --
against goldens produced by running the reference (tests/golden/next_rows.npz)."""

import numpy as np
import pytest

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import demos, optim
from tests.golden.load import bits_equal, load, normwise

pytestmark = pytest.mark.gpu


def dev(a, grad=False):
    return P.from_numpy(np.asarray(a, np.float32), requires_grad=grad)


@pytest.mark.parametrize("name", ["sigmoid", "tanh", "gelu"])
def test_activations_and_pullbacks_bit_exact(name):
    g = load("next_rows.npz")
    P.reset_tape()
    x = dev(g["act_x"], True)
    y = getattr(P, name)(x)
    assert bits_equal(y.numpy(), g[f"act_{name}"])
    store = P.backward(y, seed=dev(g["act_g"]))
    assert bits_equal(store[x].numpy(), g[f"act_{name}_grad"])


@pytest.mark.parametrize("name,ctor", [
    ("rmsprop", lambda: optim.RMSprop(lr=0.01)),
    ("rmsprop_wd", lambda: optim.RMSprop(lr=3e-3, rho=0.9, eps=1e-6, weight_decay=0.05)),
])
def test_rmsprop_multi_tensor_bit_exact(name, ctor):
    g = load("next_rows.npz")
    opt = ctor()
    p = dev(g["opt_theta0"])
    for k in range(4):
        opt.step(p, dev(g["opt_grads"][k]))
        assert bits_equal(p.numpy(), g[f"opt_{name}"][k]), (name, k)


def _parse(lines):
    rows = [l.split(",") for l in lines]
    return [r[0] for r in rows], np.array([[float(v) for v in r[1:]] for r in rows])


@pytest.mark.parametrize("key,run", [
    ("xor_lines", lambda: demos.run_xor(seed=0, epochs=300)),
    ("blobs_lines", lambda: demos.run_blobs(seed=0, epochs=60)),
    ("blobs_rms_lines", lambda: demos.run_blobs(seed=3, epochs=30, lr=0.01, optimizer="rmsprop")),
])
def test_demo_training_logs_match_reference(key, run):
    """Same seeds, init streams and log format; losses within the fp32
    tolerance (GEMMs accumulate in fp32, the reference in double), accuracies
    equal up to one sample."""
    want_ep, want = _parse(load("next_rows.npz")[key])
    res = run()
    got_ep, got = _parse(res.lines)
    assert got_ep == want_ep
    assert res.diverged_at is None
    assert normwise(got[:, 0], want[:, 0]) <= 1e-4
    if want.shape[1] > 1:
        assert np.max(np.abs(got[:, 1] - want[:, 1])) <= 1.0 / 200 + 1e-12


def test_gradcheck_suite_on_device():
    """the reference's finite-difference suite
    (gradcheck.py:317-344) over the device ops; both sides run on the B200."""
    from paper_2602_00125_b200 import gradcheck

    ok, text = gradcheck.run_suite(seeds=(0, 1, 2))
    assert ok, text
    assert text.splitlines()[-1] == "OVERALL PASS"
    assert text.count("== ") == len(gradcheck.STANDARD_CHECKS)


def test_gradcheck_catches_a_wrong_pullback():
    from paper_2602_00125_b200 import gradcheck
    from paper_2602_00125_b200.autograd import record

    def bad_square(x):  # value x*x, pullback claims 3x
        out = P.mul(x, x).detach()
        return record("bad_square", (x,), out, (lambda g: P.mul(g, P.mul(x, 3.0)),))

    x = P.uniform((3, 4), -1, 1, rng=0, requires_grad=True)
    c = P.uniform((3, 4), -1, 1, rng=1)
    rep = gradcheck.check_function(lambda: P.sum(P.mul(bad_square(x), c)), {"x": x})
    assert not rep.passed


def test_dlpack_zero_copy_exchange_with_torch():
    """device-side zero-copy exchange (the HBM analogue of
    the reference's aliasing wrap_host_array / to_host_array)."""
    torch = pytest.importorskip("torch")
    base = np.arange(12, dtype=np.float32).reshape(3, 4)
    x = P.from_numpy(base)
    tx = torch.from_dlpack(x)
    assert tx.device.type == "cuda" and tuple(tx.shape) == (3, 4)
    assert tx.data_ptr() == x.data_ptr
    assert bits_equal(tx.cpu().numpy(), base)
    tx.mul_(2.0)  # torch writes, the engine sees them
    torch.cuda.synchronize()
    assert bits_equal(x.numpy(), 2 * base)
    tv = torch.from_dlpack(P.transpose2d(x))  # strided view: no copy, strides kept
    assert tuple(tv.stride()) == (1, 4) and bits_equal(tv.cpu().numpy(), 2 * base.T)

    t = torch.randn(64, 48, device="cuda")
    e = P.from_dlpack(t)  # engine ops on torch's memory
    assert e.data_ptr == t.data_ptr() and e.shape == (64, 48)
    from oracle import tensorlite_np as O

    host = t.cpu().numpy()
    assert bits_equal(P.sum(e, axis=0).numpy(), O.axis_sum(host, 0))
    assert bits_equal(P.exp(P.transpose2d(e)).numpy(), O.exp(host.T))
    e.fill_(1.0)  # engine writes, torch sees them
    L_sync = P.ones((1,)).numpy()  # noqa: F841 (orders the engine stream)
    assert float(t.sum().item()) == 64 * 48
    del e
    import gc

    gc.collect()
    assert float(t.sum().item()) == 64 * 48  # torch's storage outlives the engine view


def test_tlnp_dlpack_roundtrip():
    torch = pytest.importorskip("torch")
    from paper_2602_00125_b200 import tlnp

    t = torch.arange(6, dtype=torch.float32, device="cuda").reshape(2, 3)
    h = tlnp.from_dlpack(t)
    y = (h * 2.0).relu()
    back = torch.from_dlpack(y)
    assert torch.equal(back, t * 2.0)


# ---------------------------------------------------------------- catalog


@pytest.mark.parametrize("i", range(5))
def test_conv2d_against_reference(i):
    """im2col -> GEMM engine -> permute; col2im in the reference's order.
    Same seeded init as the reference's Conv2D; GEMM tolerance 1e-4
    normwise (the patch GEMMs accumulate in fp32), db bit-exact."""
    from paper_2602_00125_b200 import nn
    from tests.golden import inputs as I

    g = load("catalog.npz")
    b, cin, h, w, cout, k, s, p, bias = I.CONV_CASES[i]
    layer = nn.Conv2D(cin, cout, k, stride=s, padding=p, bias=bias, rng=100 + i)
    assert bits_equal(layer.weight.numpy(), g[f"conv{i}_w"])  # same init stream
    P.reset_tape()
    x = dev(g[f"conv{i}_x"], True)
    y = layer(x)
    assert y.shape == g[f"conv{i}_y"].shape
    assert normwise(y.numpy(), g[f"conv{i}_y"]) <= 1e-4
    store = P.backward(y, seed=dev(g[f"conv{i}_g"]))
    assert normwise(store[x].numpy(), g[f"conv{i}_dx"]) <= 1e-4
    assert normwise(store[layer.weight].numpy(), g[f"conv{i}_dw"]) <= 1e-4
    if bias:
        assert bits_equal(store[layer.bias].numpy(), g[f"conv{i}_db"])


def test_batchnorm_train_eval_bit_exact():
    """Composed from the device ops in the reference's order: outputs,
    gradients and running buffers bit-exact over two train steps + eval."""
    from paper_2602_00125_b200 import nn

    g = load("catalog.npz")
    bn = nn.BatchNorm(6, eps=1e-5, momentum=0.1)
    for k in range(2):
        P.reset_tape()
        x = dev(g[f"bn{k}_x"], True)
        y = bn(x)
        store = P.backward(y, seed=dev(g[f"bn{k}_g"]))
        assert bits_equal(y.numpy(), g[f"bn{k}_y"]), k
        assert bits_equal(store[x].numpy(), g[f"bn{k}_dx"]), k
        assert bits_equal(store[bn.gamma].numpy(), g[f"bn{k}_dgamma"]), k
        assert bits_equal(store[bn.beta].numpy(), g[f"bn{k}_dbeta"]), k
        assert bits_equal(bn.running_mean.numpy(), g[f"bn{k}_rmean"]), k
        assert bits_equal(bn.running_var.numpy(), g[f"bn{k}_rvar"]), k
    bn.set_mode("eval")
    with P.no_grad():
        assert bits_equal(bn(dev(g["bn_eval_x"])).numpy(), g["bn_eval_y"])


def test_dropout_same_stream_bit_exact():
    import random

    from paper_2602_00125_b200 import nn

    g = load("catalog.npz")
    P.reset_tape()
    x = dev(g["drop_x"], True)
    y = nn.dropout(x, 0.3, "train", rng=random.Random(5))
    store = P.backward(P.sum(y))
    assert bits_equal(y.numpy(), g["drop_y"])
    assert bits_equal(store[x].numpy(), g["drop_dx"])
    assert nn.dropout(x, 0.3, "eval") is x


def test_checkpoint_resume_bit_identical(tmp_path):
    """Train 2 steps, save (params, buffers, Adam slots and step counts),
    resume in a fresh model/optimizer for 1 more step == 3 uninterrupted steps."""
    from paper_2602_00125_b200 import checkpoint, nn

    rng = np.random.default_rng(3)
    x = dev(rng.standard_normal((64, 32)).astype(np.float32))
    labels = nn.labels_buffer(rng.integers(0, 10, 64))

    def make():
        return nn.Sequential(nn.Dense(32, 48, rng=1), nn.ReLU(), nn.BatchNorm(48),
                             nn.Dense(48, 10, rng=2))

    def step(model, opt):
        P.reset_tape()
        store = P.backward(nn.cross_entropy(model(x), labels))
        optim.step_all(opt, model.parameters(), store)

    ref, ropt = make(), optim.Adam(lr=1e-2)
    for _ in range(3):
        step(ref, ropt)
    a, aopt = make(), optim.Adam(lr=1e-2)
    for _ in range(2):
        step(a, aopt)
    path = str(tmp_path / "ck.npz")
    checkpoint.save(path, a, aopt)
    b, bopt = make(), optim.Adam(lr=1e-2)
    checkpoint.load(path, b, bopt)
    step(b, bopt)
    for (n1, p1), (n2, p2) in zip(ref.named_parameters(), b.named_parameters()):
        assert n1 == n2 and bits_equal(p1.numpy(), p2.numpy()), n1
    for (n1, b1), (n2, b2) in zip(ref.named_buffers(), b.named_buffers()):
        assert n1 == n2 and bits_equal(b1.numpy(), b2.numpy()), n1


def test_comm_failure_detection_and_timeout_abort():
    """SURVEY 5 failure detection: the communicator's async error is polled;
    a comm stream that does not drain within the deadline aborts the
    communicator and raises (a dead peer fails the step instead of hanging it)."""
    from paper_2602_00125_b200 import _lib as L
    from paper_2602_00125_b200 import dist, nn

    comm = dist.Communicator(dist.Env(), force_nccl=True)
    comm.check()
    g = P.ones((1000,))
    red = dist.GradReducer(comm, timeout_s=60.0)  # timed host wait, healthy path
    red.hook(0, g)
    red.finish()
    assert bits_equal(g.numpy(), np.ones(1000, np.float32))
    n = 8192
    a = P.zeros((n, n))
    c = P.zeros((n, n))
    L.call("b2_gemm", 0, 1, n, n, n, a.data_ptr, n, a.data_ptr, n, c.data_ptr, n, None, 0,
           L.GEMM_3XBF16, comm.comm_stream)  # ~ms of work on the comm stream
    with pytest.raises(RuntimeError, match="aborted"):
        comm.wait(1e-6)
    with pytest.raises(RuntimeError):
        comm.allreduce_(P.ones((4,)))  # the aborted communicator fails loudly
    L.synchronize()
