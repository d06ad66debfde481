"""The tlnp host surface on the device (mirrors the reference's
bindings/tests/test_api.py: handles vs the direct engine, bit-exact)."""

from random import Random

import numpy as np
import pytest

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import tlnp
from oracle import tensorlite_np as O
from tests.golden.load import bits_equal, normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def fresh_state():
    tlnp.reset_tape()
    tlnp.clear_grads()
    yield
    tlnp.reset_tape()


def _vals(rng, n):
    return [rng.choice([-2.5, -1.0, -0.5, 0.0, 0.25, 1.0, 3.0]) * rng.random() for _ in range(n)]


def test_hundred_random_ops_match_oracle():
    rng = Random(1234)
    unary = ["neg", "exp", "log", "sqrt", "abs", "sum", "mean", "max", "reshape", "transpose"]
    binary = ["add", "sub", "mul", "div", "matmul"]
    for _ in range(100):
        kind = rng.choice(binary + unary)
        m, n = rng.randint(1, 4), rng.randint(1, 4)
        vals = _vals(rng, m * n)
        if kind in ("log", "sqrt"):
            vals = [abs(v) + 0.5 for v in vals]
        xa = np.array(vals, np.float32).reshape(m, n)
        hx = tlnp.tensor(xa)
        if kind == "matmul":
            d = rng.randint(1, 4)
            wa = np.array(_vals(rng, d * n), np.float32).reshape(d, n)
            got = (hx @ tlnp.tensor(wa)).numpy()
            assert normwise(got, O.matmul_xwt(xa, wa)) <= 1e-6
            continue
        if kind in binary:
            sb = rng.choice([(m, n), (1, n), (m, 1), (1, 1)])
            ba = np.array(_vals(rng, sb[0] * sb[1]), np.float32).reshape(sb)
            if kind == "div":
                ba[ba == 0] = 1.0
            op = {"add": "__add__", "sub": "__sub__", "mul": "__mul__", "div": "__truediv__"}[kind]
            got = getattr(hx, op)(tlnp.tensor(ba)).numpy()
            want = O.binary(kind, xa, ba)
        elif kind == "neg":
            got, want = (-hx).numpy(), O.neg(xa)
        elif kind == "abs":
            got, want = abs(hx).numpy(), O.absolute(xa)
        elif kind in ("exp", "log", "sqrt"):
            got, want = getattr(hx, kind)().numpy(), getattr(O, kind)(xa)
        elif kind in ("sum", "mean", "max"):
            axis = rng.choice([None, 0, 1])
            keep = rng.random() < 0.5
            got = getattr(hx, kind)(axis=axis, keepdims=keep).numpy()
            fn = {"sum": O.axis_sum, "mean": O.axis_mean, "max": lambda *a: O.axis_max(*a)[0]}[kind]
            want = fn(xa, axis, keep)
        elif kind == "reshape":
            got, want = hx.reshape(n, m).numpy(), xa.reshape(n, m)
        else:
            got, want = hx.T.numpy(), xa.T
        assert bits_equal(got, want), kind


def test_backward_chain_matches_engine_bit_exact():
    vals = [0.5, -1.5, 2.0, 3.0, -0.25, 1.0]
    x = tlnp.tensor(np.array(vals, np.float32).reshape(2, 3), requires_grad=True)
    w = tlnp.tensor(np.array(vals[::-1], np.float32).reshape(2, 3))
    loss = ((x @ w).exp().sum() / 7.0)
    loss.backward()
    got = x.grad.numpy()
    P.reset_tape()
    ex = P.from_numpy(np.array(vals, np.float32).reshape(2, 3), requires_grad=True)
    ew = P.from_numpy(np.array(vals[::-1], np.float32).reshape(2, 3))
    store = P.backward(P.div(P.sum(P.exp(P.matmul(ex, ew))), 7.0))
    assert bits_equal(got, store[ex].numpy())


def test_grad_lifecycle_and_zero_grad():
    x = tlnp.tensor([1.0, 2.0], requires_grad=True)
    assert x.grad is None
    (x * x).sum().backward()
    assert x.grad.tolist() == [2.0, 4.0]
    tlnp.reset_tape()
    assert x.grad is not None  # survives until x joins a new graph (test_api.py:39-46)
    opt = tlnp.SGD([x], lr=0.1)
    opt.zero_grad()
    assert x.grad is None


def test_operators_scalars_comparisons_and_errors():
    t = tlnp.tensor([1.0, 2.0])
    assert (1.0 + t).tolist() == [2.0, 3.0]
    assert (3 - t).tolist() == [2.0, 1.0]
    assert (2.0 / t).tolist() == [2.0, 1.0]
    with pytest.raises(TypeError):
        t + "a"
    s = tlnp.tensor(3.0)
    assert s > 2 and s == 3.0 and float(s) == 3.0
    with pytest.raises(TypeError):
        t < 1
    with pytest.raises(tlnp.ShapeError, match="inner dimensions differ"):
        tlnp.ones((2, 3)) @ tlnp.ones((2, 4))
    with pytest.raises(tlnp.BroadcastError):
        tlnp.ones((2,)) + tlnp.ones((3,))
    with pytest.raises(TypeError):
        tlnp.wrap_host_array(np.ones(3, np.float64))
    assert tlnp.wrap_host_array(np.ones(3, np.float64), allow_copy=True).copied


def test_pytorch_spellings():
    x = tlnp.tensor(np.arange(6, dtype=np.float32).reshape(2, 3) - 2.0)
    assert x.sum(dim=1).tolist() == x.sum(axis=1).tolist()
    assert x.max(dim=0, keepdim=True).shape == (1, 3)
    assert x.relu().tolist() == [[0.0, 0.0, 0.0], [1.0, 2.0, 3.0]]
    lin = tlnp.Linear(3, 4, rng=0)
    assert lin(x).shape == (2, 4)
    b = tlnp.tensor(np.ones((3, 5), np.float32))
    assert x.mm(b).shape == (2, 5)


def test_dense_same_seed_same_weights_as_reference_stream():
    d = tlnp.Dense(5, 3, rng=42)
    import math
    import random

    r = random.Random(42)
    bound = 1.0 / math.sqrt(5)
    w = np.array([r.uniform(-bound, bound) for _ in range(15)], np.float32).reshape(3, 5)
    b = np.array([r.uniform(-bound, bound) for _ in range(3)], np.float32)
    assert bits_equal(d.weight.numpy(), w) and bits_equal(d.bias.numpy(), b)


def test_optimizer_step_through_bindings_matches_engine():
    rng = np.random.default_rng(3)
    p0 = rng.standard_normal((4, 3)).astype(np.float32)
    xs = rng.standard_normal((5, 3)).astype(np.float32)
    hp = tlnp.tensor(p0, requires_grad=True)
    opt = tlnp.Adam([hp], lr=0.01)
    for _ in range(3):
        tlnp.reset_tape()
        ((tlnp.tensor(xs) @ hp) * 2.0).sum().backward()
        assert opt.step() == 1
    ep = P.from_numpy(p0, requires_grad=True)
    eopt = P.optim.Adam(lr=0.01)
    for _ in range(3):
        P.reset_tape()
        store = P.backward(P.sum(P.mul(P.matmul(P.from_numpy(xs), ep), 2.0)))
        P.optim.step_all(eopt, [ep], store)
    assert bits_equal(hp.numpy(), ep.numpy())


def test_mlp_training_through_bindings_descends():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((64, 8)).astype(np.float32)
    labels = (x[:, 0] > 0).astype(np.int64)
    model = tlnp.Sequential(tlnp.Linear(8, 16, rng=1), tlnp.ReLU(), tlnp.Linear(16, 2, rng=2))
    opt = tlnp.Adam(model.parameters(), lr=0.05)
    losses = []
    for _ in range(30):
        tlnp.reset_tape()
        loss = tlnp.cross_entropy(model(tlnp.tensor(x)), labels)
        losses.append(loss.item())
        loss.backward()
        opt.step()
    assert losses[-1] < 0.5 * losses[0]


def test_grad_store_is_per_thread():
    """backward() keeps its gradient store per host thread (next to the
    engine's per-thread tape and stream): a thread's .grad never reads another
    thread's backward, and clear_grads() only forgets the caller's."""
    import threading

    seen = {}

    def worker(tag, scale):
        tlnp.reset_tape()
        w = tlnp.tensor([1.0, 2.0, 3.0], requires_grad=True)
        (w * scale).sum().backward()
        seen[tag] = w.grad.numpy().tolist()
        tlnp.reset_tape()

    w0 = tlnp.tensor([4.0, 5.0], requires_grad=True)
    (w0 * 7.0).sum().backward()
    ts = [threading.Thread(target=worker, args=(i, float(i + 2))) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert seen == {0: [2.0, 2.0, 2.0], 1: [3.0, 3.0, 3.0]}
    assert w0.grad.numpy().tolist() == [7.0, 7.0]  # untouched by the workers' backward()
    tlnp.clear_grads()
    assert w0.grad is None
