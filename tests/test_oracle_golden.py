"""Pin the NumPy oracle to golden vectors produced by running the reference.

CPU-only. If any of these fail the oracle no longer restates tensorlite and
every device parity test built on it is void.
"""

import numpy as np
import pytest

from oracle import tensorlite_np as O
from tests.golden import inputs as I
from tests.golden.load import bits_equal, load


def test_broadcast_binary_bit_exact():
    g = load("elementwise.npz")
    n = 0
    for i, (kind, va, vb) in enumerate(I.broadcast_cases()):
        assert bits_equal(g[f"bc{i}_{kind}_a"], va)
        got = O.binary(kind, va, vb)
        assert bits_equal(got, g[f"bc{i}_{kind}_out"]), (i, kind)
        n += 1
    assert n == 60


@pytest.mark.parametrize("name", ["neg", "exp", "log", "sqrt", "absolute", "relu"])
def test_unary_bit_exact(name):
    g = load("elementwise.npz")
    fn = getattr(O, name)
    assert bits_equal(fn(g["unary_x"]), g[f"unary_{name}"])


def test_relu_grad_mask():
    g = load("elementwise.npz")
    assert bits_equal(O.relu_mask(g["unary_x"]), g["unary_relu_grad"])


def test_div_specials():
    g = load("elementwise.npz")
    assert bits_equal(O.div(g["div_special_num"], g["div_special_den"]), g["div_special_out"])


def test_reductions_bit_exact():
    g = load("reductions.npz")
    for i, (x, axes, keep) in enumerate(I.reduction_cases()):
        assert bits_equal(g[f"r{i}_x"], x)
        assert bits_equal(O.axis_sum(x, axes, keep), g[f"r{i}_sum"]), (i, "sum")
        assert bits_equal(O.axis_mean(x, axes, keep), g[f"r{i}_mean"]), (i, "mean")
        v, pos = O.axis_max(x, axes, keep)
        assert bits_equal(v, g[f"r{i}_max"]), (i, "max")
        grad = O.max_pullback(np.ones(v.shape, np.float32), pos, x.shape)
        assert bits_equal(grad, g[f"r{i}_maxgrad"]), (i, "maxgrad")


def test_chunked_sum():
    g = load("reductions.npz")
    assert bits_equal(O.axis_sum(g["chunked_x"]), g["chunked_sum"])


def test_matmul_and_grads_bit_exact():
    g = load("matmul.npz")
    for i, (x, w, gr) in enumerate(I.matmul_cases()):
        assert bits_equal(O.matmul_xwt(x, w), g[f"m{i}_y"]), i
        dx, dw = O.matmul_grads(gr, x, w)
        assert bits_equal(dx, g[f"m{i}_dx"]), i
        assert bits_equal(dw, g[f"m{i}_dw"]), i


def test_cross_entropy_bit_exact():
    g = load("ce_optim.npz")
    for i, (z, labels) in enumerate(I.ce_cases()):
        loss, _, grad = O.cross_entropy(z, labels)
        assert bits_equal(loss, g[f"ce{i}_loss"]), i
        assert bits_equal(grad, g[f"ce{i}_grad"]), i


@pytest.mark.parametrize("name,ctor", [
    ("sgd", lambda: O.SGD(lr=0.01)),
    ("sgd_mom_wd", lambda: O.SGD(lr=0.05, momentum=0.9, weight_decay=0.01)),
    ("adam", lambda: O.Adam(lr=1e-3)),
    ("adam_wd", lambda: O.Adam(lr=3e-3, betas=(0.8, 0.99), eps=1e-6, weight_decay=0.1)),
])
def test_optimizer_sequences_bit_exact(name, ctor):
    g = load("ce_optim.npz")
    opt = ctor()
    th = g["opt_theta0"]
    for k in range(4):
        th = opt.step("p", th, g["opt_grads"][k])
        assert bits_equal(th, g[f"opt_{name}"][k]), (name, k)


def _check_mlp(golden, params, x, labels, opt, steps):
    p = [tuple(t) for t in params]
    keys = [f"k{j}" for j in range(2 * len(p))]
    losses = []
    for _ in range(steps):
        r = O.mlp_train_step(p, x, labels, opt, keys=keys)
        losses.append(r["loss"])
        p = r["params"]
    assert bits_equal(np.array(losses, np.float32), golden["loss"])
    for i, ((gw, gb), (w, b)) in enumerate(zip(r["grads"], p)):
        assert bits_equal(gw, golden[f"gw{i}"]), i
        assert bits_equal(gb, golden[f"gb{i}"]), i
        assert bits_equal(w, golden[f"w{i}"]), i
        assert bits_equal(b, golden[f"b{i}"]), i


def test_config1_full_step_bit_exact():
    params, x, labels = I.config1_inputs()
    _check_mlp(load("config1.npz"), params, x, labels, O.SGD(lr=0.01), 1)


def test_config5_small_adam_bit_exact():
    params, x, labels = I.config5_inputs(width=64, classes=10, batch=32, depth=4)
    _check_mlp(load("config5_small.npz"), params, x, labels, O.Adam(lr=1e-3), 3)


def test_config2_small_bit_exact():
    g = load("config2_small.npz")
    a, b = I.config2_inputs(rows=256, cols=512)
    r = O.broadcast_reduce_config(a, b)
    for k in ("y", "e", "sum0", "sum1", "mean0", "mean1", "max0", "max1",
              "sum_all", "grad_a", "grad_b"):
        assert bits_equal(r[k], g[k]), k


def test_config3_small_bit_exact():
    g = load("config3_small.npz")
    A, B, dC = I.config3_inputs(n=96)
    C, dA, dB = O.matmul_fwd_bwd(A, B, dC)
    assert bits_equal(C, g["C"]) and bits_equal(dA, g["dA"]) and bits_equal(dB, g["dB"])


def test_config4_small_bit_exact():
    g = load("config4_small.npz")
    X, W, bias, T = I.config4_inputs(b=2, s=16, k=64)
    r = O.softmax_linear_config(X, W, bias, T)
    assert bits_equal(r["loss"], g["loss"])
    assert bits_equal(r["Y"].reshape(-1, 64), g["Y"])
    assert bits_equal(r["dX"].reshape(-1, 64), g["dX"])
    assert bits_equal(r["dW"], g["dW"])
    assert bits_equal(r["dbias"], g["dbias"])


# ---------------------------------------------------------------- SURVEY 8f rows


@pytest.mark.parametrize("name", ["sigmoid", "tanh", "gelu"])
def test_activations_and_grads_bit_exact(name):
    g = load("next_rows.npz")
    x, gy = g["act_x"], g["act_g"]
    y = getattr(O, name)(x)
    assert bits_equal(y, g[f"act_{name}"])
    assert bits_equal(O.activation_grad(name, gy, x, y), g[f"act_{name}_grad"])


@pytest.mark.parametrize("name,ctor", [
    ("rmsprop", lambda: O.RMSprop(lr=0.01)),
    ("rmsprop_wd", lambda: O.RMSprop(lr=3e-3, rho=0.9, eps=1e-6, weight_decay=0.05)),
])
def test_rmsprop_sequences_bit_exact(name, ctor):
    g = load("next_rows.npz")
    opt = ctor()
    th = g["opt_theta0"]
    for k in range(4):
        th = opt.step("p", th, g["opt_grads"][k])
        assert bits_equal(th, g[f"opt_{name}"][k]), (name, k)


def test_demo_logs_have_the_reference_format():
    """The demos' `epoch,loss[,acc]` log contract (demos.py:59, 116)."""
    g = load("next_rows.npz")
    xor, blobs = list(g["xor_lines"]), list(g["blobs_lines"])
    assert len(xor) == 301 and xor[0].startswith("0,") and xor[-1].startswith("final,")
    assert all(len(l.split(",")) == 3 for l in blobs)
    assert blobs[-1].startswith("final,")


# ---------------------------------------------------------------- catalog


def test_conv2d_oracle_against_reference():
    g = load("catalog.npz")
    for i, (b, cin, h, w, cout, k, s, p, bias) in enumerate(I.CONV_CASES):
        bv = g[f"conv{i}_b"] if bias else None
        y, pull = O.conv2d(g[f"conv{i}_x"], g[f"conv{i}_w"], bv, s, p)
        assert bits_equal(y, g[f"conv{i}_y"]), i
        dx, dw, db = pull(g[f"conv{i}_g"])
        assert bits_equal(dx, g[f"conv{i}_dx"]), i
        assert bits_equal(dw, g[f"conv{i}_dw"]), i
        if bias:
            assert bits_equal(db, g[f"conv{i}_db"]), i
