"""Generate golden vectors by running the REFERENCE itself (tensorlite).

Run here (the survey container), never on the GPU box:

    python tests/golden/make_golden.py

It imports the pure-Python reference read-only from
/root/reference/pkg/src, feeds it seeded NumPy inputs through its public API
(the same calls the reference's own tests make), and writes the outputs to
tests/golden/*.npz. The committed fixtures pin both the NumPy oracle
(tests/test_oracle_golden.py) and the device engine (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import os
import random
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import tensorlite as tl  # noqa: E402
from tensorlite import nn as tnn, optim as topt  # noqa: E402

from tests.golden.inputs import (  # noqa: E402
    config1_inputs, config2_inputs, config3_inputs, config4_inputs,
    config5_inputs, broadcast_cases, reduction_cases, matmul_cases,
    unary_values, ce_cases, CONV_CASES,
)


def T(arr, grad=False):
    arr = np.ascontiguousarray(arr, dtype=np.float32)
    t = tl.from_flat(arr.ravel().tolist(), arr.shape)
    t.requires_grad = grad
    return t


def A(t):
    return np.array(t.flat(), dtype=np.float32).reshape(t.shape)


def save(name, **arrs):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrs)
    print(f"wrote {name} ({os.path.getsize(path) / 1e6:.2f} MB)")


# ---------------------------------------------------------------------------


def gen_elementwise():
    out = {}
    for i, (kind, va, vb) in enumerate(broadcast_cases()):
        r = getattr(tl, kind)(T(va), T(vb))
        out[f"bc{i}_{kind}_a"] = va
        out[f"bc{i}_{kind}_b"] = vb
        out[f"bc{i}_{kind}_out"] = A(r)
    u = unary_values()
    out["unary_x"] = u
    for name in ("neg", "exp", "log", "sqrt", "absolute"):
        out[f"unary_{name}"] = A(getattr(tl, name)(T(u)))
    out["unary_relu"] = A(tnn.relu(T(u)))
    # relu gradient mask through the tape
    tl.reset_tape()
    x = T(u, grad=True)
    store = tl.backward(tl.sum(tnn.relu(x)))
    out["unary_relu_grad"] = A(store[x])
    # IEEE division specials (tests/test_core.py:231-238)
    num = np.array([1.0, -1.0, 0.0, 1.0], np.float32)
    den = np.array([0.0, 0.0, 0.0, -0.0], np.float32)
    out["div_special_num"], out["div_special_den"] = num, den
    out["div_special_out"] = A(tl.div(T(num), T(den)))
    save("elementwise.npz", **out)


def gen_reductions():
    out = {}
    for i, (x, axes, keep) in enumerate(reduction_cases()):
        out[f"r{i}_x"] = x
        out[f"r{i}_axes"] = np.array(axes if axes is not None else [-99], np.int64)
        out[f"r{i}_keep"] = np.array(keep)
        for kind in ("sum", "mean", "max"):
            tl.reset_tape()
            xt = T(x, grad=True)
            r = getattr(tl, kind)(xt, axis=axes, keepdims=keep)
            out[f"r{i}_{kind}"] = A(r)
            if kind == "max":  # gradient routing pins the argmax (core.py:721-726)
                store = tl.backward(tl.sum(r))
                out[f"r{i}_maxgrad"] = A(store[xt])
    # chunked double sum across a chunk boundary (tests/test_core.py:313-320)
    rng = random.Random(31)
    vals = np.array([rng.uniform(-1, 1) for _ in range(70_000)], np.float32)
    out["chunked_x"] = vals
    out["chunked_sum"] = A(tl.sum(T(vals)))
    save("reductions.npz", **out)


def gen_matmul():
    out = {}
    for i, (x, w, g) in enumerate(matmul_cases()):
        tl.reset_tape()
        xt, wt = T(x, grad=True), T(w, grad=True)
        y = tl.matmul(xt, wt)
        store = tl.backward(y, seed=T(g))
        out[f"m{i}_x"], out[f"m{i}_w"], out[f"m{i}_g"] = x, w, g
        out[f"m{i}_y"] = A(y)
        out[f"m{i}_dx"] = A(store[xt])
        out[f"m{i}_dw"] = A(store[wt])
    save("matmul.npz", **out)


def gen_ce_optim():
    out = {}
    for i, (z, labels) in enumerate(ce_cases()):
        tl.reset_tape()
        zt = T(z, grad=True)
        loss = tnn.cross_entropy(zt, labels.tolist())
        store = tl.backward(loss)
        out[f"ce{i}_z"], out[f"ce{i}_labels"] = z, labels
        out[f"ce{i}_loss"] = A(loss)
        out[f"ce{i}_grad"] = A(store[zt])
    # optimizer sequences (optim.py:54-100) on a vector of params, 4 steps
    rng = np.random.default_rng(11)
    theta0 = rng.standard_normal(257).astype(np.float32)
    grads = rng.standard_normal((4, 257)).astype(np.float32)
    out["opt_theta0"], out["opt_grads"] = theta0, grads
    for name, opt in (
        ("sgd", topt.SGD(lr=0.01)),
        ("sgd_mom_wd", topt.SGD(lr=0.05, momentum=0.9, weight_decay=0.01)),
        ("adam", topt.Adam(lr=1e-3)),
        ("adam_wd", topt.Adam(lr=3e-3, betas=(0.8, 0.99), eps=1e-6, weight_decay=0.1)),
    ):
        p = T(theta0)
        seq = []
        for k in range(4):
            opt.step(p, T(grads[k]))
            seq.append(A(p))
        out[f"opt_{name}"] = np.stack(seq)
    save("ce_optim.npz", **out)


def _mlp_step(params, x, labels, opt):
    """demos.run_blobs loop body (demos.py:110-121) on a Dense/ReLU stack."""
    tl.reset_tape()
    layers = []
    for i, (w, b) in enumerate(params):
        d = tnn.Dense(w.shape[1], w.shape[0], rng=0)
        d.weight.write_flat(w.ravel().tolist())
        d.bias.write_flat(b.ravel().tolist())
        layers.append(d)
        if i < len(params) - 1:
            layers.append(tnn.ReLU())
    model = tnn.Sequential(*layers)
    return model, layers


def run_mlp(params, x, labels, opt, steps):
    model, layers = _mlp_step(params, x, labels, opt)
    dense = [l for l in layers if isinstance(l, tnn.Dense)]
    losses, grads = [], None
    for s in range(steps):
        tl.reset_tape()
        logits = model(T(x))
        loss = tnn.cross_entropy(logits, labels.tolist())
        losses.append(loss.item())
        store = tl.backward(loss)
        grads = [(A(store[d.weight]), A(store[d.bias])) for d in dense]
        topt.step_all(opt, model.parameters(), store)
    newp = [(A(d.weight), A(d.bias)) for d in dense]
    return np.array(losses, np.float32), grads, newp


def gen_configs():
    # config 1: full size, one SGD step lr=0.01
    t0 = time.time()
    params, x, labels = config1_inputs()
    losses, grads, newp = run_mlp(params, x, labels, topt.SGD(lr=0.01), 1)
    out = {"loss": losses}
    for i, ((gw, gb), (w, b)) in enumerate(zip(grads, newp)):
        out[f"gw{i}"], out[f"gb{i}"], out[f"w{i}"], out[f"b{i}"] = gw, gb, w, b
    save("config1.npz", **out)
    print(f"  config1 reference step {time.time() - t0:.1f}s")

    # config 2 (reduced shape), bit-exact recipe
    a, b = config2_inputs(rows=256, cols=512)
    tl.reset_tape()
    at, bt = T(a, grad=True), T(b, grad=True)
    q = tl.add(tl.mul(at, bt), bt)
    y = tnn.relu(q)
    out = {"y": A(y), "e": A(tl.exp(T(np.clip(a, -10, 10))))}
    with tl.no_grad():
        for d in (0, 1):
            out[f"sum{d}"] = A(tl.sum(y, axis=d))
            out[f"mean{d}"] = A(tl.mean(y, axis=d))
            out[f"max{d}"] = A(tl.max(y, axis=d))
        out["sum_all"] = A(tl.sum(y))
    store = tl.backward(tl.sum(y))
    out["grad_a"], out["grad_b"] = A(store[at]), A(store[bt])
    save("config2_small.npz", **out)

    # config 3 (reduced): C = A@B through x.w^T with a transposed view
    A_, B_, dC = config3_inputs(n=96)
    tl.reset_tape()
    at, bt = T(A_, grad=True), T(B_, grad=True)
    C = tl.matmul(at, tl.transpose2d(bt))
    store = tl.backward(C, seed=T(dC))
    save("config3_small.npz", C=A(C), dA=A(store[at]), dB=A(store[bt]))

    # config 4 (reduced rows/width): composed softmax with detached max
    X, W, bias, Tt = config4_inputs(b=2, s=16, k=64)
    tl.reset_tape()
    xt, wt, bt = T(X.reshape(-1, X.shape[-1]), grad=True), T(W, grad=True), T(bias, grad=True)
    z = tl.add(tl.matmul(xt, tl.transpose2d(wt)), bt)
    with tl.no_grad():
        m = tl.max(z, axis=-1, keepdims=True)
    m = m.detach()
    e = tl.exp(tl.sub(z, m))
    s = tl.sum(e, axis=-1, keepdims=True)
    Y = tl.div(e, s)
    loss = tl.mean(tl.mul(Y, T(Tt.reshape(Y.shape))))
    store = tl.backward(loss)
    save("config4_small.npz", loss=A(loss), Y=A(Y), dX=A(store[xt]),
         dW=A(store[wt]), dbias=A(store[bt]))

    # config 5 (reduced width/batch): 3 Adam steps
    params, x, labels = config5_inputs(width=64, classes=10, batch=32, depth=4)
    losses, grads, newp = run_mlp(params, x, labels, topt.Adam(lr=1e-3), 3)
    out = {"loss": losses}
    for i, ((gw, gb), (w, b)) in enumerate(zip(grads, newp)):
        out[f"gw{i}"], out[f"gb{i}"], out[f"w{i}"], out[f"b{i}"] = gw, gb, w, b
    save("config5_small.npz", **out)


def gen_next_rows():
    """activations (nn.py:95-144), RMSprop (optim.py:103-122)
    and the demo training callers' logs (demos.py:42-130)."""
    from tensorlite import demos as tdemos

    out = {}
    u = unary_values()
    out["act_x"] = u
    g = np.random.default_rng(12).standard_normal(u.shape).astype(np.float32)
    out["act_g"] = g
    for name in ("sigmoid", "tanh", "gelu"):
        tl.reset_tape()
        x = T(u, grad=True)
        y = getattr(tnn, name)(x)
        store = tl.backward(y, seed=T(g))
        out[f"act_{name}"] = A(y)
        out[f"act_{name}_grad"] = A(store[x])
    rng = np.random.default_rng(13)
    theta0 = rng.standard_normal(257).astype(np.float32)
    grads = rng.standard_normal((4, 257)).astype(np.float32)
    out["opt_theta0"], out["opt_grads"] = theta0, grads
    for name, opt in (("rmsprop", topt.RMSprop(lr=0.01)),
                      ("rmsprop_wd", topt.RMSprop(lr=3e-3, rho=0.9, eps=1e-6, weight_decay=0.05))):
        p = T(theta0)
        seq = []
        for k in range(4):
            opt.step(p, T(grads[k]))
            seq.append(A(p))
        out[f"opt_{name}"] = np.stack(seq)
    xor = tdemos.run_xor(seed=0, epochs=300)
    blobs = tdemos.run_blobs(seed=0, epochs=60)
    out["xor_lines"] = np.array(xor.lines)
    out["blobs_lines"] = np.array(blobs.lines)
    blobs_rms = tdemos.run_blobs(seed=3, epochs=30, lr=0.01, optimizer="rmsprop")
    out["blobs_rms_lines"] = np.array(blobs_rms.lines)
    save("next_rows.npz", **out)




def gen_catalog():
    """Conv2D (nn.py:191-325), BatchNorm (nn.py:366-412),
    dropout (nn.py:415-437) on the reference."""
    out = {}
    rng = np.random.default_rng(41)
    for i, (b, cin, h, w, cout, k, s, p, bias) in enumerate(CONV_CASES):
        layer = tnn.Conv2D(cin, cout, k, stride=s, padding=p, bias=bias, rng=100 + i)
        x = rng.standard_normal((b, cin, h, w)).astype(np.float32)
        tl.reset_tape()
        xt = T(x, grad=True)
        y = layer(xt)
        g = rng.standard_normal(y.shape).astype(np.float32)
        store = tl.backward(y, seed=T(g))
        out[f"conv{i}_x"], out[f"conv{i}_g"] = x, g
        out[f"conv{i}_w"] = A(layer.weight)
        out[f"conv{i}_y"] = A(y)
        out[f"conv{i}_dx"] = A(store[xt])
        out[f"conv{i}_dw"] = A(store[layer.weight])
        if bias:
            out[f"conv{i}_b"] = A(layer.bias)
            out[f"conv{i}_db"] = A(store[layer.bias])
    # batchnorm: two train steps (output, grads, running buffers), then eval
    bn = tnn.BatchNorm(6, eps=1e-5, momentum=0.1)
    for k in range(2):
        x = (rng.standard_normal((16, 6)) * (k + 1) + k).astype(np.float32)
        g = rng.standard_normal((16, 6)).astype(np.float32)
        tl.reset_tape()
        xt = T(x, grad=True)
        y = bn(xt)
        store = tl.backward(y, seed=T(g))
        out[f"bn{k}_x"], out[f"bn{k}_g"] = x, g
        out[f"bn{k}_y"], out[f"bn{k}_dx"] = A(y), A(store[xt])
        out[f"bn{k}_dgamma"], out[f"bn{k}_dbeta"] = A(store[bn.gamma]), A(store[bn.beta])
        out[f"bn{k}_rmean"], out[f"bn{k}_rvar"] = A(bn.running_mean), A(bn.running_var)
    bn.set_mode("eval")
    xe = rng.standard_normal((5, 6)).astype(np.float32)
    with tl.no_grad():
        out["bn_eval_x"], out["bn_eval_y"] = xe, A(bn(T(xe)))
    # dropout with a seeded stream
    xd = rng.standard_normal((7, 9)).astype(np.float32)
    tl.reset_tape()
    xt = T(xd, grad=True)
    y = tnn.dropout(xt, 0.3, "train", rng=random.Random(5))
    store = tl.backward(tl.sum(y))
    out["drop_x"], out["drop_y"], out["drop_dx"] = xd, A(y), A(store[xt])
    save("catalog.npz", **out)


if __name__ == "__main__":
    gen_catalog()
    gen_next_rows()
    gen_elementwise()
    gen_reductions()
    gen_matmul()
    gen_ce_optim()
    gen_configs()
