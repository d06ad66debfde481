"""Every BASELINE config at its stated size, on the device, against the oracle.

* config 2 at 4096^2: bit-exact (every output and both gradients);
* config 3 at n = 1024 / 4096 / 8192: C, dA, dB within 1e-4 normwise;
* config 4 at X[64,512,1024] (every GEMM on tcgen05): loss, Y, dX, dW, dbias
  within 1e-4;
* config 5 at full width (4 x 4096 + 1000), batch 1024 of the 65536 (the
  oracle's fp64 GEMMs bound the batch), one Adam step:
  - in the reference-arithmetic GEMM mode ('ref': exact fp32 products summed
    in fp64, one f32 rounding -- core.py:802-807), the loss, all 10 gradients
    and all updated parameters against the oracle at 1e-4, with the raw
    numbers (bit-identical fraction, Adam sign flips) recorded;
  - for the fast schemes (3xBF16 default, TF32X, 3xTF32, FP32 SIMT) the
    well-posed tensors (loss, logits, activations, gradients conditioned on
    the device's relu pattern) at 1e-4, with the raw gradient error and the
    relu-flip counts recorded next to the ref mode's.

The reference pins oracle equivalence on seeded instances the same way
(pkg/tests/test_acceptance.py:79-123). Raw numbers go to
gpurun_out/full_config_parity.json when that directory exists.
"""

import json
import os

import numpy as np
import pytest

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import nn, optim
from oracle import tensorlite_np as O
from tests.golden import inputs as I
from tests.golden.load import bits_equal, normwise

pytestmark = pytest.mark.gpu

TOL = 1e-4
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_RECORD = {}


def _record(key, value):
    _RECORD[key] = value
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "full_config_parity.json"), "w") as f:
            json.dump(_RECORD, f, indent=1, sort_keys=True)


def dev(a, grad=False):
    return P.from_numpy(np.asarray(a, np.float32), requires_grad=grad)


def _bit_frac(a, b):
    a = np.ascontiguousarray(a, np.float32).view(np.uint32)
    b = np.ascontiguousarray(b, np.float32).view(np.uint32)
    return float(np.count_nonzero(a == b)) / max(a.size, 1)


# ---------------------------------------------------------------- config 2


def test_config2_full_size_bit_exact():
    a, b = I.config2_inputs()
    ref = O.broadcast_reduce_config(a, b)
    P.reset_tape()
    at, bt = dev(a, True), dev(b, True)
    y = P.fused_muladd_relu(at, bt)
    assert bits_equal(y.numpy(), ref["y"])
    assert bits_equal(P.exp(P.clamp(dev(a), -10, 10)).numpy(), ref["e"])
    with P.no_grad():
        for d in (0, 1):
            assert bits_equal(P.sum(y, axis=d).numpy(), ref[f"sum{d}"]), d
            assert bits_equal(P.mean(y, axis=d).numpy(), ref[f"mean{d}"]), d
            assert bits_equal(P.max(y, axis=d).numpy(), ref[f"max{d}"]), d
        assert bits_equal(P.sum(y).numpy(), ref["sum_all"])
    store = P.backward(P.sum(y))
    assert bits_equal(store[at].numpy(), ref["grad_a"])
    assert bits_equal(store[bt].numpy(), ref["grad_b"])
    # the composed reference ops give the same bits as the fused kernels
    P.reset_tape()
    at, bt = dev(a, True), dev(b, True)
    yc = P.relu(P.add(P.mul(at, bt), bt))
    assert bits_equal(yc.numpy(), ref["y"])
    store = P.backward(P.sum(yc))
    assert bits_equal(store[at].numpy(), ref["grad_a"])
    assert bits_equal(store[bt].numpy(), ref["grad_b"])
    _record("config2_4096x4096", {"bit_exact": True})


# ---------------------------------------------------------------- config 3


@pytest.mark.parametrize("n", [1024, 4096, 8192])
def test_config3_full_size(n):
    A, B, dC = I.config3_inputs(n=n)
    P.reset_tape()
    At, Bt = dev(A, True), dev(B, True)
    C = P.mm(At, Bt)
    store = P.backward(C, seed=dev(dC))
    Co, dAo, dBo = O.matmul_fwd_bwd(A, B, dC)
    errs = {"C": normwise(C.numpy(), Co), "dA": normwise(store[At].numpy(), dAo),
            "dB": normwise(store[Bt].numpy(), dBo)}
    _record(f"config3_n{n}", errs)
    for k, e in errs.items():
        assert e <= TOL, (n, k, e)


# ---------------------------------------------------------------- config 4


def test_config4_full_size():
    X, W, bias, T = I.config4_inputs()
    K = X.shape[-1]
    P.reset_tape()
    xt, wt, bt = dev(X, True), dev(W, True), dev(bias, True)
    z = P.add(P.mm(xt, wt), bt)
    Y = P.softmax(z)
    loss = P.mean(P.mul(Y, dev(T)))
    store = P.backward(loss)
    ref = O.softmax_linear_config(X.reshape(-1, K), W, bias, T.reshape(-1, K))
    errs = {"loss": normwise(np.float32(loss.item()), ref["loss"]),
            "Y": normwise(Y.numpy().reshape(-1, K), ref["Y"].reshape(-1, K)),
            "dX": normwise(store[xt].numpy().reshape(-1, K), ref["dX"].reshape(-1, K)),
            "dW": normwise(store[wt].numpy(), ref["dW"]),
            "dbias": normwise(store[bt].numpy(), ref["dbias"])}
    _record("config4_64x512x1024", errs)
    for k, e in errs.items():
        assert e <= TOL, (k, e)


# ---------------------------------------------------------------- config 5

C5_BATCH = 1024


@pytest.fixture(scope="module")
def c5():
    params, x, labels = I.config5_inputs(batch=C5_BATCH)
    ref = O.mlp_train_step(params, x, labels, O.Adam(lr=1e-3))
    return params, x, labels, ref


def _model(params):
    layers = []
    for i, (w, b) in enumerate(params):
        d = nn.Dense(w.shape[1], w.shape[0], rng=0)
        d.weight.write_flat(w.ravel())
        d.bias.write_flat(b.ravel())
        layers.append(d)
        if i < len(params) - 1:
            layers.append(nn.ReLU())
    return nn.Sequential(*layers), [l for l in layers if isinstance(l, nn.Dense)]


def _device_step(params, x, labels, algo):
    """One config-5 Adam step on the device; returns loss, every layer's
    output (logits last), gradients and updated parameters as host arrays."""
    from tests.test_gpu_parity import _device_forward

    P.set_gemm_algo(algo)
    try:
        model, dense = _model(params)
        P.reset_tape()
        loss = nn.cross_entropy(model(dev(x)), labels)
        store = P.backward(loss)
        grads = [(store[d.weight].numpy(), store[d.bias].numpy()) for d in dense]
        optim.step_all(optim.Adam(lr=1e-3), model.parameters(), store)
        newp = [(d.weight.numpy(), d.bias.numpy()) for d in dense]
        with P.no_grad():  # the same fused kernels, deterministic: the step's activations
            acts = _device_forward(params, x)
        return float(loss.item()), acts, grads, newp
    finally:
        P.set_gemm_algo(None)


def test_config5_full_width_reference_arithmetic(c5):
    """Exact-arithmetic control: with the reference's own GEMM arithmetic every
    non-GEMM kernel is already bit-exact, so the whole step -- loss, all 10
    gradients, all 10 updated parameter tensors -- must meet 1e-4 against the
    oracle with no conditioning."""
    params, x, labels, ref = c5
    loss, acts, grads, newp = _device_step(params, x, labels, "ref")
    rec = {"loss": normwise(np.float32(loss), ref["loss"]),
           "logits": normwise(acts[-1], ref["logits"]),
           "logits_bit_frac": _bit_frac(acts[-1], ref["logits"])}
    flips = total = 0
    for i, ((gw, gb), (w, b), (rw, rb), (pw, pb)) in enumerate(
            zip(grads, newp, ref["grads"], ref["params"])):
        rec[f"gW{i}"], rec[f"gb{i}"] = normwise(gw, rw), normwise(gb, rb)
        rec[f"W{i}"], rec[f"b{i}"] = normwise(w, pw), normwise(b, pb)
        rec[f"gW{i}_bit_frac"] = _bit_frac(gw, rw)
        rec[f"W{i}_bit_frac"] = _bit_frac(w, pw)
        flips += int(np.count_nonzero(np.sign(gw) != np.sign(rw)))
        total += rw.size
    rec["adam_sign_flips"] = f"{flips}/{total}"
    _record("config5_ref_arithmetic", rec)
    for k, v in rec.items():
        if isinstance(v, float) and not k.endswith("bit_frac"):
            assert v <= TOL, (k, v)


@pytest.mark.parametrize("algo", ["3xbf16", "tf32x", "3xtf32", "simt"])
def test_config5_full_width_fast_schemes(c5, algo):
    """The fp32-accurate fast schemes at full width: the well-posed tensors at
    1e-4; the raw (unconditioned) gradient error and the relu flips recorded."""
    from tests.test_gpu_parity import _conditioned_step, _mm64

    params, x, labels, ref = c5
    loss, acts, grads, _ = _device_step(params, x, labels, algo)
    z, cgrads = _conditioned_step(params, acts, labels, _mm64)
    n = len(params)
    rec = {"loss": normwise(np.float32(loss), ref["loss"]),
           "logits": normwise(acts[-1], ref["logits"])}
    flips = total = 0
    worst_act = worst_cond = worst_raw = 0.0
    for i in range(n):
        want = O.relu(z[i]) if i < n - 1 else z[i]
        worst_act = max(worst_act, normwise(acts[i + 1], want))
        if i < n - 1:
            flips += int(np.count_nonzero((acts[i + 1] > 0) != (z[i] > 0)))
            total += z[i].size
    for (gw, gb), (cw, cb), (rw, rb) in zip(grads, cgrads, ref["grads"]):
        worst_cond = max(worst_cond, normwise(gw, cw), normwise(gb, cb))
        worst_raw = max(worst_raw, normwise(gw, rw), normwise(gb, rb))
    rec.update(activations=worst_act, grads_conditioned=worst_cond, grads_raw=worst_raw,
               relu_flips=f"{flips}/{total}")
    _record(f"config5_{algo}", rec)
    assert rec["loss"] <= TOL and rec["logits"] <= TOL, rec
    assert worst_act <= TOL and worst_cond <= TOL, rec
    assert flips <= max(1, total // 10000), rec


def test_config4_full_size_fused_linear_and_loss():
    """The fused form of config 4 (nn.Linear with the bias in the GEMM
    epilogue, softmax_mul_mean) at full size against the oracle."""
    X, W, bias, T = I.config4_inputs()
    K = X.shape[-1]
    P.reset_tape()
    xt, wt, bt = dev(X.reshape(-1, K), True), dev(W, True), dev(bias, True)
    z = P.linear(xt, P.transpose2d(wt), bt)
    loss = P.softmax_mul_mean(z, dev(T.reshape(-1, K)))
    store = P.backward(loss)
    ref = O.softmax_linear_config(X.reshape(-1, K), W, bias, T.reshape(-1, K))
    errs = {"loss": normwise(np.float32(loss.item()), ref["loss"]),
            "dX": normwise(store[xt].numpy(), ref["dX"].reshape(-1, K)),
            "dW": normwise(store[wt].numpy(), ref["dW"]),
            "dbias": normwise(store[bt].numpy(), ref["dbias"])}
    _record("config4_64x512x1024_fused", errs)
    for k, e in errs.items():
        assert e <= TOL, (k, e)


def test_config2_full_size_single_pass_bit_exact():
    """The whole config-2 workload in ONE read of a (b2_muladd_relu_stats)
    gives the oracle's bits for every output and both gradients."""
    a, b = I.config2_inputs()
    ref = O.broadcast_reduce_config(a, b)
    out = P.muladd_relu_stats(dev(a), dev(b))
    for k in ("y", "e", "sum0", "sum1", "mean0", "mean1", "max0", "max1", "sum_all", "grad_a",
              "grad_b"):
        assert bits_equal(out[k].numpy(), ref[k]), k
    _record("config2_single_pass", {"bit_exact": True})


def test_config5_bf16_variant_against_its_exact_arithmetic_control(c5):
    """The bf16 variant at full width (batch 1024, one Adam step) and its
    exact-arithmetic control ('ref_bf16': the same bf16-rounded operands,
    exact products, compensated fp64 sums).

    * control vs the fp32 oracle: loss and logits within the bf16 tolerance
      2e-2; the hidden-layer gradients' deviation is recorded -- it is the
      cost of bf16 operands themselves (no accumulation error is left), which
      is why 2e-2 on hidden-layer gradients is out of reach for any
      bf16-operand implementation at random init;
    * the device's bf16 variant vs the control: loss and logits within 5e-3,
      gradients conditioned on the device's relu pattern within 5e-3."""
    from tests.test_gpu_parity import _conditioned_step, _mm_bf16

    params, x, labels, ref = c5
    closs, cacts, cgrads, _ = _device_step(params, x, labels, "ref_bf16")
    loss, acts, grads, _ = _device_step(params, x, labels, "bf16")
    rec = {"control_loss_vs_fp32": normwise(np.float32(closs), ref["loss"]),
           "control_logits_vs_fp32": normwise(cacts[-1], ref["logits"])}
    for i, ((gw, gb), (rw, rb)) in enumerate(zip(cgrads, ref["grads"])):
        rec[f"control_gW{i}_vs_fp32"] = normwise(gw, rw)
    rec["variant_loss_vs_control"] = normwise(np.float32(loss), np.float32(closs))
    rec["variant_logits_vs_control"] = normwise(acts[-1], cacts[-1])
    z, egrads = _conditioned_step(params, acts, labels, _mm_bf16)
    rec["variant_grads_conditioned"] = max(
        max(normwise(gw, ew), normwise(gb, eb)) for (gw, gb), (ew, eb) in zip(grads, egrads))
    _record("config5_bf16_control", rec)
    assert rec["control_loss_vs_fp32"] <= 2e-2 and rec["control_logits_vs_fp32"] <= 2e-2, rec
    # a 1-ulp fp32 accumulation difference that straddles a bf16 rounding
    # boundary moves the next layer's operand by 2^-8: a few elements per
    # layer, ~2.5e-3 normwise on the logits at this width
    assert rec["variant_loss_vs_control"] <= 1e-3 and rec["variant_logits_vs_control"] <= 5e-3, rec
    assert rec["variant_grads_conditioned"] <= 5e-3, rec
