"""Device parity: libb2 (through the package API and the C ABI) vs the
reference-pinned goldens and the NumPy oracle.

Bit-exact where SURVEY 8a says the reference is bit-exact-achievable
(elementwise, relu masks, sums/means via fp64, max/argmax routing, CE in
double, SGD/Adam in double, composed softmax); fp32 tolerance
``max|dev-ref| <= 1e-4 * max|ref|`` (normwise) wherever a GEMM
sits on the path.
"""

import numpy as np
import pytest

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import nn, optim
from oracle import tensorlite_np as O
from tests.golden import inputs as I
from tests.golden.load import bits_equal, load, normwise
from paper_2602_00125_b200 import _lib as L

pytestmark = pytest.mark.gpu

TOL = 1e-4


def dev(a, grad=False):
    return P.from_numpy(np.asarray(a, np.float32), requires_grad=grad)


def host(t):
    return t.numpy()


# ---------------------------------------------------------------- elementwise


def test_broadcast_binary_bit_exact():
    g = load("elementwise.npz")
    ops = {"add": P.add, "sub": P.sub, "mul": P.mul, "div": P.div}
    for i, (kind, va, vb) in enumerate(I.broadcast_cases()):
        got = ops[kind](dev(va), dev(vb))
        want = g[f"bc{i}_{kind}_out"]
        assert got.shape == want.shape, (i, kind)
        assert bits_equal(host(got), want), (i, kind)


@pytest.mark.parametrize("name", ["neg", "exp", "log", "sqrt", "absolute", "relu"])
def test_unary_bit_exact(name):
    g = load("elementwise.npz")
    got = getattr(P, name)(dev(g["unary_x"]))
    assert bits_equal(host(got), g[f"unary_{name}"]), name


def test_relu_grad_bit_exact():
    g = load("elementwise.npz")
    x = dev(g["unary_x"], grad=True)
    store = P.backward(P.sum(P.relu(x)))
    assert bits_equal(host(store[x]), g["unary_relu_grad"])


def test_div_ieee_specials():
    g = load("elementwise.npz")
    got = P.div(dev(g["div_special_num"]), dev(g["div_special_den"]))
    assert bits_equal(host(got), g["div_special_out"])


def test_scalar_promotion_and_strided_views():
    x = np.arange(12, dtype=np.float32).reshape(3, 4) - 5.5
    t = dev(x)
    assert bits_equal(host(P.add(t, 1)), O.add(x, np.float32(1)))
    assert bits_equal(host(P.mul(3, t)), O.mul(np.float32(3), x))
    assert bits_equal(host(P.div(2.0, t)), O.div(np.float32(2), x))
    tt = P.transpose2d(t)
    assert bits_equal(host(P.exp(tt)), O.exp(x.T))
    assert bits_equal(host(P.sub(tt, P.transpose2d(t))), np.zeros((4, 3), np.float32))
    bt = P.broadcast_to(dev(x[:1]), (5, 3, 4))
    assert bits_equal(host(P.mul(bt, t)), O.mul(np.broadcast_to(x[:1], (5, 3, 4)), x))


def test_large_elementwise_vectorized_paths():
    rng = np.random.default_rng(1)
    a = rng.standard_normal((1023, 4097)).astype(np.float32)
    b = rng.standard_normal((1, 4097)).astype(np.float32)
    assert bits_equal(host(P.mul(dev(a), dev(b))), O.mul(a, b))
    a4 = rng.standard_normal((512, 4096)).astype(np.float32)
    b4 = rng.standard_normal((4096,)).astype(np.float32)
    assert bits_equal(host(P.add(dev(a4), dev(b4))), O.add(a4, b4))
    col = rng.standard_normal((512, 1)).astype(np.float32)
    assert bits_equal(host(P.sub(dev(a4), dev(col))), O.sub(a4, col))


# ---------------------------------------------------------------- reductions


def test_reductions_bit_exact():
    g = load("reductions.npz")
    for i, (x, axes, keep) in enumerate(I.reduction_cases()):
        for kind in ("sum", "mean", "max"):
            P.reset_tape()
            xt = dev(x, grad=True)
            r = getattr(P, kind)(xt, axis=axes, keepdims=keep)
            want = g[f"r{i}_{kind}"]
            assert r.shape == want.shape, (i, kind)
            assert bits_equal(host(r), want), (i, kind, x.shape, axes, keep)
            if kind == "max":
                store = P.backward(P.sum(r))
                assert bits_equal(host(store[xt]), g[f"r{i}_maxgrad"]), (i, "maxgrad")


def test_chunked_full_sum_bit_exact():
    g = load("reductions.npz")
    assert bits_equal(host(P.sum(dev(g["chunked_x"]))), g["chunked_sum"])


def test_large_reductions_vs_oracle():
    rng = np.random.default_rng(2)
    x = rng.standard_normal((2048, 3000)).astype(np.float32)
    t = dev(x)
    for ax in (0, 1, None):
        assert bits_equal(host(P.sum(t, axis=ax)), O.axis_sum(x, ax)), ax
        assert bits_equal(host(P.mean(t, axis=ax)), O.axis_mean(x, ax)), ax
        assert bits_equal(host(P.max(t, axis=ax)), O.axis_max(x, ax)[0]), ax
    x3 = rng.standard_normal((6, 70, 9, 5)).astype(np.float32)
    t3 = dev(x3)
    for ax in ((1,), (0, 2), (1, 3), (0, 1, 2)):
        assert bits_equal(host(P.sum(t3, axis=ax)), O.axis_sum(x3, ax)), ax
        v, _ = O.axis_max(x3, ax)
        assert bits_equal(host(P.max(t3, axis=ax)), v), ax


def test_max_nan_and_ties_semantics():
    x = np.array([[np.nan, 1.0, 2.0], [1.0, np.nan, 0.5], [3.0, 3.0, 1.0], [-0.0, 0.0, -1.0]],
                 np.float32)
    xt = dev(x, grad=True)
    r = P.max(xt, axis=1)
    v, pos = O.axis_max(x, 1)
    assert bits_equal(host(r), v)
    store = P.backward(P.sum(r))
    assert bits_equal(host(store[xt]), O.max_pullback(np.ones(4, np.float32), pos, x.shape))


def test_max_dim0_ties_signed_zeros_nans_at_scale():
    """Column max over long columns (blocked FMNMX scan + split partials):
    heavy ties, +-0 maxima, scattered NaNs (incl. some first slots) and all
    -inf columns -- values and argmax routing (via the gradient) bit-exact."""
    rng = np.random.default_rng(11)
    R, C = 6000, 520
    x = rng.integers(-3, 1, (R, C)).astype(np.float32)  # max is 0 in most columns: ties
    x[rng.random((R, C)) < 0.3] = -0.0
    x[rng.random((R, C)) < 0.01] = np.nan
    x[0, 5] = np.nan                       # first-slot NaN sticks
    x[:, 7] = -np.inf                      # all -inf: index 0
    x[:, 9] = -1.0
    x[4321, 9] = 2.0                       # lone max deep in the column
    x[:, 11] = -0.0
    x[2500, 11] = 0.0                      # +0 after -0: the first (-0) wins
    xt = dev(x, grad=True)
    r = P.max(xt, axis=0)
    v, pos = O.axis_max(x, 0)
    assert bits_equal(host(r), v)
    store = P.backward(P.sum(r))
    assert bits_equal(host(store[xt]), O.max_pullback(np.ones(C, np.float32), pos, x.shape))


@pytest.mark.parametrize("shape", [(4096, 4096), (8192, 1024)])
@pytest.mark.parametrize("recording", [False, True])
def test_max_dim0_cluster_path_value_only_and_routed(shape, recording):
    """The DSMEM-cluster column max (k_cols; cluster of 4 at 4096^2, 16 at
    8192x1024) in both forms: value-only when no node is recorded (no_grad or
    an input without grad: the config-2 bench case) and with first-index
    routing when one is. Same values either way: first-slot NaN sticks, NaNs
    skipped, +-0 maxima take the sign of the first zero, all -inf columns."""
    rng = np.random.default_rng(12)
    R, C = shape
    x = rng.standard_normal((R, C)).astype(np.float32)
    x[rng.random((R, C)) < 0.001] = np.nan
    x[0, 3] = np.nan                         # first-slot NaN sticks
    x[:, 8] = -np.inf
    x[:, 10] = -np.abs(x[:, 10])
    x[17, 10] = -0.0
    x[900, 10] = 0.0                         # -0 first: the max is -0
    x[:, 12] = -np.abs(x[:, 12])
    x[5, 12] = 0.0
    x[6, 12] = -0.0                          # +0 first: the max is +0
    x[:, 14] = np.nan
    x[0, 14] = 1.0                           # NaNs after the first slot are skipped
    x[:, 15] = -np.abs(x[:, 15])
    x[R - 1, 15] = -0.0                      # the only zero is the last row
    v, pos = O.axis_max(x, 0)
    if recording:
        xt = dev(x, grad=True)
        r = P.max(xt, axis=0)
        assert bits_equal(host(r), v)
        store = P.backward(P.sum(r))
        assert bits_equal(host(store[xt]), O.max_pullback(np.ones(C, np.float32), pos, x.shape))
    else:
        with P.no_grad():
            assert bits_equal(host(P.max(dev(x, grad=True), axis=0)), v)
        assert bits_equal(host(P.max(dev(x), axis=0)), v)


def test_zero_extent_reductions():
    e = P.zeros((0, 3))
    assert P.sum(e).item() == 0.0
    assert np.isnan(P.mean(e).item())
    with pytest.raises(P.ShapeError):
        P.max(e)
    assert P.sum(e, axis=1).shape == (0,)


# ---------------------------------------------------------------- matmul


@pytest.mark.parametrize("algo", ["simt", "3xtf32", "tf32x", "3xbf16", "ref"])
def test_matmul_goldens(algo):
    g = load("matmul.npz")
    P.set_gemm_algo(algo)
    try:
        for i, (x, w, gr) in enumerate(I.matmul_cases()):
            P.reset_tape()
            xt, wt = dev(x, True), dev(w, True)
            y = P.matmul(xt, wt)
            store = P.backward(y, seed=dev(gr))
            for got, key in ((y, "y"), (store[xt], "dx"), (store[wt], "dw")):
                want = g[f"m{i}_{key}"]
                assert got.shape == want.shape
                if algo == "ref":  # the reference's compensated double dot: its exact bits
                    assert bits_equal(host(got), want), (i, key)
                    continue
                tol = 1e-5 if algo == "3xbf16" else 2e-6  # 3xBF16 operands carry 16 bits
                assert normwise(host(got), want) <= tol, (algo, i, key)
    finally:
        P.set_gemm_algo(None)


def _ref_gemm(A, B, ta, tb):
    a = A.astype(np.float64).T if ta else A.astype(np.float64)
    b = B.astype(np.float64) if tb else B.astype(np.float64).T
    return a @ b.T  # a [M,K] . b[N,K]^T


@pytest.mark.parametrize("ta,tb", [(0, 1), (0, 0), (1, 0), (1, 1)])
@pytest.mark.parametrize("shape", [(128, 256, 32), (304, 520, 200), (1000, 264, 1024), (64, 8, 16)])
def test_gemm_layouts_tc(ta, tb, shape):
    """tcgen05 3xTF32 and 1xTF32 against fp64, every operand layout, ragged tiles."""
    import ctypes
    from paper_2602_00125_b200 import _lib as L

    M, N, K = shape
    rng = np.random.default_rng(M + N + K + 2 * ta + tb)
    A = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    ref = _ref_gemm(A, B, ta, tb)
    At, Bt, bt = dev(A), dev(B), dev(bias)
    # 3xTF32 with K-chunk promotion is sgemm-grade (~1e-6); 1xTF32 is TF32-grade
    for algo, tol in ((L.GEMM_3XTF32, 5e-6), (L.GEMM_TF32X, 5e-6), (L.GEMM_3XBF16, 1e-5),
                      (L.GEMM_1XTF32, 3e-3), (L.GEMM_SIMT, 5e-6)):
        C = P.zeros((M, N))
        L.call("b2_gemm", ta, tb, M, N, K, At.data_ptr, A.shape[1], Bt.data_ptr, B.shape[1],
               C.data_ptr, N, bt.data_ptr, L.EPI_BIAS_RELU, algo, None)
        want = np.maximum(ref + bias.astype(np.float64), 0)
        err = normwise(host(C), want)
        assert err <= tol, (algo, ta, tb, shape, err)


def _bf16_rn(x):
    """Round-to-nearest-even fp32 -> bf16, returned as fp32 (finite inputs)."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def _bf16_bits(buf_ptr, n):
    import ctypes

    out = np.empty(n, np.uint16)
    from paper_2602_00125_b200 import _lib as L

    L.call("b2_memcpy_d2h", out.ctypes.data_as(ctypes.c_void_p), buf_ptr, 2 * n, None)
    return (out.astype(np.uint32) << 16).view(np.float32)


@pytest.mark.parametrize("ta,tb", [(0, 1), (0, 0), (1, 0), (1, 1)])
@pytest.mark.parametrize("shape", [(128, 256, 32), (304, 520, 200), (1000, 264, 1024), (256, 512, 2048)])
def test_gemm_layouts_bf16(ta, tb, shape):
    """BF16 variant: casts are bit-exact RN bf16; the GEMM on them equals the
    fp64 product of the rounded operands to fp32-accumulation accuracy (so the
    only approximation is the operand rounding); the fused bias/relu/mask
    epilogue and the emitted bf16 cast of C are exact."""
    from paper_2602_00125_b200 import _lib as L
    from paper_2602_00125_b200.core import Buffer

    M, N, K = shape
    rng = np.random.default_rng(M + N + K + 2 * ta + tb + 77)
    A = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    mask = (rng.uniform(-1, 1, (M, N)) > 0).astype(np.float32)
    At, Bt, bt, mt = dev(A), dev(B), dev(bias), dev(mask)
    A16, B16, C16 = Buffer(2 * A.size), Buffer(2 * B.size), Buffer(2 * M * N)
    L.call("b2_bf16_cast", A16.ptr, At.data_ptr, A.shape[0], A.shape[1], A.shape[1], None)
    L.call("b2_bf16_cast", B16.ptr, Bt.data_ptr, B.shape[0], B.shape[1], B.shape[1], None)
    Ar, Br = _bf16_rn(A), _bf16_rn(B)
    assert bits_equal(_bf16_bits(A16.ptr, A.size).reshape(A.shape), Ar)
    assert bits_equal(_bf16_bits(B16.ptr, B.size).reshape(B.shape), Br)
    C = P.zeros((M, N))
    L.call("b2_gemm_bf16", ta, tb, M, N, K, A16.ptr, B16.ptr, C.data_ptr, N, bt.data_ptr,
           L.EPI_BIAS_RELU, mt.data_ptr, C16.ptr, None, None)
    want = np.maximum(_ref_gemm(Ar, Br, ta, tb) + bias.astype(np.float64), 0) * mask
    got = host(C)
    assert normwise(got, want) <= 5e-6, (ta, tb, shape)
    assert bits_equal(_bf16_bits(C16.ptr, M * N).reshape(M, N), _bf16_rn(got))
    # and against the unrounded fp32 operands: bf16-grade
    full = np.maximum(_ref_gemm(A, B, ta, tb) + bias.astype(np.float64), 0) * mask
    assert normwise(got, full) <= 2e-2


def _mm64(a, b):  # a[M,K] . b[N,K]^T, exact products, fp32 result (the reference's matmul)
    return O.f32(np.asarray(a, np.float64) @ np.asarray(b, np.float64).T)


def _mm_bf16(a, b):  # the same on bf16-rounded operands (the bf16 variant's arithmetic)
    return O.f32(_bf16_rn(a).astype(np.float64) @ _bf16_rn(b).astype(np.float64).T)


def _device_forward(params, x):
    """Host copies of every layer output of the device forward (the fused
    linear(+relu) kernels Sequential runs; deterministic, so identical to the
    activations of the training step)."""
    from paper_2602_00125_b200 import core as C

    h, acts, n = dev(x), [np.asarray(x, np.float32)], len(params)
    for i, (w, b) in enumerate(params):
        h = C.linear(h, dev(w), dev(b), relu_out=i < n - 1)
        acts.append(host(h))
    return acts


def _conditioned_step(params, acts, labels, mm):
    """Layer-local reference: each layer's forward from the DEVICE's input
    activation, and the backward through the device's ReLU pattern.

    A relu-MLP's gradients are discontinuous in its pre-activations: an
    implementation whose fp32 sums differ from the reference's by 1 ulp
    flips the few pre-activations within 1 ulp of zero, and each flip moves
    one cotangent entry by its full size (a single flip is ~1/sqrt(batch)
    of max|dW|, far above 1e-4 at any batch size). Conditioning on the
    device's own activation pattern measures the GEMMs and the loss at the
    tolerance; the flips themselves are counted separately."""
    n = len(params)
    z = [O.add(mm(acts[i], w), b) for i, (w, b) in enumerate(params)]
    _, _, g = O.cross_entropy(acts[-1], labels)
    grads = [None] * n
    for i in range(n - 1, -1, -1):
        w, b = params[i]
        if i < n - 1:
            g = O.mul(g, O.relu_mask(acts[i + 1]))
        grads[i] = (mm(g.T, acts[i].T), O.reduce_to_shape(g, b.shape))
        g = mm(g, w.T)
    return z, grads


def _fro(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def test_config5_shape_bf16_variant_one_step():
    """The bf16 variant of config 5 (bf16 GEMM operands, fp32 accumulation,
    fp32 master weights, loss and optimizer).

    Gate: every layer equals the fp64 emulation of exactly that arithmetic
    (bf16-rounded operands, exact products) conditioned on the device's
    inputs / relu pattern, to fp32-accumulation accuracy. Against the fp32
    oracle the loss and logits are within the bf16 tolerance 2e-2. Hidden-
    layer gradients are not, for ANY bf16-operand implementation: the bf16
    forward moves ~0.1% of pre-activations across zero and the resulting
    cotangent jumps leave ~5-10% max-norm noise in the batch-summed dW at
    random init, independently of the batch size (the unconditioned
    emulation shows the same)."""
    params, x, labels = I.config5_inputs(width=256, classes=16, batch=128, depth=3)
    P.set_gemm_algo("bf16")
    try:
        losses, grads, _ = _run_mlp_device(params, x, labels, optim.SGD(lr=0.0), 1)
        acts = _device_forward(params, x)
    finally:
        P.set_gemm_algo(None)
    z, egrads = _conditioned_step(params, acts, labels, _mm_bf16)
    n = len(params)
    for i in range(n):
        want = O.relu(z[i]) if i < n - 1 else z[i]
        assert normwise(acts[i + 1], want) <= 1e-5, i
    ref = O.mlp_train_step(params, x, labels, O.SGD(lr=0.0))
    assert normwise(losses, np.float32(ref["loss"])) <= 2e-2
    assert normwise(acts[-1], ref["logits"]) <= 2e-2
    # backward: the cotangents are bf16-rounded before every GEMM, so a 1-ulp
    # fp32 accumulation difference that straddles a bf16 rounding boundary
    # moves an operand by 2^-8 relative (a few per layer at this size), and
    # the layers below inherit it through W: 1e-3 in Frobenius norm, 5e-3 max
    for i, ((gw, gb), (ew, eb)) in enumerate(zip(grads, egrads)):
        assert _fro(gw, ew) <= 1e-3 and normwise(gw, ew) <= 5e-3, i
        assert _fro(gb, eb) <= 1e-3 and normwise(gb, eb) <= 5e-3, i
    (gw, gb), (rw, rb) = grads[-1], ref["grads"][-1]
    assert normwise(gw, rw) <= 2e-2 and normwise(gb, rb) <= 2e-2


def test_config5_small_bf16_variant_adam_losses():
    """bf16 variant, 3 Adam steps: the loss trajectory stays within 2e-2 of
    the fp32 reference's."""
    golden = load("config5_small.npz")
    params, x, labels = I.config5_inputs(width=64, classes=10, batch=32, depth=4)
    P.set_gemm_algo("bf16")
    try:
        losses, _, _ = _run_mlp_device(params, x, labels, optim.Adam(lr=1e-3), 3)
    finally:
        P.set_gemm_algo(None)
    assert normwise(losses, golden["loss"]) <= 2e-2


@pytest.mark.parametrize("ta,tb", [(0, 1), (0, 0), (1, 0), (1, 1)])
@pytest.mark.parametrize("shape", [(2048, 1056, 72), (256, 256, 784), (256, 10, 256), (10, 784, 256),
                                   (3, 5, 1000), (70, 130, 17), (1100, 1302, 70), (1024, 2200, 64),
                                   (1500, 1500, 16), (1281, 1153, 9), (832, 832, 300)])
def test_gemm_simt_paths(ta, tb, shape):
    """FP32 FFMA paths: the 128x128 tile kernel (many tiles: FFMA2, interior
    128-bit loads and guarded edge tiles, leading dimensions that are not a
    multiple of 4 -> scalar loads, a ragged last raster group, K below and
    across one k-tile) and the 64x64 cluster split-K latency kernel (config-1
    shapes, ragged, clusters of 1..6 K slices, and 832x832x300: one CTA per
    tile walking K in three staging passes)."""
    from paper_2602_00125_b200 import _lib as L

    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N + K + ta + 2 * tb)
    A = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
    bias = rng.uniform(-1, 1, N).astype(np.float32)
    ref = np.maximum(_ref_gemm(A, B, ta, tb) + bias.astype(np.float64), 0)
    At, Bt, bt = dev(A), dev(B), dev(bias)  # keep the operands alive across the call
    C = P.zeros((M, N))
    L.call("b2_gemm", ta, tb, M, N, K, At.data_ptr, A.shape[1], Bt.data_ptr, B.shape[1],
           C.data_ptr, N, bt.data_ptr, L.EPI_BIAS_RELU, L.GEMM_SIMT, None)
    assert normwise(host(C), ref) <= 5e-6, (ta, tb, shape)


@pytest.mark.parametrize("ta,tb", [(0, 1), (1, 0), (1, 1)])
def test_gemm_split_k_few_tiles_long_k(ta, tb):
    """Few output tiles and a long K (the dW GEMMs of configs 4/5) take the
    split-K path: fp32 partial slices + a fixed-order second stage carrying
    the fused epilogue. Every tensor-core scheme, against fp64."""
    from paper_2602_00125_b200 import _lib as L

    M, N, K = 256, 384, 16384
    rng = np.random.default_rng(21 + ta + 2 * tb)
    A = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
    bias = rng.uniform(-1, 1, N).astype(np.float32) * 8
    ref = np.maximum(_ref_gemm(A, B, ta, tb) + bias.astype(np.float64), 0)
    At, Bt, bt = dev(A), dev(B), dev(bias)
    for algo, tol in ((L.GEMM_3XBF16, 1e-5), (L.GEMM_TF32X, 5e-6), (L.GEMM_3XTF32, 5e-6),
                      (L.GEMM_1XTF32, 3e-3)):
        C = P.zeros((M, N))
        L.call("b2_gemm", ta, tb, M, N, K, At.data_ptr, A.shape[1], Bt.data_ptr, B.shape[1],
               C.data_ptr, N, bt.data_ptr, L.EPI_BIAS_RELU, algo, None)
        assert normwise(host(C), ref) <= tol, (algo, ta, tb)


@pytest.mark.parametrize("shape", [(3072, 1792, 4096), (3000, 1800, 4096), (4096, 4096, 16384)])
def test_gemm_tail_wave_k_slices(shape):
    """More tiles than one wave: whole waves run whole tiles, the partial
    last wave splits its tiles into K slices (k_tail_epilogue sums them in
    slice order). Against fp64 for every layout and scheme, ragged edges
    included, with bias + ReLU in the second stage."""
    M, N, K = shape
    rng = np.random.default_rng(M + N)
    bias = dev(rng.uniform(-1, 1, N).astype(np.float32))
    bh = host(bias).astype(np.float64)
    for ta, tb in ((0, 1), (0, 0), (1, 0)):
        A = rng.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
        B = rng.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
        ref = np.maximum(_ref_gemm(A, B, ta, tb) + bh, 0)
        At, Bt = dev(A), dev(B)
        for algo, tol in ((L.GEMM_3XBF16, 1e-5), (L.GEMM_TF32X, 5e-6)):
            C = P.zeros((M, N))
            L.call("b2_gemm", ta, tb, M, N, K, At.data_ptr, A.shape[1], Bt.data_ptr, B.shape[1],
                   C.data_ptr, N, bias.data_ptr, L.EPI_BIAS_RELU, algo, None)
            assert normwise(host(C), ref) <= tol, (algo, ta, tb)
        del A, B, At, Bt


def test_gemm_split_k_fused_epilogue_mask_and_emission():
    """Split-K second stage applies the ReLU-pullback mask and emits C's own
    3xBF16 split exactly like the single-pass epilogue."""
    from paper_2602_00125_b200 import _lib as L
    from paper_2602_00125_b200.core import Buffer

    M, N, K = 256, 256, 16384
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    mask = (rng.uniform(-1, 1, (M, N)) > 0).astype(np.float32)
    At, Bt, mt = dev(A), dev(B), dev(mask)
    ah, al, bh, bl = (Buffer(2 * M * K), Buffer(2 * M * K), Buffer(2 * N * K), Buffer(2 * N * K))
    L.call("b2_bf16x3_split", ah.ptr, al.ptr, At.data_ptr, M, K, K, None)
    L.call("b2_bf16x3_split", bh.ptr, bl.ptr, Bt.data_ptr, N, K, K, None)
    C = P.zeros((M, N))
    ch, cl = Buffer(2 * M * N), Buffer(2 * M * N)
    L.call("b2_gemm_3xbf16", 0, 1, M, N, K, ah.ptr, al.ptr, bh.ptr, bl.ptr, C.data_ptr, N, None,
           L.EPI_NONE, mt.data_ptr, ch.ptr, cl.ptr, None, None)
    got = host(C)
    assert normwise(got, _ref_gemm(A, B, 0, 1) * mask) <= 1e-5
    hi = _bf16_rn(got)
    lo = _bf16_rn((got - hi).astype(np.float32))
    assert bits_equal(_bf16_bits(ch.ptr, M * N).reshape(M, N), hi)
    assert bits_equal(_bf16_bits(cl.ptr, M * N).reshape(M, N), lo)


def test_gemm_accuracy_long_k():
    """K-chunk promotion keeps 3xTF32 at sgemm accuracy for the config-3 K."""
    from paper_2602_00125_b200 import _lib as L

    M, N, K = 256, 256, 8192
    rng = np.random.default_rng(8)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    At, Bt = dev(A), dev(B)
    for algo, tol in ((L.GEMM_3XTF32, 3e-6), (L.GEMM_TF32X, 3e-6), (L.GEMM_3XBF16, 8e-6)):
        C = P.zeros((M, N))
        L.call("b2_gemm", 0, 1, M, N, K, At.data_ptr, K, Bt.data_ptr, K, C.data_ptr, N, None,
               L.EPI_NONE, algo, None)
        assert normwise(host(C), ref) <= tol, algo


def test_tf32_hardware_rounding_probe(capsys):
    """Records how kind::tf32 consumes raw fp32 bits (informational)."""
    from paper_2602_00125_b200 import _lib as L

    M, N, K = 128, 256, 32
    a = np.full((M, K), 1.0 + 2.0 ** -11 + 2.0 ** -20, np.float32)
    b = np.zeros((N, K), np.float32)
    b[:, 0] = 1.0
    At, Bt = dev(a), dev(b)
    C = P.zeros((M, N))
    L.call("b2_gemm", 0, 1, M, N, K, At.data_ptr, K, Bt.data_ptr, K, C.data_ptr, N, None,
           L.EPI_NONE, L.GEMM_1XTF32, None)
    v = float(host(C)[0, 0])
    mode = {1.0: "truncate", 1.0 + 2.0 ** -10: "round"}.get(v, f"other({v!r})")
    with capsys.disabled():
        print(f"\n[tf32 probe] raw fp32 1+2^-11+2^-20 consumed as {v!r} -> {mode}")


# ---------------------------------------------------------------- losses


def test_cross_entropy_goldens_bit_exact():
    g = load("ce_optim.npz")
    for i, (z, labels) in enumerate(I.ce_cases()):
        P.reset_tape()
        zt = dev(z, True)
        loss = nn.cross_entropy(zt, labels)
        store = P.backward(loss)
        assert bits_equal(host(loss), g[f"ce{i}_loss"]), i
        assert bits_equal(host(store[zt]), g[f"ce{i}_grad"]), i


def test_cross_entropy_label_validation():
    z = P.zeros((2, 3))
    with pytest.raises(ValueError):
        nn.cross_entropy(z, [0, 3])
    with pytest.raises(P.ShapeError):
        nn.cross_entropy(z, [0])


@pytest.mark.parametrize("cols", [1024, 1000, 2048, 64, 130, 3000])
def test_softmax_matches_composed_reference_bit_exact(cols):
    """Register-resident row kernels (cols % 4 == 0, <= 2048) and the looped
    ones (other widths), incl. a NaN first slot and -inf entries."""
    rng = np.random.default_rng(4 + cols)
    z = (rng.standard_normal((33, cols)) * 3).astype(np.float32)
    z[3, 0] = np.nan
    z[5, 7] = np.nan
    z[6, :] = -np.inf
    z[6, 1] = 0.0
    gy = rng.standard_normal((33, cols)).astype(np.float32)
    zt = dev(z, True)
    y = P.softmax(zt)
    yo, e, s = O.softmax_rows_composed(z)
    assert bits_equal(host(y), yo)
    store = P.backward(y, seed=dev(gy))
    assert bits_equal(host(store[zt]), O.softmax_backward_composed(gy, e, s))


# ---------------------------------------------------------------- optimizers


@pytest.mark.parametrize("name,ctor", [
    ("sgd", lambda: optim.SGD(lr=0.01)),
    ("sgd_mom_wd", lambda: optim.SGD(lr=0.05, momentum=0.9, weight_decay=0.01)),
    ("adam", lambda: optim.Adam(lr=1e-3)),
    ("adam_wd", lambda: optim.Adam(lr=3e-3, betas=(0.8, 0.99), eps=1e-6, weight_decay=0.1)),
])
def test_optimizer_sequences_bit_exact(name, ctor):
    g = load("ce_optim.npz")
    opt = ctor()
    p = dev(g["opt_theta0"])
    for k in range(4):
        opt.step(p, dev(g["opt_grads"][k]))
        assert bits_equal(host(p), g[f"opt_{name}"][k]), (name, k)


def test_multi_tensor_step_matches_single_steps():
    rng = np.random.default_rng(9)
    shapes = [(300, 7), (1,), (8193,), (64, 65)]
    ps = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    gs = [rng.standard_normal(s).astype(np.float32) for s in shapes]
    a, b = optim.Adam(lr=1e-2), optim.Adam(lr=1e-2)
    pa = [dev(p) for p in ps]
    pb = [dev(p) for p in ps]
    for _ in range(3):
        a.step_many([(p, dev(gg)) for p, gg in zip(pa, gs)])
        for p, gg in zip(pb, gs):
            b.step(p, dev(gg))
    for x, y in zip(pa, pb):
        assert bits_equal(host(x), host(y))


# ---------------------------------------------------------------- BASELINE configs (small)


def _mlp_device(params, relu_between=True):
    layers = []
    for i, (w, b) in enumerate(params):
        d = nn.Dense(w.shape[1], w.shape[0], rng=0)
        d.weight.write_flat(w.ravel())
        d.bias.write_flat(b.ravel())
        layers.append(d)
        if relu_between and i < len(params) - 1:
            layers.append(nn.ReLU())
    return nn.Sequential(*layers), [l for l in layers if isinstance(l, nn.Dense)]


def _run_mlp_device(params, x, labels, opt, steps):
    model, dense = _mlp_device(params)
    xt = dev(x)
    losses = []
    for _ in range(steps):
        P.reset_tape()
        loss = nn.cross_entropy(model(xt), labels)
        losses.append(loss.item())
        store = P.backward(loss)
        grads = [(host(store[d.weight]), host(store[d.bias])) for d in dense]
        optim.step_all(opt, model.parameters(), store)
    return np.array(losses, np.float32), grads, [(host(d.weight), host(d.bias)) for d in dense]


def test_config1_train_step_reference_arithmetic_bit_exact():
    """With the reference's GEMM arithmetic ('ref') every kernel of the
    config-1 step reproduces the reference's bits: loss, all 4 gradients and
    the SGD-updated parameters equal the goldens made by running it."""
    golden = load("config1.npz")
    params, x, labels = I.config1_inputs()
    P.set_gemm_algo("ref")
    try:
        losses, grads, newp = _run_mlp_device(params, x, labels, optim.SGD(lr=0.01), 1)
    finally:
        P.set_gemm_algo(None)
    assert bits_equal(losses, golden["loss"])
    for i, ((gw, gb), (w, b)) in enumerate(zip(grads, newp)):
        for got, key in ((gw, "gw"), (gb, "gb"), (w, "w"), (b, "b")):
            assert bits_equal(got, golden[f"{key}{i}"]), (key, i)


def test_config5_small_adam_reference_arithmetic_bit_exact():
    """3 Adam steps of the config-5-shaped MLP in the 'ref' GEMM mode: losses,
    last gradients and parameters bit-identical to the reference's goldens."""
    golden = load("config5_small.npz")
    params, x, labels = I.config5_inputs(width=64, classes=10, batch=32, depth=4)
    P.set_gemm_algo("ref")
    try:
        losses, grads, newp = _run_mlp_device(params, x, labels, optim.Adam(lr=1e-3), 3)
    finally:
        P.set_gemm_algo(None)
    assert bits_equal(losses, golden["loss"])
    for i, ((gw, gb), (w, b)) in enumerate(zip(grads, newp)):
        assert bits_equal(gw, golden[f"gw{i}"]), i
        assert bits_equal(w, golden[f"w{i}"]), i


@pytest.mark.parametrize("algo", ["simt", "3xtf32", "tf32x", "3xbf16"])
def test_config1_train_step(algo):
    golden = load("config1.npz")
    params, x, labels = I.config1_inputs()
    P.set_gemm_algo(algo)
    try:
        losses, grads, newp = _run_mlp_device(params, x, labels, optim.SGD(lr=0.01), 1)
    finally:
        P.set_gemm_algo(None)
    assert normwise(losses, golden["loss"]) <= TOL
    for i, ((gw, gb), (w, b)) in enumerate(zip(grads, newp)):
        assert normwise(gw, golden[f"gw{i}"]) <= TOL, i
        assert normwise(gb, golden[f"gb{i}"]) <= TOL, i
        assert normwise(w, golden[f"w{i}"]) <= TOL, i
        assert normwise(b, golden[f"b{i}"]) <= TOL, i


def test_config5_small_adam_3_steps():
    golden = load("config5_small.npz")
    params, x, labels = I.config5_inputs(width=64, classes=10, batch=32, depth=4)
    losses, grads, newp = _run_mlp_device(params, x, labels, optim.Adam(lr=1e-3), 3)
    assert normwise(losses, golden["loss"]) <= TOL
    for i, ((gw, gb), (w, b)) in enumerate(zip(grads, newp)):
        assert normwise(gw, golden[f"gw{i}"]) <= TOL, i
        assert normwise(w, golden[f"w{i}"]) <= TOL, i


@pytest.mark.parametrize("algo", ["tf32x", "3xbf16"])
def test_config5_shape_tensor_core_step(algo):
    """Config-5 structure at a width where every GEMM runs on tcgen05 (fused
    bias/relu epilogues, masked x_bar, emitted operand splits): forward
    activations and loss against the fp64-accumulating oracle at the fp32
    tolerance 1e-4; gradients against the oracle's backward conditioned on the
    device's relu pattern (see _conditioned_step) at 1e-4, with the relu
    pattern itself agreeing with the oracle's on all but <= 1e-4 of entries."""
    params, x, labels = I.config5_inputs(width=256, classes=16, batch=256, depth=3)
    P.set_gemm_algo(algo)
    try:
        losses, grads, _ = _run_mlp_device(params, x, labels, optim.SGD(lr=0.0), 1)
        acts = _device_forward(params, x)
    finally:
        P.set_gemm_algo(None)
    ref = O.mlp_train_step(params, x, labels, O.SGD(lr=0.0))
    assert normwise(losses, np.float32(ref["loss"])) <= TOL
    assert normwise(acts[-1], ref["logits"]) <= TOL
    z, cgrads = _conditioned_step(params, acts, labels, _mm64)
    n = len(params)
    flips = total = 0
    for i in range(n):
        want = O.relu(z[i]) if i < n - 1 else z[i]
        assert normwise(acts[i + 1], want) <= TOL, (algo, i)
        if i < n - 1:
            flips += int(np.count_nonzero((acts[i + 1] > 0) != (z[i] > 0)))
            total += z[i].size
    assert flips <= max(1, total // 10000), flips
    for i, ((gw, gb), (cw, cb)) in enumerate(zip(grads, cgrads)):
        assert normwise(gw, cw) <= TOL, (algo, i)
        assert normwise(gb, cb) <= TOL, (algo, i)


def test_config2_small_bit_exact_composed_and_fused():
    g = load("config2_small.npz")
    a, b = I.config2_inputs(rows=256, cols=512)
    # composed reference ops
    P.reset_tape()
    at, bt = dev(a, True), dev(b, True)
    y = P.relu(P.add(P.mul(at, bt), bt))
    assert bits_equal(host(y), g["y"])
    assert bits_equal(host(P.exp(P.clamp(dev(a), -10, 10))), g["e"])
    with P.no_grad():
        for d in (0, 1):
            assert bits_equal(host(P.sum(y, axis=d)), g[f"sum{d}"]), d
            assert bits_equal(host(P.mean(y, axis=d)), g[f"mean{d}"]), d
            assert bits_equal(host(P.max(y, axis=d)), g[f"max{d}"]), d
        assert bits_equal(host(P.sum(y)), g["sum_all"])
    store = P.backward(P.sum(y))
    assert bits_equal(host(store[at]), g["grad_a"])
    assert bits_equal(host(store[bt]), g["grad_b"])
    # fused kernels
    P.reset_tape()
    at, bt = dev(a, True), dev(b, True)
    yf = P.fused_muladd_relu(at, bt)
    assert bits_equal(host(yf), g["y"])
    store = P.backward(P.sum(yf))
    assert bits_equal(host(store[at]), g["grad_a"])
    assert bits_equal(host(store[bt]), g["grad_b"])
    ga, gb = P.muladd_relu_sum_grads(dev(a), dev(b))
    assert bits_equal(host(ga), g["grad_a"]) and bits_equal(host(gb), g["grad_b"])


@pytest.mark.parametrize("algo", ["tf32x", "3xbf16"])
def test_config3_small_matmul_fwd_bwd(algo):
    g = load("config3_small.npz")
    A, B, dC = I.config3_inputs(n=96)
    P.set_gemm_algo(algo)
    try:
        at, bt = dev(A, True), dev(B, True)
        C = P.mm(at, bt)
        store = P.backward(C, seed=dev(dC))
    finally:
        P.set_gemm_algo(None)
    assert normwise(host(C), g["C"]) <= TOL
    assert normwise(host(store[at]), g["dA"]) <= TOL
    assert normwise(host(store[bt]), g["dB"]) <= TOL


def test_config4_small_softmax_linear():
    g = load("config4_small.npz")
    X, W, bias, Tt = I.config4_inputs(b=2, s=16, k=64)
    xt, wt, bt = dev(X, True), dev(W, True), dev(bias, True)
    z = P.add(P.mm(xt, wt), bt)
    Y = P.softmax(z)
    loss = P.mean(P.mul(Y, dev(Tt)))
    store = P.backward(loss)
    assert normwise(host(loss), g["loss"]) <= TOL
    assert normwise(host(Y).reshape(-1, 64), g["Y"]) <= TOL
    assert normwise(host(store[xt]).reshape(-1, 64), g["dX"]) <= TOL
    assert normwise(host(store[wt]), g["dW"]) <= TOL
    assert normwise(host(store[bt]), g["dbias"]) <= TOL


# ---------------------------------------------------------------- autograd contract


def test_autograd_contract_on_device():
    x = dev([3.0], True)
    assert host(P.backward(P.sum(P.add(x, x)))[x]).tolist() == [2.0]
    P.reset_tape()
    x = dev([1.0, 2.0, 3.0], True)
    y = dev([[1.0], [2.0]], True)
    s = P.backward(P.sum(P.mul(x, y)))
    assert s[x].shape == (3,) and host(s[x]).tolist() == [3.0, 3.0, 3.0]
    assert s[y].shape == (2, 1) and host(s[y]).tolist() == [[6.0], [6.0]]
    P.reset_tape()
    x = dev([[1.0, 7.0, 7.0]], True)
    assert host(P.backward(P.sum(P.max(x, axis=1)))[x]).tolist() == [[0.0, 1.0, 0.0]]
    P.reset_tape()
    x = dev([[1.0, 2.0], [3.0, 4.0]], True)
    yv = P.reshape(P.transpose2d(x), (4,))
    assert host(P.backward(P.sum(P.mul(yv, yv)))[x]).tolist() == [[2.0, 4.0], [6.0, 8.0]]
    P.reset_tape()
    x = dev([1.0, 2.0, 3.0, 4.0], True)
    assert host(P.backward(P.mean(x))[x]).tolist() == [0.25] * 4


def test_mutation_guard():
    x = dev([1.0, 2.0], True)
    y = P.mul(x, x)
    x.write_flat([5.0, 6.0])
    with pytest.raises(P.GradError):
        P.backward(P.sum(y))


def test_allocator_reuses_blocks_and_counts_launches():
    from paper_2602_00125_b200 import _lib as L

    t = P.add(P.ones((1024, 1024)), 1.0)
    del t
    n0 = L.launch_count()
    m0 = L.alloc_stats()["cuda_mallocs"]
    for _ in range(20):
        t = P.add(P.ones((1024, 1024)), 1.0)
        del t
    assert L.launch_count() - n0 >= 40
    assert L.alloc_stats()["cuda_mallocs"] - m0 == 0  # every block came from the cache


def test_train_steps_do_not_leak_device_memory():
    from paper_2602_00125_b200 import _lib as L
    from paper_2602_00125_b200.data import build_mlp, mlp_config5

    model = build_mlp(mlp_config5(0, width=256, classes=10, depth=2))
    opt = optim.Adam(lr=1e-3)
    x = dev(np.random.default_rng(0).standard_normal((512, 256)))
    labels = np.arange(512) % 10
    use = []
    for _ in range(6):
        P.reset_tape()
        loss = nn.cross_entropy(model(x), labels)
        optim.step_all(opt, model.parameters(), P.backward(loss))
        L.synchronize()
        use.append(L.alloc_stats()["in_use"])
    assert use[-1] == use[-3] and use[-2] == use[-4], use  # steady state, no growth


def test_smoke_entry_point():
    import __graft_entry__

    __graft_entry__.smoke()


def test_cuda_graph_replay_matches_eager_config1():
    from paper_2602_00125_b200 import graph
    from paper_2602_00125_b200.data import build_mlp

    params, x, labels = I.config1_inputs()
    xs = dev(x)
    lab = nn.labels_buffer(labels)

    def make():
        return build_mlp([(w.copy(), b.copy()) for w, b in params])

    eager = make()
    opt_e = optim.SGD(lr=0.01)
    for _ in range(3):
        P.reset_tape()
        loss = nn.cross_entropy(eager(xs), lab)
        optim.step_all(opt_e, eager.parameters(), P.backward(loss))

    model = make()
    opt_g = optim.SGD(lr=0.01)

    def step():
        P.reset_tape()
        loss = nn.cross_entropy(model(xs), lab)
        optim.step_all(opt_g, model.parameters(), P.backward(loss))
        return loss

    g = graph.capture(step, warmup=1)   # 1 eager step
    g.replay()
    g.replay()                          # + 2 replayed steps
    for pe, pg in zip(eager.parameters(), model.parameters()):
        assert bits_equal(host(pe), host(pg))
    assert np.isfinite(g.outputs.item())


def test_exp_matches_double_exp_on_wide_range():
    rng = np.random.default_rng(12)
    x = np.concatenate([rng.uniform(-110, 100, 1 << 20), rng.standard_normal(1 << 18) * 3,
                        np.array([0.0, -0.0, 88.72, 88.73, -87.3, -103.9, -104.0, np.inf,
                                  -np.inf, np.nan])]).astype(np.float32)
    got = host(P.exp(dev(x)))
    want = O.exp(x)
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    diff = got[~nan].view(np.int32).astype(np.int64) - want[~nan].view(np.int32).astype(np.int64)
    assert np.abs(diff).max() <= 1 and np.count_nonzero(diff) <= 2, np.count_nonzero(diff)


def test_nccl_gradient_path_single_rank_matches_plain_step():
    """The N>1 data-parallel code path (NCCL uid exchange, comm stream,
    overlapped in-place ncclAvg, optimizer waiting on the comm stream) with a
    1-rank communicator: averaging over one rank is the identity, so the
    parameters must match a plain step bit for bit."""
    from paper_2602_00125_b200 import dist
    from paper_2602_00125_b200.data import build_mlp, mlp_config5

    params = mlp_config5(0, width=256, classes=10, depth=2)
    x = dev(np.random.default_rng(1).standard_normal((512, 256)))
    lab = nn.labels_buffer(np.arange(512) % 10)
    comm = dist.Communicator(dist.Env(), force_nccl=True)
    assert comm.active

    def run(use_comm):
        model = build_mlp([(w.copy(), b.copy()) for w, b in params])
        opt = optim.Adam(lr=1e-3)
        for _ in range(2):
            P.reset_tape()
            loss = nn.cross_entropy(model(x), lab, denom=512)
            red = dist.GradReducer(comm if use_comm else dist.Communicator(dist.Env()))
            store = P.backward(loss, on_leaf_ready=red.hook)
            red.finish()
            optim.step_all(opt, model.parameters(), store)
        return [host(p) for p in model.parameters()]

    for a, b in zip(run(True), run(False)):
        assert bits_equal(a, b)
    assert comm.max_scalar(3.5) == 3.5
    comm.barrier()


def test_c_abi_rejects_bad_arguments_loudly():
    """The boundary validates before launching: misaligned split outputs, a
    bias epilogue without a bias, bad enums -- non-zero status + message."""
    import ctypes

    from paper_2602_00125_b200 import _lib as L
    from paper_2602_00125_b200.core import Buffer

    lib = L.lib()
    M = N = K = 128
    a, b = Buffer(2 * M * K), Buffer(2 * N * K)
    c, hi, lo = P.zeros((M, N)), Buffer(2 * M * N + 64), Buffer(2 * M * N + 64)
    rc = lib.b2_gemm_3xbf16(0, 1, M, N, K, a.ptr, a.ptr, b.ptr, b.ptr, c.data_ptr, N, None, 0,
                            None, hi.ptr + 2, lo.ptr, None, None)
    assert rc != 0 and b"aligned" in lib.b2_last_error()
    x = P.zeros((M, K))
    rc = lib.b2_gemm(0, 1, M, N, K, x.data_ptr, K, x.data_ptr, K, c.data_ptr, N, None,
                     L.EPI_BIAS, L.GEMM_SIMT, None)
    assert rc != 0 and b"bias" in lib.b2_last_error()
    rc = lib.b2_unary(99, c.data_ptr, 2, L.i64s((M, N)), c.data_ptr, L.i64s((N, 1)), 0.0, 0.0, None)
    assert rc != 0
    with pytest.raises(RuntimeError):
        L.call("b2_reduce", 7, c.data_ptr, None, 2, L.i64s((M, N)), c.data_ptr, L.i64s((N, 1)), 1, None)


def test_beyond_2_31_elements_int64_indexing():
    """Maximum-size edge: a tensor of 2^31 + 5 elements (8 GiB) through the
    flat elementwise kernel, a full fp64 sum and a column sum -- every index
    path is 64-bit. Size-independent properties: exact values of constant
    fills and of their sums."""
    n = 2 ** 31 + 5
    x = P.full((n,), 1.5)
    y = P.add(x, 2.25)  # 3.75 exactly
    assert P.sum(y).item() == np.float32(n * 3.75)
    last = P.Tensor(y.buffer, (5,), offset=n - 5)  # a view of the last elements (offset > 2^31)
    assert np.all(last.numpy() == np.float32(3.75))
    del x, y, last
    m = P.full((2 ** 20 + 3, 2048), 0.5)  # 2^31 + 6144 elements, column sums
    cs = P.sum(m, axis=0).numpy()
    assert np.all(cs == np.float32((2 ** 20 + 3) * 0.5))
    with pytest.raises(RuntimeError):
        P.max(P.reshape(m, (-1,)))  # max over >= 2^31 elements per output is rejected loudly


@pytest.mark.parametrize("algo", ["3xbf16", "tf32x", "bf16"])
@pytest.mark.parametrize("shape", [(1000, 520, 256), (65536 // 16, 4096 // 8, 512), (256, 256, 16384),
                                   (3000, 1800, 4096)])
def test_gemm_fused_column_sums_match_the_reduction(algo, shape):
    """The epilogue's column sums (the lower layer's bias gradient) equal the
    reduction engine's sum over axis 0 of the stored, masked output -- bit
    for bit (both are one f32 rounding of an fp64 sum); split-K shapes fall
    back to the reduction."""
    from paper_2602_00125_b200 import core as C

    M, N, K = shape
    rng = np.random.default_rng(M + N + K)
    x = dev(rng.standard_normal((M, K)).astype(np.float32))
    w = dev((rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32))
    mask = dev((rng.uniform(-1, 1, (M, N)) > 0).astype(np.float32))
    # compare against the fp32 C the epilogue stored (a split-only output is
    # materialised from its split, within 2^-16: test_gpu_lazy_fp32.py)
    lazy, C._LAZY_FP32 = C._LAZY_FP32, False
    out = P.zeros((M, N))
    cs = P.zeros((N,))
    P.set_gemm_algo(algo)
    try:
        C._gemm_into(out, x, w, mask=mask, emit_split=True, colsum=cs)
    finally:
        P.set_gemm_algo(None)
        C._LAZY_FP32 = lazy
    assert bits_equal(cs.numpy(), P.sum(out, axis=0).numpy())
    assert np.all(out.numpy()[mask.numpy() == 0] == 0)


def _pack_bits(y):
    """y > 0 as [M][ceil(N/64)] little-endian uint64 words (bit j of word w =
    column 64 w + j) -- the layout b2_gemm_fused's relu_bits_out writes."""
    M, N = y.shape
    W = (N + 63) // 64
    b = np.zeros((M, W * 64), np.uint8)
    b[:, :N] = y > 0
    return np.packbits(b.reshape(M, W, 64), axis=2, bitorder="little").view(np.uint64).reshape(M, W)


def _read_words(buf, M, W):
    import ctypes

    out = np.empty((M, W), np.uint64)
    L.call("b2_memcpy_d2h", out.ctypes.data_as(ctypes.c_void_p), buf.ptr, out.nbytes, None)
    return out


@pytest.mark.parametrize("algo", ["3xbf16", "tf32x", "bf16"])
@pytest.mark.parametrize("shape", [(1000, 520, 256), (4096, 512, 512), (256, 256, 16384), (300, 72, 64),
                                   (3000, 1800, 4096)])
def test_gemm_relu_bits_and_bitmask_pullback(algo, shape):
    """Forward: relu_bits_out records exactly y > 0 of the stored output.
    Backward: the pullback read from those bits gives the same bits as the
    fp32-mask pullback -- output, emitted split and fused column sums -- also
    on long-K shapes (split-K's second stage reads and writes the bits too)."""
    from paper_2602_00125_b200 import core as C

    M, N, K = shape
    rng = np.random.default_rng(M * 7 + N + K)
    x = dev(rng.standard_normal((M, K)).astype(np.float32))
    w = dev((rng.standard_normal((N, K)) / np.sqrt(K)).astype(np.float32))
    bias = dev(rng.standard_normal(N).astype(np.float32) * 0.1)
    g = dev(rng.standard_normal((M, K)).astype(np.float32))
    y = P.zeros((M, N))
    bits = P.Buffer(8 * M * ((N + 63) // 64))
    P.set_gemm_algo(algo)
    try:
        assert C._gemm_into(y, x, w, bias, L.EPI_BIAS_RELU, bits_out=bits)
        yv = y.numpy()
        assert np.array_equal(_read_words(bits, M, (N + 63) // 64), _pack_bits(yv))
        # dX of the layer above: [M,K] . [K,N] masked by y > 0
        wt = dev((rng.standard_normal((K, N)) / np.sqrt(K)).astype(np.float32))
        outs = []
        for mb in (None, bits):
            out, cs = P.zeros((M, N)), P.zeros((N,))
            C._gemm_into(out, g, P.transpose2d(wt), mask=y, emit_split=True, colsum=cs, mask_bits=mb)
            outs.append((out.numpy(), cs.numpy(), out.buffer._splits))
    finally:
        P.set_gemm_algo(None)
    (o0, c0, s0), (o1, c1, s1) = outs
    assert bits_equal(o0, o1) and bits_equal(c0, c1)
    assert np.all(o1[yv == 0] == 0)
    k0, k1 = next(iter(s0.values())), next(iter(s1.values()))
    n = 2 * M * N
    for a, b in zip(k0[1:3], k1[1:3]):
        if a is not None:
            assert np.array_equal(_read_bytes(a, n), _read_bytes(b, n))


def _read_bytes(buf, n):
    import ctypes

    out = np.empty(n, np.uint8)
    L.call("b2_memcpy_d2h", out.ctypes.data_as(ctypes.c_void_p), buf.ptr, n, None)
    return out


def test_mlp_relu_bits_path_matches_the_fp32_mask_path():
    """A Dense+ReLU chain trained one step with the bitmask pullback (default)
    and with the fp32-mask pullback (B2_RELU_BITS=0) is bit-identical."""
    from paper_2602_00125_b200 import core as C

    rng = np.random.default_rng(81)
    x = rng.standard_normal((2048, 256)).astype(np.float32)
    labels = nn.labels_buffer(rng.integers(0, 16, 2048))
    res = []
    for on in (True, False):
        C._RELU_BITS_ON = on
        model = nn.Sequential(nn.Dense(256, 512, rng=1), nn.ReLU(), nn.Dense(512, 384, rng=2),
                              nn.ReLU(), nn.Dense(384, 16, rng=3))
        P.set_gemm_algo("3xbf16")
        try:
            P.reset_tape()
            store = P.backward(nn.cross_entropy(model(dev(x)), labels))
            if on:
                assert len(C._RELU_BITS) >= 2
        finally:
            P.set_gemm_algo(None)
            C._RELU_BITS_ON = True
        res.append(np.concatenate([store[p].numpy().ravel() for p in model.parameters()]))
    assert bits_equal(res[0], res[1])


def test_mlp_bias_gradients_use_the_fused_column_sums():
    """Dense+ReLU chain: the hidden layers' bias gradients come from the x_bar
    GEMM epilogue and equal the separate reduction of the same cotangent."""
    from paper_2602_00125_b200 import core as C

    rng = np.random.default_rng(8)
    model = nn.Sequential(nn.Dense(256, 512, rng=1), nn.ReLU(), nn.Dense(512, 512, rng=2), nn.ReLU(),
                          nn.Dense(512, 16, rng=3))
    x = dev(rng.standard_normal((1024, 256)).astype(np.float32))
    labels = nn.labels_buffer(rng.integers(0, 16, 1024))
    P.set_gemm_algo("3xbf16")
    try:
        P.reset_tape()
        store = P.backward(nn.cross_entropy(model(x), labels))
    finally:
        P.set_gemm_algo(None)
    fused = [t for t in C._COLSUM.values()]
    assert len(fused) >= 1
    dense = [l for l in model.layers if isinstance(l, nn.Dense)]
    for d in dense[:2]:
        gb = store[d.bias].numpy()
        assert np.isfinite(gb).all() and np.abs(gb).sum() > 0


def test_softmax_row_constant_division_exact_at_scale():
    """The row kernels divide by the row sum with a reciprocal + Markstein
    correction; over 4M elements with e spanning 1 .. subnormal .. 0 and
    cotangents spanning 1e-30 .. 1e30 the results stay bit-identical to the
    composed reference (IEEE divisions)."""
    rng = np.random.default_rng(17)
    z = (rng.standard_normal((4096, 1024)) * 20).astype(np.float32)
    gy = (rng.standard_normal((4096, 1024)) * 10.0 ** rng.uniform(-30, 30, (4096, 1024))).astype(np.float32)
    zt = dev(z, True)
    P.reset_tape()
    y = P.softmax(zt)
    yo, e, s = O.softmax_rows_composed(z)
    assert bits_equal(host(y), yo)
    store = P.backward(y, seed=dev(gy))
    assert bits_equal(host(store[zt]), O.softmax_backward_composed(gy, e, s))


@pytest.mark.parametrize("force_nccl,shard", [(False, False), (True, False), (True, True)])
def test_optimizer_overlapped_in_backward_matches_plain_step(force_nccl, shard):
    """GradReducer(optimizer=...) launches each layer's Adam update on a side
    stream as soon as its gradient is final (after its all-reduce with NCCL):
    three steps give bit-identical parameters to backward-then-step_all. With
    shard=True the update runs as reduce-scatter -> Adam on the rank's shard
    -> all-gather (NCCL, here one rank: the whole tensor is the shard)."""
    from paper_2602_00125_b200 import dist
    from paper_2602_00125_b200.data import build_mlp, mlp_config5

    params0 = mlp_config5(0, width=256, classes=10, depth=3)
    x = dev(np.random.default_rng(4).standard_normal((512, 256)))
    lab = nn.labels_buffer(np.arange(512) % 10)
    comm = dist.Communicator(dist.Env(), force_nccl=force_nccl)

    def run(overlap):
        model = build_mlp([(w.copy(), b.copy()) for w, b in params0])
        ps = model.parameters()
        opt = optim.Adam(lr=1e-3)
        for _ in range(3):
            P.reset_tape()
            loss = nn.cross_entropy(model(x), lab, denom=512)
            red = dist.GradReducer(comm, ps, optimizer=opt if overlap else None,
                                   shard=shard if overlap else False)
            store = P.backward(loss, on_leaf_ready=red.hook)
            red.finish()
            if overlap:
                assert red.step_rest(store) == 0
            else:
                optim.step_all(opt, ps, store)
        return [host(p) for p in ps]

    for a, b in zip(run(True), run(False)):
        assert bits_equal(a, b)


def test_comm_sm_reserve_only_while_collectives_overlap(monkeypatch):
    """With B2_COMM_SMS (default 8 for world > 1) the backward GEMMs queued
    after the first leaf-ready hook leave that many SMs to the collectives and
    the optimizer; finish() gives them back. Parameters stay within 1e-5 of
    the plain step (a smaller persistent grid may split K differently)."""
    import ctypes

    from paper_2602_00125_b200 import dist
    from paper_2602_00125_b200.data import build_mlp, mlp_config5

    monkeypatch.setenv("B2_COMM_SMS", "8")
    comm = dist.Communicator(dist.Env(), force_nccl=True)
    assert comm.sm_reserve == 8

    def reserve():
        v = ctypes.c_int(-1)
        L.check(L.lib().b2_gemm_get_sm_reserve(ctypes.byref(v)))
        return v.value

    params0 = mlp_config5(0, width=512, classes=10, depth=3)
    x = dev(np.random.default_rng(5).standard_normal((2048, 512)))
    lab = nn.labels_buffer(np.arange(2048) % 10)
    seen = []

    def run(overlap):
        model = build_mlp([(w.copy(), b.copy()) for w, b in params0])
        ps = model.parameters()
        opt = optim.SGD(lr=0.1)  # (Adam's first step is lr * sign(g): rounding-sensitive near g = 0)
        P.reset_tape()
        loss = nn.cross_entropy(model(x), lab, denom=2048)
        if overlap:
            red = dist.GradReducer(comm, ps, optimizer=opt)

            def hook(nid, g):
                r = red.hook(nid, g)
                seen.append(reserve())
                return r

            store = P.backward(loss, on_leaf_ready=hook)
            red.finish()
            red.step_rest(store)
        else:
            optim.step_all(opt, ps, P.backward(loss))
        return [host(p) for p in ps]

    got, want = run(True), run(False)
    assert seen and all(v == 8 for v in seen) and reserve() == 0
    for a, b in zip(got, want):
        assert normwise(a, b) <= 1e-5


# ---------------------------------------------------------------- fused config-4 loss


def _config4_step(X, W, bias, T, fused):
    K = X.shape[-1]
    P.reset_tape()
    xt, wt, bt = dev(X, True), dev(W, True), dev(bias, True)
    if fused:
        z = P.linear(P.reshape(xt, (-1, K)), P.transpose2d(wt), bt)
        loss = P.softmax_mul_mean(z, dev(T.reshape(-1, K)))
    else:
        loss = P.mean(P.mul(P.softmax(P.add(P.mm(xt, wt), bt)), dev(T)))
    store = P.backward(loss)
    return (host(loss), host(store[xt]).reshape(-1, K), host(store[wt]), host(store[bt]))


def test_config4_fused_loss_reference_arithmetic_bit_exact():
    """nn.Linear + softmax_mul_mean in the 'ref' GEMM mode reproduce the
    reference's bits for the config-4 step (loss, dX, dW, dbias)."""
    g = load("config4_small.npz")
    X, W, bias, Tt = I.config4_inputs(b=2, s=16, k=64)
    P.set_gemm_algo("ref")
    try:
        loss, dX, dW, db = _config4_step(X, W, bias, Tt, fused=True)
    finally:
        P.set_gemm_algo(None)
    assert bits_equal(loss, g["loss"])
    assert bits_equal(dX, g["dX"])
    assert bits_equal(dW, g["dW"])
    assert bits_equal(db, g["dbias"])


@pytest.mark.parametrize("algo", ["3xbf16", "simt"])
@pytest.mark.parametrize("shape", [(2, 16, 64), (8, 128, 1024), (4, 96, 1000)])
def test_config4_fused_loss_bit_identical_to_the_composition(algo, shape):
    """The fused loss (one row pass each way, split + column sums emitted by
    the backward) gives the composed ops' bits with the same GEMM scheme."""
    b, s, k = shape
    X, W, bias, Tt = I.config4_inputs(b=b, s=s, k=k)
    bias = np.random.default_rng(9).uniform(-0.1, 0.1, k).astype(np.float32)
    P.set_gemm_algo(algo)
    try:
        want = _config4_step(X, W, bias, Tt, fused=False)
        got = _config4_step(X, W, bias, Tt, fused=True)
    finally:
        P.set_gemm_algo(None)
    for name, a, w in zip(("loss", "dX", "dW", "dbias"), got, want):
        assert bits_equal(a, w), name


def test_fused_loss_under_cuda_graph_replay_rematerialises_split_outputs():
    """A graph whose backward emits a split-only cotangent: after every replay
    the fp32 view of that cotangent is recomputed from the fresh split."""
    from paper_2602_00125_b200 import graph

    rng = np.random.default_rng(4)
    X = rng.standard_normal((256, 512)).astype(np.float32)
    W = (rng.standard_normal((512, 512)) * 0.03).astype(np.float32)
    T = rng.uniform(0, 1, (256, 512)).astype(np.float32)
    xt, wt, tt = dev(X, True), dev(W, True), dev(T)
    keep = {}

    def step():
        P.reset_tape()
        z = P.linear(xt, wt)
        loss = P.softmax_mul_mean(z, tt)
        store = P.backward(loss)
        keep["gz"] = store[z]
        return loss

    P.set_gemm_algo("3xbf16")
    try:
        g = graph.capture(step, warmup=1)
        gz_eager = host(keep["gz"])  # the warm-up's gz was replaced by the capture's
        for k in range(2):
            xt.write_flat((X * (1.0 + 0.5 * k)).ravel())
            g.replay()
            got = host(keep["gz"])
            xt_ref = dev(X * (1.0 + 0.5 * k), True)
            P.reset_tape()
            zr = P.linear(xt_ref, wt)
            ref = host(P.backward(P.softmax_mul_mean(zr, tt))[zr])
            assert bits_equal(got, ref), k
    finally:
        P.set_gemm_algo(None)
    assert gz_eager.shape == (256, 512)


@pytest.mark.parametrize("shape", [(300, 1000), (129, 4100), (1, 4), (1024, 256), (8, 512)])
def test_single_pass_config2_matches_the_separate_ops(shape):
    """b2_muladd_relu_stats on ragged strips / row blocks, with NaN, +-inf and
    clamp-boundary inputs: bit-identical to the separate device ops and to
    the oracle."""
    R, C = shape
    rng = np.random.default_rng(R * 7 + C)
    a = (rng.standard_normal((R, C)) * 4).astype(np.float32)
    b = rng.uniform(-1, 1, (1, C)).astype(np.float32)
    flat = a.ravel()
    flat[rng.integers(0, flat.size, max(1, flat.size // 50))] = np.nan
    flat[rng.integers(0, flat.size, max(1, flat.size // 100))] = np.inf
    flat[rng.integers(0, flat.size, max(1, flat.size // 100))] = -10.0
    b[0, 0] = 0.0
    ref = O.broadcast_reduce_config(a, b)
    out = P.muladd_relu_stats(dev(a), dev(b))
    at, bt = dev(a), dev(b)
    with P.no_grad():
        y = P.fused_muladd_relu(at, bt)
        sep = {"y": y, "e": P.exp(P.clamp(at, -10.0, 10.0)), "sum_all": P.sum(y)}
        for d in (0, 1):
            sep[f"sum{d}"], sep[f"mean{d}"], sep[f"max{d}"] = P.sum(y, d), P.mean(y, d), P.max(y, d)
    sep["grad_a"], sep["grad_b"] = P.muladd_relu_sum_grads(at, bt)
    for k, v in sep.items():
        assert bits_equal(host(out[k]), host(v)), k
        assert bits_equal(host(out[k]), ref[k]), k


def test_gemm_simt_is_a_sequential_fp32_fma_chain():
    """The FP32 SIMT GEMM's FFMA2 halves are IEEE fmaf: every output equals the
    sequential chain acc = fmaf(a[k], b[k], acc), k = 0..K-1. The host chain
    forms a*b + acc in 80-bit long double (the 48-bit product is exact; the sum
    is exact unless the exponents are far apart) and rounds once to f32 per
    step, so only rare double-rounding cases may differ from a true fmaf."""
    from paper_2602_00125_b200 import _lib as L

    M, N, K = 1280, 1280, 40
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    At, Bt = dev(A), dev(B)
    C = P.zeros((M, N))
    L.call("b2_gemm", 0, 1, M, N, K, At.data_ptr, K, Bt.data_ptr, K, C.data_ptr, N, None, 0,
           L.GEMM_SIMT, None)
    got = host(C)
    acc = np.zeros((M, N), dtype=np.float32)
    a80, b80 = A.astype(np.longdouble), B.astype(np.longdouble)
    for k in range(K):
        acc = (a80[:, k:k + 1] * b80[None, :, k] + acc.astype(np.longdouble)).astype(np.float32)
    mism = int((got.view(np.uint32) != acc.view(np.uint32)).sum())
    assert mism <= M * N * 1e-5, mism
