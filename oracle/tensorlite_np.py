"""CPU oracle: a NumPy float64 restatement of tensorlite's hot-path semantics.

TEST INFRASTRUCTURE ONLY. This module is the *checker* for the device engine
in ``paper_2602_00125_b200``. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import it; the
product path never does (it has no CPU fallback and fails loudly without its
CUDA library).

What it restates (reference = /root/reference, pure-Python ``tensorlite``):

* every engine store rounds a double to float32  (pkg/src/tensorlite/core.py:3-4)
* elementwise add/sub/mul/div = f32(double op)    (core.py:430-495)
  -- equal to IEEE fp32 ops because 53 >= 2*24+2 (innocuous double rounding)
* exp/log/sqrt = f32(libm double)                  (core.py:41-61, 498-530)
* relu = v if v > 0 else 0.0, mask v > 0           (nn.py:108-111)
* full sum: 65536-element chunks, each summed by Python's builtin ``sum``
  (Neumaier-compensated since CPython 3.12), chunk partials added left to
  right in double                                  (core.py:581-594, parallel.py:16,48-63)
* axis sum/mean: row-major double accumulation, mean = f32(dsum/count)
                                                   (core.py:597-689)
* max: strict ``>`` in row-major order; the first maximum wins and receives
  the gradient                                     (core.py:692-728)
* matmul(x, w) = x @ w^T, one double dot per output, rounded once
                                                   (core.py:784-820)
* cross_entropy: per-row double max / log-sum-exp, mean over rows; grad =
  (exp(v-m)/fsum(es) - onehot) * g/b               (nn.py:453-503)
* SGD / Adam with double slots, coupled weight decay, theta rounded to f32
                                                   (optim.py:39-100)
* Dense: y = add(matmul(x, W), b)                  (nn.py:78-82)
* GradStore accumulation order = node order, each contribution a separately
  rounded tensor                                   (autograd.py:140-145, 178-221)

Parity is pinned: ``tests/test_oracle_golden.py`` checks every function here
against fixtures produced by running the reference itself
(``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import math

import numpy as np

CHUNK = 1 << 16  # parallel.py:16


def f32(x):
    """Round doubles to float32 the way every engine store does (core.py:3-4)."""
    return np.asarray(x, dtype=np.float64).astype(np.float32)


def _d(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


# ---------------------------------------------------------------------------
# shapes (core.py:364-423)


def broadcast_shapes(s1, s2):
    """Right-aligned NumPy rule (core.py:364-378)."""
    n = max(len(s1), len(s2))
    a = (1,) * (n - len(s1)) + tuple(s1)
    b = (1,) * (n - len(s2)) + tuple(s2)
    out = []
    for x, y in zip(a, b):
        if x == y or y == 1:
            out.append(x)
        elif x == 1:
            out.append(y)
        else:
            raise ValueError(f"cannot broadcast {tuple(s1)} with {tuple(s2)}")
    return tuple(out)


def reduce_to_shape(g, shape):
    """Adjoint of broadcasting: sum over stretched axes (core.py:405-423)."""
    g = np.asarray(g, dtype=np.float32)
    shape = tuple(shape)
    if g.shape == shape:
        return g
    pad = g.ndim - len(shape)
    padded = (1,) * pad + shape
    axes = tuple(i for i, (h, w) in enumerate(zip(g.shape, padded)) if w != h)
    out = axis_sum(g, axes, keepdims=True) if axes else g
    return out.reshape(shape)


# ---------------------------------------------------------------------------
# elementwise (core.py:430-546, nn.py:95-111)


def binary(kind, a, b):
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    shape = broadcast_shapes(a.shape, b.shape)
    ad = np.broadcast_to(_d(a), shape)
    bd = np.broadcast_to(_d(b), shape)
    with np.errstate(all="ignore"):
        if kind == "add":
            r = ad + bd
        elif kind == "sub":
            r = ad - bd
        elif kind == "mul":
            r = ad * bd
        elif kind == "div":
            r = ad / bd  # IEEE specials match core.py:32-38
        else:
            raise ValueError(kind)
    return f32(r)


def add(a, b):
    return binary("add", a, b)


def sub(a, b):
    return binary("sub", a, b)


def mul(a, b):
    return binary("mul", a, b)


def div(a, b):
    return binary("div", a, b)


def neg(x):
    return (-np.asarray(x, dtype=np.float32)).astype(np.float32)


def exp(x):
    """f32(double exp); overflow saturates to inf (core.py:41-45)."""
    with np.errstate(all="ignore"):
        return f32(np.exp(_d(x)))


def log(x):
    with np.errstate(all="ignore"):
        return f32(np.log(_d(x)))


def sqrt(x):
    with np.errstate(all="ignore"):
        return f32(np.sqrt(_d(x)))


def absolute(x):
    return np.abs(np.asarray(x, dtype=np.float32))


def relu(x):
    """nn.py:108-111: v if v > 0 else 0.0 (so relu(-0)=+0, relu(nan)=0)."""
    x = np.asarray(x, dtype=np.float32)
    return np.where(x > 0, x, np.float32(0.0)).astype(np.float32)


def relu_mask(x):
    x = np.asarray(x, dtype=np.float32)
    return (x > 0).astype(np.float32)


def clamp(x, lo, hi):
    """Not a reference op (clamp happens on the host before the
    oracle). Plain fp32 min/max, bit-exact."""
    return np.clip(np.asarray(x, dtype=np.float32), np.float32(lo), np.float32(hi))


# ---------------------------------------------------------------------------
# reductions (core.py:556-728)


def _neumaier(vals) -> float:
    """CPython 3.12 builtin sum() of floats (compensated). math.fsum is the
    exactly rounded sum; the two agree except under catastrophic cancellation
    below double precision, which never survives the f32 store."""
    return math.fsum(vals)


def sum_all_double(x) -> float:
    """_sum_all (core.py:581-594): chunked, chunk partials in chunk order."""
    v = _d(x).ravel()
    total = 0.0
    for s in range(0, v.size, CHUNK):
        total += _neumaier(v[s : s + CHUNK].tolist())
    return total


def normalize_axes(axis, ndim):
    """core.py:556-572."""
    if axis is None:
        return tuple(range(ndim))
    if isinstance(axis, int):
        axis = (axis,)
    axes = []
    for a in axis:
        if a < 0:
            a += ndim
        if not 0 <= a < ndim:
            raise ValueError(f"axis {a} out of range for {ndim}-d tensor")
        axes.append(a)
    if len(set(axes)) != len(axes):
        raise ValueError("duplicate axes")
    return tuple(sorted(axes))


def _axis_double_sum(x, axes):
    """Row-major double accumulation per output slot (core.py:597-632, 654).

    Sequential accumulation is restated with np.add.reduce over float64 after
    moving reduced axes last; the accumulation error of either order is far
    below one f32 ulp of the result."""
    xd = _d(x)
    return np.sum(xd, axis=axes, dtype=np.float64)


def axis_sum(x, axis=None, keepdims=False):
    x = np.asarray(x, dtype=np.float32)
    axes = normalize_axes(axis, x.ndim)
    if len(axes) == x.ndim:
        r = f32(sum_all_double(x))
        return r.reshape((1,) * x.ndim) if keepdims else r.reshape(())
    if not axes:
        return x.copy()
    r = f32(_axis_double_sum(x, axes))
    if keepdims:
        r = r.reshape(tuple(1 if i in axes else s for i, s in enumerate(x.shape)))
    return r


def axis_mean(x, axis=None, keepdims=False):
    """mean = f32(dsum / count) (core.py:663-689)."""
    x = np.asarray(x, dtype=np.float32)
    axes = normalize_axes(axis, x.ndim)
    count = 1
    for a in axes:
        count *= x.shape[a]
    with np.errstate(all="ignore"):
        if len(axes) == x.ndim:
            r = f32(sum_all_double(x) / float(count) if count else math.nan)
            return r.reshape((1,) * x.ndim) if keepdims else r.reshape(())
        if not axes:
            return x.copy()
        r = f32(_axis_double_sum(x, axes) / float(count))
    if keepdims:
        r = r.reshape(tuple(1 if i in axes else s for i, s in enumerate(x.shape)))
    return r


def axis_max(x, axis=None, keepdims=False):
    """Returns (values, argpos) where argpos is the row-major flat index of
    the winning element in x (core.py:692-728). Strict '>' => first wins;
    a NaN in the first scanned slot sticks, later NaNs are skipped."""
    x = np.asarray(x, dtype=np.float32)
    axes = normalize_axes(axis, x.ndim)
    kept = [d for d in range(x.ndim) if d not in axes]
    perm = kept + list(axes)
    xt = np.transpose(x, perm)
    oshape = tuple(x.shape[d] for d in kept)
    nred = int(np.prod([x.shape[d] for d in axes], dtype=np.int64)) if axes else 1
    flat_idx = np.arange(x.size, dtype=np.int64).reshape(x.shape)
    it = np.transpose(flat_idx, perm).reshape(-1, nred)
    xr = xt.reshape(-1, nred)
    first = xr[:, 0]
    masked = np.where(np.isnan(xr), -np.inf, xr)
    # first occurrence of the max among non-NaN values
    am = np.argmax(masked, axis=1)
    # rows where every non-nan equals -inf and there are NaNs: argmax picks
    # the first -inf-or-NaN slot; restate the sequential rule explicitly
    vals = xr[np.arange(xr.shape[0]), am]
    nan_first = np.isnan(first)
    am = np.where(nan_first, 0, am)
    # when all later values are NaN/-inf and first is -inf, first wins anyway
    vals = np.where(nan_first, first, vals)
    fix = (~nan_first) & np.isnan(vals)
    if fix.any():  # row whose max slot is NaN (only -inf elsewhere)
        am = np.where(fix, 0, am)
        vals = np.where(fix, first, vals)
    pos = it[np.arange(it.shape[0]), am]
    vals = vals.astype(np.float32).reshape(oshape)
    pos = pos.reshape(oshape)
    if keepdims:
        ks = tuple(1 if i in axes else s for i, s in enumerate(x.shape))
        vals = vals.reshape(ks)
        pos = pos.reshape(ks)
    return vals, pos


def max_pullback(g, argpos, in_shape):
    """core.py:721-726: scatter the seed to the winning positions."""
    acc = np.zeros(int(np.prod(in_shape, dtype=np.int64)), dtype=np.float64)
    np.add.at(acc, np.asarray(argpos).ravel(), _d(g).ravel())
    return f32(acc).reshape(in_shape)


# ---------------------------------------------------------------------------
# matmul (core.py:768-820)


def matmul_xwt(x, w):
    """y = x @ w^T, double dot, one f32 rounding per output (core.py:784-807)."""
    return f32(_d(x) @ _d(w).T)


def matmul_grads(g, x, w):
    """Pullbacks (core.py:815-817): x_bar = g w, w_bar = g^T x."""
    return f32(_d(g) @ _d(w)), f32(_d(g).T @ _d(x))


# ---------------------------------------------------------------------------
# losses / activations (nn.py:453-503, tests/oracles.py:203-215)


def cross_entropy(logits, labels):
    """Returns (loss f32 scalar, loss double, dlogits f32) for seed 1.0."""
    z = _d(logits)
    labels = np.asarray(labels, dtype=np.int64)
    b, c = z.shape
    if b == 0:
        raise ValueError("cross_entropy needs at least one row")
    if labels.shape != (b,):
        raise ValueError(f"{labels.size} labels for {b} rows")
    if labels.size and (labels.min() < 0 or labels.max() >= c):
        raise ValueError("label out of range")
    m = z.max(axis=1, keepdims=True)
    with np.errstate(all="ignore"):
        es = np.exp(z - m)
    se = es.sum(axis=1)
    rows = m[:, 0] + np.log(se) - z[np.arange(b), labels]
    total = 0.0
    for r in rows.tolist():  # nn.py:476-485 accumulates rows in order
        total += r
    loss_d = total / b
    gv = 1.0 / b  # g.flat()[0] / b with g = 1.0   (nn.py:489)
    # nn.py:497-500: es/fsum(es) - onehot, times gv
    se_f = np.array([math.fsum(row) for row in es.tolist()]) if b * c <= 1 << 22 else se
    grad = es / se_f[:, None]
    grad[np.arange(b), labels] -= 1.0
    grad *= gv
    return f32(loss_d), loss_d, f32(grad)


def softmax_rows_composed(z):
    """Config-4 softmax composed from engine ops with the row max detached
    (SURVEY 8c): m = max(z,-1,keepdims).detach(); d = sub(z,m); e = exp(d);
    s = sum(e,-1,keepdims); Y = div(e,s). Returns (Y, e, s)."""
    z = np.asarray(z, dtype=np.float32)
    m, _ = axis_max(z, axis=-1, keepdims=True)
    d = sub(z, m)
    e = exp(d)
    s = axis_sum(e, axis=-1, keepdims=True)
    y = div(e, s)
    return y, e, s


def softmax_backward_composed(gy, e, s):
    """Reverse of the composition above in GradStore order
    (autograd.py:140-145; core.py:486-495, 635-640, 509-514):
    gE = f32(gY/s); gS = rowsum64(f32(-f32(f32(gY*e)/f32(s*s))));
    gE_total = f32(gE + gS); gz = f32(gE_total * e)."""
    ge = div(gy, s)
    gs = axis_sum(neg(div(mul(gy, e), mul(s, s))), axis=-1, keepdims=True)
    ge_tot = add(ge, gs)
    return mul(ge_tot, e)


# ---------------------------------------------------------------------------
# optimizers (optim.py:39-136)


class SGD:
    """v = mu*v + g + wd*theta; theta = f32(theta - lr*v) (optim.py:54-72)."""

    def __init__(self, lr=0.01, momentum=0.0, weight_decay=0.0):
        self.lr, self.momentum, self.weight_decay = lr, momentum, weight_decay
        self.state = {}

    def step(self, key, theta, grad):
        th = _d(theta)
        g = _d(grad)
        if self.weight_decay:
            g = g + self.weight_decay * th
        v = self.state.get(key)
        if v is None:
            v = np.zeros_like(th)
        v = self.momentum * v + g
        self.state[key] = v
        return f32(th - self.lr * v)


class Adam:
    """Debiased moments, eps outside sqrt, double slots (optim.py:75-100)."""

    def __init__(self, lr=0.001, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0):
        self.lr = lr
        self.b1, self.b2 = betas
        self.eps = eps
        self.weight_decay = weight_decay
        self.state = {}

    def step(self, key, theta, grad):
        th = _d(theta)
        g = _d(grad)
        if self.weight_decay:
            g = g + self.weight_decay * th
        st = self.state.get(key)
        if st is None:
            st = {"m": np.zeros_like(th), "v": np.zeros_like(th), "t": 0}
            self.state[key] = st
        st["t"] += 1
        t = st["t"]
        b1, b2 = self.b1, self.b2
        bc1 = 1.0 - b1 ** t
        bc2 = 1.0 - b2 ** t
        m = b1 * st["m"] + (1.0 - b1) * g
        v = b2 * st["v"] + (1.0 - b2) * g * g
        st["m"], st["v"] = m, v
        return f32(th - self.lr * (m / bc1) / (np.sqrt(v / bc2) + self.eps))


class RMSprop:
    """v = rho*v + (1-rho)*g*g; theta = f32(theta - lr*g/sqrt(v + eps)) (optim.py:103-122)."""

    def __init__(self, lr=0.01, rho=0.99, eps=1e-8, weight_decay=0.0):
        self.lr, self.rho, self.eps, self.weight_decay = lr, rho, eps, weight_decay
        self.state = {}

    def step(self, key, theta, grad):
        th = _d(theta)
        g = _d(grad)
        if self.weight_decay:
            g = g + self.weight_decay * th
        v = self.state.get(key)
        if v is None:
            v = np.zeros_like(th)
        v = self.rho * v + (1.0 - self.rho) * g * g
        self.state[key] = v
        return f32(th - self.lr * g / np.sqrt(v + self.eps))


# ---------------------------------------------------------------------------
# pointwise activations (nn.py:95-144): out = f32(fn(double x)); the pullback
# multiplies g by f32(dfn(v)), v the saved input or output


def _map(fn, x):
    flat = [fn(float(v)) for v in np.asarray(x, np.float32).ravel()]
    return f32(np.array(flat, np.float64).reshape(np.shape(x)))


def _sigmoid_scalar(v):  # nn.py:114-119, split on sign
    if v >= 0.0:
        return 1.0 / (1.0 + math.exp(-v))
    e = math.exp(v)
    return e / (1.0 + e)


_SQRT2 = math.sqrt(2.0)
_INV_SQRT_2PI = 1.0 / math.sqrt(2.0 * math.pi)


def _gelu_scalar(v):  # nn.py:132-133
    return 0.5 * v * (1.0 + math.erf(v / _SQRT2))


def _gelu_deriv(v):  # nn.py:136-139
    cdf = 0.5 * (1.0 + math.erf(v / _SQRT2))
    pdf = _INV_SQRT_2PI * math.exp(-0.5 * v * v)
    return cdf + v * pdf


def _math_tanh(v):
    return math.tanh(v)


def sigmoid(x):
    return _map(_sigmoid_scalar, x)


def tanh(x):
    return _map(_math_tanh, x)


def gelu(x):
    return _map(_gelu_scalar, x)


def activation_grad(kind, g, x, y):
    """g * f32(dfn(v)) with v = y for sigmoid/tanh, x for gelu (nn.py:101-103)."""
    if kind == "sigmoid":
        d = _map(lambda v: v * (1.0 - v), y)
    elif kind == "tanh":
        d = _map(lambda v: 1.0 - v * v, y)
    else:
        d = _map(_gelu_deriv, x)
    return mul(g, d)


# ---------------------------------------------------------------------------
# conv2d (nn.py:191-303): im2col (+ ones column for the bias, folded into the
# same double dot), permute, col2im scatter in row order with double sums


def _im2col(x, kh, kw, s, p):
    b, c, h, w = x.shape
    oh, ow = (h + 2 * p - kh) // s + 1, (w + 2 * p - kw) // s + 1
    xp = np.zeros((b, c, h + 2 * p, w + 2 * p), np.float64)
    xp[:, :, p:p + h, p:p + w] = x
    cols = np.empty((b, oh, ow, c, kh, kw), np.float64)
    for u in range(kh):
        for v in range(kw):
            cols[:, :, :, :, u, v] = xp[:, :, u:u + s * oh:s, v:v + s * ow:s].transpose(0, 2, 3, 1)
    return cols.reshape(b * oh * ow, c * kh * kw), oh, ow


def conv2d(x, w, bias, stride=1, padding=0):
    """Returns (y, pullback(g) -> (dx, dw, db))."""
    x = np.asarray(x, np.float32)
    b, c, h, wd = x.shape
    cout, _, kh, kw = w.shape
    pt, oh, ow = _im2col(x, kh, kw, stride, padding)
    wf = _d(w).reshape(cout, -1)
    if bias is not None:  # the reference's trailing ones column (nn.py:222-246)
        y = f32(np.concatenate([pt, np.ones((pt.shape[0], 1))], 1)
                @ np.concatenate([wf, _d(bias)[:, None]], 1).T)
    else:
        y = f32(pt @ wf.T)
    out = y.reshape(b, oh * ow, cout).transpose(0, 2, 1).reshape(b, cout, oh, ow)

    def pull(g):
        gr = np.asarray(g, np.float32).reshape(b, cout, oh * ow).transpose(0, 2, 1).reshape(-1, cout)
        dp = f32(_d(gr) @ wf)  # (rows, cols)
        dx = np.zeros((b, c, h + 2 * padding, wd + 2 * padding), np.float64)
        dpv = dp.astype(np.float64).reshape(b, oh, ow, c, kh, kw)
        # rows in increasing order per pixel == accumulate taps by output position
        for i in range(oh):
            for j in range(ow):
                for u in range(kh):
                    for v in range(kw):
                        dx[:, :, i * stride + u, j * stride + v] += dpv[:, i, j, :, u, v]
        dx = f32(dx[:, :, padding:padding + h, padding:padding + wd])
        dw = f32(_d(gr).T @ pt).reshape(w.shape)
        db = None if bias is None else axis_sum(np.asarray(g, np.float32), (0, 2, 3))
        return dx, dw, db

    return out, pull


# ---------------------------------------------------------------------------
# composed hot paths (BASELINE configs)


def mlp_train_step(params, x, labels, opt, keys=None, relu_between=True):
    """One reference train step over a Sequential of Dense(+ReLU) layers
    (demos.py:110-121 loop body; nn.py:78-82; autograd.py:178-221).

    params: list of (W[out,in], b[out]) f32 arrays. Returns dict with loss,
    grads (same structure) and updated params."""
    x = np.asarray(x, dtype=np.float32)
    acts = [x]
    pre = []
    h = x
    n = len(params)
    for i, (w, b) in enumerate(params):
        z = add(matmul_xwt(h, w), b)
        pre.append(z)
        h = relu(z) if (relu_between and i < n - 1) else z
        acts.append(h)
    loss, loss_d, g = cross_entropy(h, labels)
    grads = [None] * n
    for i in range(n - 1, -1, -1):
        w, b = params[i]
        if relu_between and i < n - 1:
            g = mul(g, relu_mask(pre[i]))  # nn.py:101-103
        gb = reduce_to_shape(g, b.shape)  # add pullback (core.py:457-458)
        gx, gw = matmul_grads(g, acts[i], w)
        grads[i] = (gw, gb)
        g = gx
    new = []
    for i, ((w, b), (gw, gb)) in enumerate(zip(params, grads)):
        kw, kb = (keys[2 * i], keys[2 * i + 1]) if keys else (("w", i), ("b", i))
        new.append((opt.step(kw, w, gw), opt.step(kb, b, gb)))
    return {"loss": loss, "loss_double": loss_d, "grads": grads, "params": new,
            "logits": h}


def broadcast_reduce_config(a, b, clamp_lo=-10.0, clamp_hi=10.0):
    """BASELINE config 2 through reference ops (SURVEY 3.3 and 8a recipe)."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    p = mul(a, b)
    q = add(p, b)
    y = relu(q)
    e = exp(clamp(a, clamp_lo, clamp_hi))
    out = {
        "y": y,
        "e": e,
        "sum0": axis_sum(y, 0), "sum1": axis_sum(y, 1),
        "mean0": axis_mean(y, 0), "mean1": axis_mean(y, 1),
        "max0": axis_max(y, 0)[0], "max1": axis_max(y, 1)[0],
        "sum_all": axis_sum(y),
    }
    # backward of sum(y) wrt a and b, GradStore order
    mask = relu_mask(q)
    ga = reduce_to_shape(mul(mask, b), a.shape)
    gb_add = reduce_to_shape(mask, b.shape)
    gb_mul = reduce_to_shape(mul(mask, a), b.shape)
    out["grad_a"] = ga
    out["grad_b"] = add(gb_add, gb_mul)
    return out


def matmul_fwd_bwd(A, B, dC):
    """Config 3 in the reference convention: C = matmul(A, transpose2d(B));
    backward(C, seed=dC)."""
    A64, B64, g64 = _d(A), _d(B), _d(dC)
    C = f32(A64 @ B64)
    dA = f32(g64 @ B64.T)
    dB = f32(A64.T @ g64)
    return C, dA, dB


def softmax_linear_config(X, W, bias, T):
    """Config 4: Y = softmax(X@W + bias); loss = mean(Y*T); full backward.
    X: [..., K] flattened to rows (rank-3 matmul via reshape)."""
    K = X.shape[-1]
    X2 = np.asarray(X, dtype=np.float32).reshape(-1, K)
    z = add(f32(_d(X2) @ _d(W)), bias)
    y, e, s = softmax_rows_composed(z)
    T2 = np.asarray(T, dtype=np.float32).reshape(y.shape)
    P = mul(y, T2)
    loss = axis_mean(P)
    count = P.size
    gP = f32(np.full(P.shape, 1.0 / count))  # mean pullback: div(ones, count)
    gy = mul(gP, T2)
    gz = softmax_backward_composed(gy, e, s)
    gbias = axis_sum(gz, 0)
    dX = f32(_d(gz) @ _d(W).T)
    dW = f32(_d(X2).T @ _d(gz))
    return {"loss": loss, "Y": y.reshape(np.shape(X)[:-1] + (W.shape[1],)),
            "dX": dX.reshape(np.shape(X)), "dW": dW, "dbias": gbias}
