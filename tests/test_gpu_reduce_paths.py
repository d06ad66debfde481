"""The single-launch reduction paths (reduce.cu), bit-exact against the oracle.

* column reductions folded through distributed shared memory (`k_cols`: 32-
  column strips x a cluster of row splits) -- sum, mean, max with the
  reference's scan semantics (core.py:692-728: strict '>', first index wins,
  first-slot NaN sticks, -0 before +0);
* row reductions whose split partials are folded by the last-arriving CTA
  (`k_rows` + per-stream arrival counters) -- repeated launches re-arm the
  counters, and CUDA-graph replays reuse them.
"""

import numpy as np
import pytest

import paper_2602_00125_b200 as P
from oracle import tensorlite_np as O
from paper_2602_00125_b200 import _lib as L, graph
from tests.golden.load import bits_equal

pytestmark = pytest.mark.gpu


def dev(a, grad=False):
    return P.from_numpy(np.asarray(a, np.float32), requires_grad=grad)


@pytest.mark.parametrize("shape", [(4096, 4096), (2048, 3000), (4096, 2080), (1024, 4100)])
def test_cluster_column_sum_mean(shape):
    rng = np.random.default_rng(sum(shape))
    x = (rng.standard_normal(shape) * rng.uniform(0.1, 50, shape[1])).astype(np.float32)
    t = dev(x)
    assert bits_equal(P.sum(t, axis=0).numpy(), O.axis_sum(x, 0))
    assert bits_equal(P.mean(t, axis=0).numpy(), O.axis_mean(x, 0))
    assert bits_equal(P.sum(t, axis=0, keepdims=True).numpy(), O.axis_sum(x, 0, keepdims=True))


def test_cluster_middle_axis_sum_and_max():
    rng = np.random.default_rng(5)
    x = rng.standard_normal((3, 2048, 1028)).astype(np.float32)
    t = dev(x)
    assert bits_equal(P.sum(t, axis=1).numpy(), O.axis_sum(x, 1))
    assert bits_equal(P.max(t, axis=1).numpy(), O.axis_max(x, 1)[0])


def test_cluster_column_max_semantics_and_routing():
    """Heavy ties, +-0 maxima, NaNs (some in the first slot), all -inf
    columns, lone maxima deep in a column: values and the argmax routing
    (through the gradient) bit-exact on a shape that takes the cluster path."""
    rng = np.random.default_rng(17)
    R, C = 4096, 2080
    x = rng.integers(-3, 1, (R, C)).astype(np.float32)
    x[rng.random((R, C)) < 0.3] = -0.0
    x[rng.random((R, C)) < 0.01] = np.nan
    x[0, 5] = np.nan
    x[:, 7] = -np.inf
    x[:, 9] = -1.0
    x[4001, 9] = 2.0
    x[:, 11] = -0.0
    x[2500, 11] = 0.0
    x[:, 13] = -np.inf
    x[3000, 13] = np.nan
    xt = dev(x, grad=True)
    r = P.max(xt, axis=0)
    v, pos = O.axis_max(x, 0)
    assert bits_equal(r.numpy(), v)
    store = P.backward(P.sum(r))
    assert bits_equal(store[xt].numpy(), O.max_pullback(np.ones(C, np.float32), pos, x.shape))
    P.reset_tape()


@pytest.mark.parametrize("shape", [(1, 1 << 24), (3, 1 << 20), (37, 65536), (5, 100003)])
def test_split_row_reductions_fold_in_the_last_cta(shape):
    rng = np.random.default_rng(shape[0])
    x = rng.standard_normal(shape).astype(np.float32)
    x[:, -1] += 1e6  # a large term at the end of each row
    t = dev(x)
    want_s = O.axis_sum(x, 1)
    want_m = O.axis_max(x, 1)[0]
    for _ in range(3):  # counters re-arm between launches
        assert bits_equal(P.sum(t, axis=1).numpy(), want_s)
        assert bits_equal(P.mean(t, axis=1).numpy(), O.axis_mean(x, 1))
        assert bits_equal(P.max(t, axis=1).numpy(), want_m)
    assert bits_equal(P.sum(t).numpy(), O.axis_sum(x, None))


def test_split_row_max_argmax_routing():
    rng = np.random.default_rng(23)
    x = rng.integers(-5, 5, (2, 1 << 20)).astype(np.float32)  # many ties at the max
    x[1, 0] = np.nan                                          # first slot sticks
    xt = dev(x, grad=True)
    r = P.max(xt, axis=1)
    v, pos = O.axis_max(x, 1)
    assert bits_equal(r.numpy(), v)
    store = P.backward(P.sum(r))
    assert bits_equal(store[xt].numpy(), O.max_pullback(np.ones(2, np.float32), pos, x.shape))
    P.reset_tape()


def test_single_launch_reductions_under_graph_replay():
    rng = np.random.default_rng(3)
    xs = [rng.standard_normal((2, 1 << 21)).astype(np.float32) for _ in range(2)]
    cols = rng.standard_normal((4096, 1024)).astype(np.float32)
    ts = [dev(v) for v in xs]
    tc = dev(cols)
    outs = []

    def body():
        outs.clear()
        with P.no_grad():
            for t in ts:
                outs.append(P.sum(t))
                outs.append(P.max(t, axis=1))
            outs.append(P.sum(tc, axis=0))
            outs.append(P.max(tc, axis=0))

    g = graph.capture(body, warmup=1)
    for _ in range(3):
        g.replay()
        L.synchronize()
        got = [o.numpy() for o in outs]
        k = 0
        for v in xs:
            assert bits_equal(got[k], O.axis_sum(v, None))
            assert bits_equal(got[k + 1], O.axis_max(v, 1)[0])
            k += 2
        assert bits_equal(got[k], O.axis_sum(cols, 0))
        assert bits_equal(got[k + 1], O.axis_max(cols, 0)[0])
