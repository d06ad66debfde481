"""CPU tests of the host-side logic that needs no kernel: broadcasting rules,
axis normalisation, view construction, GEMM operand-layout detection, and the
autograd tape contract (tensorlite/autograd.py semantics) on view-only ops."""

import pytest

from paper_2602_00125_b200 import autograd as A
from paper_2602_00125_b200 import core as C
from paper_2602_00125_b200.errors import BroadcastError, GradError, ShapeError


def fake(shape, strides=None, offset=0, grad=False):
    """A Tensor with no storage: enough for shape/stride logic and views."""
    return C.Tensor(None, shape, strides, offset, requires_grad=grad)


def test_broadcast_shapes_rules():
    assert C.broadcast_shapes((2, 1, 4), (3, 1)) == (2, 3, 4)
    assert C.broadcast_shapes((), (5,)) == (5,)
    assert C.broadcast_shapes((4096, 4096), (1, 4096)) == (4096, 4096)
    with pytest.raises(BroadcastError):
        C.broadcast_shapes((2,), (3,))


def test_expand_strides_are_stride_zero_views():
    t = fake((1, 4096))
    assert C._expand_strides(t, (4096, 4096)) == (0, 1)
    t = fake((3, 1))
    assert C._expand_strides(t, (2, 3, 5)) == (0, 1, 0)
    with pytest.raises(BroadcastError):
        C._expand_strides(fake((3,)), (4,))


def test_normalize_axes_and_reduced_shapes():
    assert C._normalize_axes(None, 3) == (0, 1, 2)
    assert C._normalize_axes(-1, 2) == (1,)
    assert C._normalize_axes((2, 0), 3) == (0, 2)
    with pytest.raises(ShapeError):
        C._normalize_axes(2, 2)
    with pytest.raises(ShapeError):
        C._normalize_axes((0, 0), 2)
    assert C._reduced_shapes((4, 5, 6), (1,), False) == ((4, 1, 6), (4, 6))
    assert C._reduced_shapes((4, 5, 6), (0, 2), True) == ((1, 5, 1), (1, 5, 1))
    assert C._mask((0, 2)) == 0b101


def test_views_share_storage_and_strides():
    t = fake((2, 3))
    tt = C.transpose2d(t)
    assert tt.shape == (3, 2) and tt.strides == (1, 3)
    r = C.reshape(t, (3, -1))
    assert r.shape == (3, 2) and r.buffer is t.buffer
    b = C.broadcast_to(fake((2, 1)), (2, 5))
    assert b.strides == (1, 0)
    with pytest.raises(ShapeError):
        C.reshape(t, (-1, -1))
    with pytest.raises(ShapeError):
        C.reshape(t, (4, -1))
    with pytest.raises(ShapeError):
        C.transpose2d(fake((3,)))


def test_gemm_operand_layouts_read_views_in_place():
    # the reference's three matmul layouts map onto K-/MN-major operands, no copies
    x = fake((256, 784))                    # x: [M,K] row-major
    w = fake((256, 784))                    # W: [N,K] row-major  -> x.W^T (NT)
    assert C._as_A(x)[:2] == (0, 784)
    assert C._as_B(w)[:2] == (1, 784)
    g = fake((256, 10))
    wt = C.transpose2d(fake((10, 256)))     # x_bar = g . W : B stored [K, N]
    assert C._as_B(wt)[:2] == (0, 256)
    gt = C.transpose2d(g)                    # w_bar = g^T . x : A stored [K, M]
    assert C._as_A(gt)[:2] == (1, 10)
    xt = C.transpose2d(x)
    assert C._as_B(xt)[:2] == (0, 784)


def test_tape_records_only_with_grad_and_while_recording():
    A.reset_tape()
    x, y = fake((2, 2), grad=True), fake((2, 2))
    out = A.record("op", (x, y), fake((2, 2)), (lambda g: g, lambda g: g))
    assert out.requires_grad and len(A.tape()) == 2       # leaf x + op node
    assert out.node.parents == (x.node.id,)
    with A.no_grad():
        o2 = A.record("op", (x,), fake((2, 2)), (lambda g: g,))
    assert not o2.requires_grad and len(A.tape()) == 2
    o3 = A.record("op", (y,), fake((2, 2)), (lambda g: g,))
    assert not o3.requires_grad


def test_epochs_make_nodes_stale():
    A.reset_tape()
    x = fake((1,), grad=True)
    out = A.record("op", (x,), fake((1,)), (lambda g: g,))
    A.reset_tape()
    with pytest.raises(GradError):
        A.backward(out, seed=fake((1,)))


def test_backward_seed_rules():
    A.reset_tape()
    x = fake((3,), grad=True)
    out = A.record("op", (x,), fake((3,)), (lambda g: g,))
    with pytest.raises(GradError):
        A.backward(out)                      # non-scalar loss needs a seed
    with pytest.raises(ShapeError):
        A.backward(out, seed=fake((2,)))


def test_backward_walk_order_and_leaf_ready_hook():
    A.reset_tape()
    seen, ready = [], []
    x = fake((1,), grad=True)
    h = A.record("f", (x,), fake((1,)), (lambda g: (seen.append("f"), g)[1],))
    o = A.record("g", (h,), fake((1,)), (lambda g: (seen.append("g"), g)[1],))
    seed = fake((1,))
    store = A.backward(o, seed=seed, on_leaf_ready=lambda nid, g: ready.append(nid))
    assert seen == ["g", "f"]                # decreasing node ids
    assert ready == [x.node.id]
    assert store.get(x) is seed              # first contribution stored as is (aliasing)
    assert A.tape().pullback_calls == 2
