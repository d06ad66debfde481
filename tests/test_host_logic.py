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


# The reference's public names (tensorlite/__init__.py:8-66, bindings/src/tlnp.py:36-45 and the
# handle / module / optimizer methods its tests call): a program written against the reference
# must find every one of them here.
_ENGINE_NAMES = """BroadcastError DeterminismError GradError GradStore ShapeError Tensor abs_ absolute add
autograd backward broadcast_shapes broadcast_to core div errors exp from_buffer from_flat full gradcheck
is_recording log matmul max max_workers mean mul neg nn no_grad ones ones_like optim parallel record
reduce_to_shape reset_tape reshape sqrt sub sum tape tensor thread_limit transpose2d uniform zero_grad zeros
zeros_like""".split()
_TLNP_NAMES = """Adam BatchNorm BroadcastError Conv2D Dense DeterminismError Dropout GELU GradError Module
RMSprop ReLU SGD Sequential ShapeError Sigmoid Tanh Tensor cross_entropy full matmul mse no_grad ones
reset_tape tensor to_host_array uniform wrap_host_array zeros""".split()
_HANDLE_NAMES = """T __abs__ __add__ __bool__ __eq__ __float__ __ge__ __getitem__ __gt__ __le__ __len__ __lt__
__matmul__ __mul__ __ne__ __neg__ __radd__ __rmul__ __rsub__ __rtruediv__ __setitem__ __sub__ __truediv__
backward detach exp grad log max mean numpy requires_grad requires_grad_ reshape sqrt sum
transpose""".split()


def test_reference_public_names_are_all_present():
    import importlib

    import paper_2602_00125_b200 as P
    from paper_2602_00125_b200 import tlnp

    missing = [n for n in _ENGINE_NAMES if not hasattr(P, n)]
    for sub in ("autograd", "core", "errors"):
        importlib.import_module(f"paper_2602_00125_b200.{sub}")
    missing = [n for n in missing if not hasattr(P, n)]
    assert not missing, missing
    assert not [n for n in _TLNP_NAMES if not hasattr(tlnp, n)]
    assert not [n for n in _HANDLE_NAMES if not hasattr(tlnp.Tensor, n)]
    # forwarded introspection and flags of a handle are instance attributes
    assert set(("shape", "ndim", "size", "item", "tolist")) <= set(tlnp.Tensor._FORWARDED)
    assert set(("origin", "copied")) <= set(tlnp.Tensor.__slots__)
    for cls in (tlnp.Dense, tlnp.Sequential):
        assert not [n for n in ("eval", "train", "parameters", "named_parameters") if not hasattr(cls, n)]
    for cls in (tlnp.SGD, tlnp.Adam, tlnp.RMSprop):
        assert hasattr(cls, "step") and hasattr(cls, "zero_grad")


def test_worker_setting_contract(monkeypatch):
    """max_workers / thread_limit / TENSORLITE_THREADS keep the reference's
    semantics (parallel.py:25-46); spans are worker-independent CHUNK cuts."""
    import threading

    from paper_2602_00125_b200 import parallel

    monkeypatch.delenv("TENSORLITE_THREADS", raising=False)
    base = parallel.max_workers()
    assert 1 <= base <= 8
    monkeypatch.setenv("TENSORLITE_THREADS", "3")
    assert parallel.max_workers() == 3
    monkeypatch.setenv("TENSORLITE_THREADS", "zero")
    assert parallel.max_workers() == base
    with parallel.thread_limit(5):
        assert parallel.max_workers() == 5
        with parallel.thread_limit(0):
            assert parallel.max_workers() == 1
        seen = []
        t = threading.Thread(target=lambda: seen.append(parallel.max_workers()))
        t.start()
        t.join()
        assert seen == [base]  # a limit belongs to the thread that set it
        assert parallel.max_workers() == 5
    assert parallel.max_workers() == base
    assert parallel.spans(0) == [] and parallel.spans(-3) == []
    assert parallel.spans(5) == [(0, 5)]
    cuts = parallel.spans(3 * parallel.CHUNK + 7)
    assert cuts[0] == (0, parallel.CHUNK) and cuts[-1] == (3 * parallel.CHUNK, 3 * parallel.CHUNK + 7)
    assert all(a[1] == b[0] for a, b in zip(cuts, cuts[1:]))
