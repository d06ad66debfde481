"""Randomised fused-GEMM cases (the reference's Hypothesis
strategies, applied to the device GEMM the way tests/test_core.py:47-64
applies them to elementwise ops).

Each example draws a shape (ragged M/N, short and long K, single-wave,
multi-wave and tail-wave tile counts), an operand layout (x or w handed in
as transposed views: NT / NN / TN / TT), a scheme (3xBF16, TF32X, BF16) and a
set of epilogue stages (bias, ReLU, relu bits, fp32 or bit mask, column sums,
split emission), runs one b2_gemm_fused launch through core._gemm_into and
checks every output it asked for:

* C against an fp64 NumPy product with the same epilogue (normwise);
* relu bits == packbits(C > 0) exactly; masked entries exactly zero;
* the emitted split == the split of the stored C, bit for bit;
* the column sums against fp64 column sums of the stored C.
"""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
from paper_2602_00125_b200 import core as C
from tests.golden.load import normwise

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _eager_fp32_outputs(monkeypatch):
    # these cases check the kernel's emitted split against its own fp32 C, so
    # every GEMM stores C (the lazy split-only outputs: test_gpu_lazy_fp32.py)
    monkeypatch.setattr(C, "_LAZY_FP32", False)

TOL = {"3xbf16": 1e-5, "tf32x": 5e-6, "bf16": 2e-5}
SEEN = {"cases": 0, "bits_written": 0, "split_checked": 0, "colsum": 0, "masked": 0}

SHAPES = [(264, 136, 96), (1000, 520, 256), (3000, 1800, 1024), (2304, 2304, 1024),
          (512, 1024, 4096), (4104, 256, 64), (72, 4096, 512), (2560, 2048, 2048)]


def _bf16_rn(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


def _split_ref(c, kind):
    if kind == "3xbf16":
        hi = _bf16_rn(c)
        return hi, _bf16_rn((c - hi).astype(np.float32))
    if kind == "tf32x":
        t = (np.ascontiguousarray(c, np.float32).view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
        return _bf16_rn(t), _bf16_rn((c - t).astype(np.float32))
    return _bf16_rn(c), None


def _read(buf, n, dtype):
    import ctypes

    out = np.empty(n, dtype)
    L.call("b2_memcpy_d2h", out.ctypes.data_as(ctypes.c_void_p), buf.ptr, out.nbytes, None)
    return out


def _bf16_arr(buf, n):
    return (_read(buf, n, np.uint16).astype(np.uint32) << 16).view(np.float32)


def _pack_bits(y):
    M, N = y.shape
    W = (N + 63) // 64
    b = np.zeros((M, W * 64), np.uint8)
    b[:, :N] = y > 0
    return np.packbits(b.reshape(M, W, 64), axis=2, bitorder="little").view(np.uint64).reshape(M, W)


@st.composite
def case(draw):
    shape = draw(st.sampled_from(SHAPES))
    algo = draw(st.sampled_from(["3xbf16", "tf32x", "bf16"]))
    ta, tb = draw(st.booleans()), draw(st.booleans())
    bias = draw(st.booleans())
    relu = draw(st.booleans())
    mask = draw(st.sampled_from([None, "fp32", "bits"]))
    colsum = draw(st.booleans())
    emit = draw(st.booleans())
    seed = draw(st.integers(0, 2 ** 16))
    return shape, algo, ta, tb, bias, relu, mask, colsum, emit, seed


@settings(max_examples=40, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.too_slow, HealthCheck.data_too_large])
@given(case())
def test_fused_gemm_random_cases(c):
    (M, N, K), algo, ta, tb, use_bias, relu, mask_kind, use_colsum, emit, seed = c
    rng = np.random.default_rng(seed)
    xa = rng.standard_normal((K, M) if ta else (M, K)).astype(np.float32)
    wa = (rng.standard_normal((K, N) if tb else (N, K)) / np.sqrt(K)).astype(np.float32)
    x = P.transpose2d(P.from_numpy(xa)) if ta else P.from_numpy(xa)       # (M, K) view
    w = P.transpose2d(P.from_numpy(wa)) if tb else P.from_numpy(wa)       # (N, K) view
    xv = xa.T if ta else xa
    wv = wa.T if tb else wa
    bias = P.from_numpy(rng.uniform(-0.5, 0.5, N).astype(np.float32)) if use_bias else None
    epi = {(False, False): L.EPI_NONE, (True, False): L.EPI_BIAS, (False, True): L.EPI_RELU,
           (True, True): L.EPI_BIAS_RELU}[(use_bias, relu)]
    m_np = None
    mask = bits = None
    if mask_kind is not None:
        m_np = (rng.uniform(-1, 1, (M, N)) > 0).astype(np.float32)
        mask = P.from_numpy(m_np)
        if mask_kind == "bits":
            words = _pack_bits(m_np)
            bits = P.Buffer(words.nbytes)
            import ctypes

            L.call("b2_memcpy_h2d", bits.ptr, words.ctypes.data_as(ctypes.c_void_p), words.nbytes, None)
    bits_out = P.Buffer(8 * M * ((N + 63) // 64)) if relu else None
    out = P.zeros((M, N))
    cs = P.zeros((N,)) if use_colsum else None
    P.set_gemm_algo(algo)
    try:
        wrote_bits = C._gemm_into(out, x, w, bias, epi, mask=mask, emit_split=emit, colsum=cs,
                                  mask_bits=bits, bits_out=bits_out)
    finally:
        P.set_gemm_algo(None)
    got = out.numpy()
    SEEN["cases"] += 1
    SEEN["bits_written"] += bool(wrote_bits)
    SEEN["colsum"] += use_colsum
    SEEN["masked"] += m_np is not None
    # fp64 reference with the same epilogue (bf16 scheme: on bf16-rounded operands)
    xr, wr = (_bf16_rn(xv), _bf16_rn(wv)) if algo == "bf16" else (xv, wv)
    ref = xr.astype(np.float64) @ wr.astype(np.float64).T
    if use_bias:
        ref = ref + bias.numpy().astype(np.float64)
    if relu:
        ref = np.maximum(ref, 0.0)
    if m_np is not None:
        ref = ref * (m_np > 0)
        assert np.all(got[m_np == 0] == 0)
    assert normwise(got, ref) <= TOL[algo], (M, N, K, algo, ta, tb)
    if relu and wrote_bits:
        words = _read(bits_out, M * ((N + 63) // 64), np.uint64).reshape(M, -1)
        yb = got if m_np is None else None
        if yb is not None:  # bits record the ReLU output before any pullback mask
            assert np.array_equal(words, _pack_bits(yb))
    if use_colsum:
        want = got.astype(np.float64).sum(axis=0)
        scale = np.abs(got).astype(np.float64).sum(axis=0) + 1e-30
        assert np.max(np.abs(cs.numpy() - want) / scale) <= 1e-6
    if emit and N % 8 == 0:
        kind = algo
        entry = out.buffer._splits and out.buffer._splits.get((kind, out.offset, M, N, N))
        if entry:
            SEEN["split_checked"] += 1
            hi_ref, lo_ref = _split_ref(got, kind)
            assert np.array_equal(_bf16_arr(entry[1], M * N).reshape(M, N).view(np.uint32),
                                  hi_ref.view(np.uint32))
            if lo_ref is not None:
                assert np.array_equal(_bf16_arr(entry[2], M * N).reshape(M, N).view(np.uint32),
                                      lo_ref.view(np.uint32))


def test_fuzz_covered_the_fused_paths():
    """The random cases above reached the tensor-core epilogue stages."""
    assert SEEN["cases"] >= 30, SEEN
    assert SEEN["bits_written"] >= 5 and SEEN["split_checked"] >= 5, SEEN
    assert SEEN["colsum"] >= 5 and SEEN["masked"] >= 5, SEEN
