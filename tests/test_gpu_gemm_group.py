"""Grouped tensor-core GEMM launches (b2_gemm_fused_group): up to three
independent fused GEMMs -- the x_bar and w_bar GEMMs of a matmul pullback
(core.py:815-817 of the reference) -- share one persistent launch whose
units are drawn from one queue. Every output (C, emitted split, relu bits,
column sums) must be BIT-IDENTICAL to launching each descriptor alone with
b2_gemm_fused, for every regime the host policy picks: few tiles (K slices
to fill the chip once), dynamic draws with a long-K problem split into
slices (config 4's dX + dW), dynamic draws of whole tiles (config 5's dX +
dW), mixed operand layouts, all three schemes, and empty problems.
Then the same through the autograd engine: a linear/matmul backward with
grouping on equals the one with grouping off.
"""

import ctypes

import numpy as np
import pytest

import paper_2602_00125_b200 as P
from paper_2602_00125_b200 import _lib as L
from paper_2602_00125_b200 import core as C

pytestmark = pytest.mark.gpu


def _read(ptr, nbytes):
    out = np.empty(nbytes, np.uint8)
    L.call("b2_memcpy_d2h", out.ctypes.data_as(ctypes.c_void_p), ptr, nbytes, None)
    return out


class Problem:
    """One GEMM problem with its own operands and every epilogue output."""

    def __init__(self, rng, M, N, K, ta, tb, algo, *, bias=False, relu=False, mask_bits=False,
                 colsum=False, split=False, bits_out=False):
        self.M, self.N, self.K, self.ta, self.tb, self.algo = M, N, K, ta, tb, algo
        ar, ac = (K, M) if ta else (M, K)
        br, bc = (N, K) if tb else (K, N)
        a = rng.standard_normal((ar, ac), dtype=np.float32)
        b = rng.uniform(-0.05, 0.05, (br, bc)).astype(np.float32)
        self.keep = [P.from_numpy(a), P.from_numpy(b)]
        A, B = self.keep
        if algo == L.GEMM_3XBF16:
            self.a = [P.Buffer(2 * a.size), P.Buffer(2 * a.size)]
            self.b = [P.Buffer(2 * b.size), P.Buffer(2 * b.size)]
            L.call("b2_bf16x3_split", self.a[0].ptr, self.a[1].ptr, A.data_ptr, ar, ac, ac, None)
            L.call("b2_bf16x3_split", self.b[0].ptr, self.b[1].ptr, B.data_ptr, br, bc, bc, None)
            self.lda, self.ldb = ac, bc
        elif algo == L.GEMM_TF32X:
            self.a = [A.buffer, P.Buffer(2 * a.size), P.Buffer(2 * a.size)]
            self.b = [B.buffer, P.Buffer(2 * b.size), P.Buffer(2 * b.size)]
            L.call("b2_bf16x2_split", self.a[1].ptr, self.a[2].ptr, A.data_ptr, ar, ac, ac, None)
            L.call("b2_bf16x2_split", self.b[1].ptr, self.b[2].ptr, B.data_ptr, br, bc, bc, None)
            self.lda, self.ldb = ac, bc
        else:  # BF16 variant
            self.a = [P.Buffer(2 * a.size)]
            self.b = [P.Buffer(2 * b.size)]
            L.call("b2_bf16_cast", self.a[0].ptr, A.data_ptr, ar, ac, ac, None)
            L.call("b2_bf16_cast", self.b[0].ptr, B.data_ptr, br, bc, bc, None)
            self.lda, self.ldb = ac, bc
        self.bias = P.from_numpy(rng.standard_normal(N).astype(np.float32)) if bias else None
        self.epi = ((L.EPI_BIAS_RELU if relu else L.EPI_BIAS) if bias else
                    (L.EPI_RELU if relu else L.EPI_NONE))
        words = (N + 63) // 64
        self.mask_bits = None
        if mask_bits:
            bits = rng.integers(0, 2 ** 63, (M, words), dtype=np.int64)
            self.mask_bits = P.Buffer(8 * M * words)
            L.call("b2_memcpy_h2d", self.mask_bits.ptr, bits.ctypes.data_as(ctypes.c_void_p),
                   bits.nbytes, None)
        self.want = dict(colsum=colsum, split=split, bits_out=bits_out)

    def outputs(self):
        """Fresh output buffers + a descriptor writing them."""
        M, N = self.M, self.N
        o = {"C": P.Buffer(4 * M * N)}
        if self.want["split"]:
            o["hi"] = P.Buffer(2 * M * N)
            if self.algo != L.GEMM_BF16:
                o["lo"] = P.Buffer(2 * M * N)
        if self.want["colsum"]:
            o["cs"] = P.Buffer(4 * N)
        if self.want["bits_out"]:
            o["bits"] = P.Buffer(8 * M * ((N + 63) // 64))
        d = L.GemmDesc()
        d.algo, d.trans_a, d.trans_b, d.M, d.N, d.K = self.algo, self.ta, self.tb, self.M, self.N, self.K
        for i, x in enumerate(self.a):
            d.a[i] = x.ptr
        for i, x in enumerate(self.b):
            d.b[i] = x.ptr
        d.lda, d.ldb, d.C, d.ldc = self.lda, self.ldb, o["C"].ptr, N
        d.bias = self.bias.data_ptr if self.bias is not None else None
        d.epilogue = self.epi
        d.mask_bits = self.mask_bits.ptr if self.mask_bits is not None else None
        d.c_hi = o["hi"].ptr if "hi" in o else None
        d.c_lo = o["lo"].ptr if "lo" in o else None
        d.colsum = o["cs"].ptr if "cs" in o else None
        d.relu_bits_out = o["bits"].ptr if "bits" in o else None
        return d, o


def _group(probs):
    descs, outs = [], []
    for p in probs:
        d, o = p.outputs()
        descs.append(d)
        outs.append(o)
    arr = (L.GemmDesc * len(descs))(*descs)
    L.call("b2_gemm_fused_group", arr, len(descs), None)
    return outs


def _check_group(probs, exact=True):
    """exact: every output bit-identical to separate launches (the group keeps
    each problem's own K partition); else (a group of few tiles, which splits
    K its own way) C within 1e-5 normwise of the separate launches and the
    grouped launch bit-identical when repeated."""
    alone = []
    for p in probs:
        d, o = p.outputs()
        L.call("b2_gemm_fused", ctypes.byref(d), None)
        alone.append(o)
    grouped = _group(probs)
    again = _group(probs) if not exact else grouped
    L.synchronize()
    for i, (a, g, h) in enumerate(zip(alone, grouped, again)):
        for k in a:
            x, y = _read(a[k].ptr, a[k].nbytes), _read(g[k].ptr, g[k].nbytes)
            if exact:
                assert np.array_equal(x, y), f"problem {i} output {k} differs grouped vs alone"
            else:
                assert np.array_equal(y, _read(h[k].ptr, h[k].nbytes)), f"problem {i} {k}: not deterministic"
                if k == "C":
                    xa, ya = x.view(np.float32), y.view(np.float32)
                    assert np.abs(xa - ya).max() <= 1e-5 * np.abs(xa).max()


def test_group_few_tiles_config3_shape():
    """n = 1024 dA (NN) + dB (TN): few tiles -> the group fills the chip once
    with K slices of its own (one unit per CTA)."""
    rng = np.random.default_rng(1)
    _check_group([Problem(rng, 1024, 1024, 1024, 0, 0, L.GEMM_3XBF16),
                  Problem(rng, 1024, 1024, 1024, 1, 1, L.GEMM_3XBF16)], exact=False)


def test_group_dynamic_long_k_split_config4_shape():
    """dX [8192 x 1024, K = 1024] + dW [1024 x 1024, K = 8192] with the bias
    gradient: the long-K problem is sliced, units drawn dynamically."""
    rng = np.random.default_rng(2)
    _check_group([Problem(rng, 8192, 1024, 1024, 0, 0, L.GEMM_3XBF16, split=True, colsum=True),
                  Problem(rng, 1024, 1024, 8192, 1, 1, L.GEMM_3XBF16)])


def test_group_dynamic_whole_tiles_config5_head_shape():
    """config-5 head pullback shape at a smaller batch: dX with the ReLU
    pullback from bits, column sums and split emission + dW (K = batch)."""
    rng = np.random.default_rng(3)
    _check_group([Problem(rng, 8192, 2048, 1000, 0, 0, L.GEMM_3XBF16, mask_bits=True, colsum=True,
                          split=True),
                  Problem(rng, 1000, 2048, 8192, 1, 0, L.GEMM_3XBF16)])


def test_group_three_problems_mixed_epilogues():
    rng = np.random.default_rng(4)
    _check_group([Problem(rng, 2048, 1536, 512, 0, 1, L.GEMM_3XBF16, bias=True, relu=True,
                          bits_out=True, split=True),
                  Problem(rng, 520, 264, 4096, 1, 0, L.GEMM_3XBF16, colsum=True),
                  Problem(rng, 3000, 2056, 256, 0, 0, L.GEMM_3XBF16, bias=True)])


@pytest.mark.parametrize("algo", ["tf32x", "bf16"])
def test_group_other_schemes(algo):
    a = {"tf32x": L.GEMM_TF32X, "bf16": L.GEMM_BF16}[algo]
    rng = np.random.default_rng(5)
    _check_group([Problem(rng, 4096, 2048, 1024, 0, 0, a, split=True, colsum=True),
                  Problem(rng, 2048, 1024, 4096, 1, 1, a)])


def test_group_skips_empty_and_rejects_mixed_algos():
    rng = np.random.default_rng(6)
    p = Problem(rng, 1024, 512, 256, 0, 1, L.GEMM_3XBF16)
    d, o = p.outputs()
    empty = L.GemmDesc()
    empty.algo, empty.M, empty.N, empty.K = L.GEMM_3XBF16, 0, 512, 256
    arr = (L.GemmDesc * 2)(d, empty)
    L.call("b2_gemm_fused_group", arr, 2, None)
    q = Problem(rng, 1024, 512, 256, 0, 1, L.GEMM_BF16)
    d2, _ = q.outputs()
    with pytest.raises(Exception, match="differ in algo"):
        L.call("b2_gemm_fused_group", (L.GemmDesc * 2)(d, d2), 2, None)
    with pytest.raises(Exception, match="1 to 3"):
        L.call("b2_gemm_fused_group", (L.GemmDesc * 1)(d), 4, None)


@pytest.mark.parametrize("shape", [(1024, 1024, 1024), (8192, 1024, 1024), (2048, 4096, 1000)])
def test_autograd_backward_grouped_equals_ungrouped(monkeypatch, shape):
    """A Linear(+ReLU) -> Linear chain's backward: the engine groups each
    node's x_bar/w_bar GEMMs; gradients bit-identical with grouping off
    (within 1e-5 for the few-tile shape, whose group splits K its own way)."""
    M, K, N = shape
    rng = np.random.default_rng(7)
    x = P.from_numpy(rng.standard_normal((M, K), dtype=np.float32), requires_grad=True)
    w1 = P.from_numpy(rng.uniform(-0.03, 0.03, (N, K)).astype(np.float32), requires_grad=True)
    b1 = P.from_numpy(rng.uniform(-0.1, 0.1, N).astype(np.float32), requires_grad=True)
    w2 = P.from_numpy(rng.uniform(-0.03, 0.03, (512, N)).astype(np.float32), requires_grad=True)
    seed = P.from_numpy(rng.standard_normal((M, 512), dtype=np.float32))

    def grads(on):
        monkeypatch.setattr(C, "_GROUP_ON", on)
        P.reset_tape()
        h = C.linear(x, w1, b1, relu_out=True)
        y = C.matmul(h, w2)
        st = P.backward(y, seed=seed)
        return [st[t].numpy() for t in (x, w1, b1, w2)]

    on, off, on2 = grads(True), grads(False), grads(True)
    for a, b, c in zip(on, off, on2):
        assert np.array_equal(a.view(np.uint32), c.view(np.uint32))
        if M * N >= 8192 * 1024:
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        else:
            assert np.abs(a - b).max() <= 1e-5 * np.abs(b).max()


def test_cluster_split_k_bit_identical_to_l2_partials(tmp_path):
    """Few-tile GEMMs whose K slices fold through distributed shared memory
    inside a cluster (B2_GEMM_CSPLIT, default on) give the same bits -- C,
    emitted split, relu bits, column sums -- as the K-slice partials through
    L2 + k_tail_epilogue, for 2 / 4 / 8 slices, ragged edges and every
    epilogue stage."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        f = tmp_path / f"cs{flag}.npz"
        env = dict(os.environ, B2_GEMM_CSPLIT=flag, PYTHONPATH=root)
        r = subprocess.run([sys.executable, os.path.join(root, "tests", "csplit_cases.py"), str(f)],
                           env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    a, b = outs
    assert set(a.files) == set(b.files)
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k


def test_bf16_512_row_pair_tiles_match_256_row_tiles(tmp_path):
    """The bf16 variant's 512-row pair tiles (MODE 6, default for big launches)
    give the 256-row path's bits -- C, its bf16 cast, relu bits, column sums --
    for K <= 4096 (one accumulation chunk either way), ragged M/N included;
    beyond (one chunk instead of K = 4096 promotion) within bf16 noise."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        f = tmp_path / f"m2_{flag}.npz"
        env = dict(os.environ, B2_GEMM_M2=flag, PYTHONPATH=root)
        r = subprocess.run([sys.executable, os.path.join(root, "tests", "m2_cases.py"), str(f)],
                           env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    a, b = outs
    for k in a.files:
        if k.startswith("2_"):  # K = 16384: 4 promotion chunks vs one
            if k == "2_C":
                x, y = a[k].view(np.float32), b[k].view(np.float32)
                assert np.abs(x - y).max() <= 1e-4 * np.abs(y).max()
            continue
        assert np.array_equal(a[k], b[k]), k
