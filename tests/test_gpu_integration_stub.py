"""Execute the reference-side ctypes binding shown in INTEGRATION.md verbatim.

The block is what a maintainer would add to tensorlite to route the matmul
seam (pkg/src/tensorlite/core.py:802-807, matmul.block) through libb2. It is
extracted from the document and run as written (B2_LIB points it at the
in-tree library), then fed the reference's own matmul goldens: in the
B2_GEMM_REF mode the seam must return the reference's bits, in auto mode the
fp32 tolerance.
"""

import os
import re

import numpy as np
import pytest

from tests.golden import inputs as I
from tests.golden.load import bits_equal, load, normwise

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub_source():
    with open(os.path.join(ROOT, "INTEGRATION.md")) as f:
        doc = f.read()
    blocks = re.findall(r"```python\n(.*?)```", doc, re.S)
    stub = [b for b in blocks if "def matmul_block" in b]
    assert len(stub) == 1, "INTEGRATION.md must hold exactly one matmul_block stub"
    return stub[0]


def test_integration_stub_runs_verbatim_and_matches_reference_bits(monkeypatch):
    monkeypatch.setenv("B2_LIB", os.path.join(ROOT, "paper_2602_00125_b200", "libb2.so"))
    ns = {"__name__": "tensorlite_b2_stub"}
    exec(compile(_stub_source(), "INTEGRATION.md:stub", "exec"), ns)
    g = load("matmul.npz")
    for i, (x, w, _) in enumerate(I.matmul_cases()):
        want = g[f"m{i}_y"]
        got = ns["matmul_block"](x, w)
        assert got.shape == want.shape
        assert bits_equal(got, want), i
        fast = ns["matmul_block"](x, w, algo=ns["B2_GEMM_AUTO"])
        assert normwise(fast, want) <= 1e-5, i
    # errors surface through b2_last_error (restype c_char_p): a bad extent
    with pytest.raises(RuntimeError, match="libb2: b2_gemm: negative extent"):
        ns["_check"](ns["_b2"].b2_gemm(0, 1, -1, 1, 1, None, 1, None, 1, None, 1, None, 0, 0,
                                       None))
