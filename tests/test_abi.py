"""CPU checks of the drop-in boundary: libb2.so loads and exports every entry
point include/b2.h declares; the Python binding declares the same set; and
with no GPU every compute call fails loudly (there is no CPU fallback)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "b2.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(b2_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    fns = header_functions()
    for required in ("b2_alloc", "b2_free", "b2_binary", "b2_unary", "b2_reduce", "b2_gemm",
                     "b2_xent_fwd", "b2_xent_bwd", "b2_softmax_fwd", "b2_adam_multi",
                     "b2_sgd_multi", "b2_allreduce_f32", "b2_comm_init"):
        assert required in fns


def test_library_exports_every_header_symbol():
    from paper_2602_00125_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_binding_covers_the_header():
    from paper_2602_00125_b200 import _lib

    assert set(header_functions()) == set(_lib.exported_symbols())


def test_binding_loads_and_binds():
    from paper_2602_00125_b200 import _lib

    L = _lib.lib()
    maj, mnr = ctypes.c_int(), ctypes.c_int()
    assert L.b2_version(ctypes.byref(maj), ctypes.byref(mnr)) == 0


def _has_gpu():
    from paper_2602_00125_b200 import _lib

    n = ctypes.c_int(0)
    _lib.lib().b2_device_count(ctypes.byref(n))
    return n.value > 0


def test_no_cpu_fallback_without_a_device():
    if _has_gpu():
        pytest.skip("a GPU is visible")
    import paper_2602_00125_b200 as P

    with pytest.raises(RuntimeError, match="no CUDA device"):
        P.zeros((2, 2))
    with pytest.raises(RuntimeError):
        P.tensor([1.0, 2.0])


def test_kernels_are_sm100a():
    """The shipped library carries sm_100a SASS with tcgen05/TMA instructions
    (the tensor-core GEMM), bulk copies, and FFMA2 (the FP32 SIMT GEMM's
    two-FMAs-per-instruction inner loop)."""
    import shutil
    import subprocess

    from paper_2602_00125_b200 import _lib

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    for mnem in ("UTCHMMA", "UTMALDG", "LDTM", "UBLKCP", "FFMA2"):
        assert mnem in out, mnem
